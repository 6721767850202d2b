"""No-op pyplot: every axes/figure call is accepted; savefig writes a
signature-only PNG placeholder at the requested path (the reference's report
tests check that non-empty figure files exist)."""

from pathlib import Path

_PNG = b"\x89PNG\r\n\x1a\n"  # a signature-only placeholder (no pixels are rendered)


class _Any:
    def __getattr__(self, name):
        return _Any()

    def __call__(self, *args, **kwargs):
        return _Any()

    def __getitem__(self, key):
        return _Any()

    def __iter__(self):
        return iter(())


class _Fig(_Any):
    def savefig(self, path, *args, **kwargs):
        Path(path).write_bytes(_PNG)


def subplots(*args, **kwargs):
    return _Fig(), _Any()


def figure(*args, **kwargs):
    return _Fig()


def savefig(path, *args, **kwargs):
    Path(path).write_bytes(_PNG)


def close(*args, **kwargs):
    return None
