"""Minimal stand-in for matplotlib (not installed in this image) so that the
reference's `noise2fast.report` -- and through it `noise2fast.cli` -- import.
Test infrastructure only: figures are written as empty files, the CSV and
manifest outputs of the reference CLI are untouched."""


def use(*args, **kwargs):
    return None
