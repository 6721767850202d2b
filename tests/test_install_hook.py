"""The drop-in wiring into the installed reference package:
``install()`` rebinds ``noise2fast.trainer.train_single_channel`` and the
benchmark metrics, and the opt-in ``sitecustomize`` hook does it in every
interpreter, including the reference CLI's ``spawn`` pool workers
(cli.py:207-211).  CPU-only; needs the reference tree (this container), so it
skips where /root/reference is absent (the GPU box)."""

import os
import subprocess
import sys
import textwrap

import pytest

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")

SCRIPT = textwrap.dedent("""
    import multiprocessing as mp

    def routed():
        import noise2fast.imaging as im
        import noise2fast.trainer as t
        import paper_2108_10209_b200 as n
        return (t.train_single_channel is n.train_single_channel,
                im.psnr.__module__ == "paper_2108_10209_b200.metrics")

    def child(q):
        q.put(routed())

    if __name__ == "__main__":
        print("main", *routed())
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=child, args=(q,))
        p.start()
        print("worker", *q.get(timeout=120))
        p.join()
""")


def test_sitecustomize_hook_routes_main_and_spawned_workers(tmp_path):
    script = tmp_path / "probe.py"
    script.write_text(SCRIPT)
    env = dict(os.environ)
    env.update(
        PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "paper_2108_10209_b200", "autoinstall"), ROOT,
                                    REF_SRC]),
        N2F_B200_INSTALL="1", PYTHONDONTWRITEBYTECODE="1", NUMBA_CACHE_DIR=str(tmp_path / "nbc"))
    out = subprocess.run([sys.executable, str(script)], env=env, cwd=tmp_path, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.split("\n")
    assert "main True True" in lines and "worker True True" in lines, out.stdout


def test_install_without_hook_leaves_reference_untouched(tmp_path):
    """Without N2F_B200_INSTALL the reference runs its own code."""
    env = dict(os.environ)
    env.pop("N2F_B200_INSTALL", None)
    env.update(PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "paper_2108_10209_b200", "autoinstall"),
                                           ROOT, REF_SRC]),
               PYTHONDONTWRITEBYTECODE="1", NUMBA_CACHE_DIR=str(tmp_path / "nbc"))
    code = ("import noise2fast.trainer as t; "
            "print(t.train_single_channel.__module__)")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=tmp_path, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == "noise2fast.trainer"
