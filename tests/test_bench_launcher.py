"""bench.py's multi-GPU plumbing on CPU: `--gpus N` without a torchrun
environment launches N ranks itself (one process per GPU), joins them in a
gloo group (no NCCL: images share nothing) and reports the job from rank 0;
`--dry-run` skips only the GPU work."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_launches_two_ranks_with_gloo():
    d = _run("--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "0")
    assert d["n_gpus"] == 2 and d["backend"] == "gloo"
    assert len(set(d["rank_pids"])) == 2 and os.getpid() not in d["rank_pids"]


def test_bench_single_process_default():
    d = _run("--dry-run", "--steps", "1", "--warmup", "0")
    assert d["n_gpus"] == 1 and d["backend"] == "none" and len(d["rank_pids"]) == 1
