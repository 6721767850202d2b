"""Opt-in interpreter hook: with N2F_B200_INSTALL=1 and this directory on
PYTHONPATH, every Python process (including the reference CLI's spawned
worker processes, cli.py:207-211) routes noise2fast.trainer's hot path
through the B200 engine at start-up.  See INTEGRATION.md."""

import os

if os.environ.get("N2F_B200_INSTALL") == "1":
    try:
        import paper_2108_10209_b200

        paper_2108_10209_b200.install()
    except ImportError:  # reference package not importable in this process
        pass
