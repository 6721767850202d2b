"""pytest plugin for running the REFERENCE's own test suite against this
engine: loaded with `-p n2f_install_plugin` before any test module is
imported (the reference tests bind `train_single_channel` at import,
test_trainer.py:10-19), it routes the installed reference package through
the B200 engine with `install()` and counts the engine fits the suite runs.
The spawned CLI workers get the same routing from the autoinstall
sitecustomize hook (N2F_B200_INSTALL=1)."""

import functools
import json
import os

import noise2fast.trainer as _ref_trainer

import paper_2108_10209_b200 as _n2f
from paper_2108_10209_b200 import trainer as _eng

_n2f.install()
assert _ref_trainer.train_single_channel is _eng.train_single_channel

FITS = {"n": 0, "epochs": 0}
_orig = _eng.train_single_channel


@functools.wraps(_orig)
def _counted(*args, **kwargs):
    res = _orig(*args, **kwargs)
    FITS["n"] += 1
    FITS["epochs"] += int(res.epochs_run)
    return res


_counted.__n2f_engine__ = True
_ref_trainer.train_single_channel = _counted


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("N2F_REFSUITE_REPORT")
    if out:
        with open(out, "w") as f:
            json.dump({"engine_fits": FITS["n"], "engine_epochs": FITS["epochs"],
                       "routed": getattr(_ref_trainer.train_single_channel, "__n2f_engine__", False),
                       "exitstatus": int(exitstatus)}, f)
