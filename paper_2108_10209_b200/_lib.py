"""ctypes binding of libn2f.so (include/n2f.h).

There is deliberately no fallback: if the CUDA library is missing or cannot
be loaded, every entry point raises.  Build it with
``python -m paper_2108_10209_b200.build``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("N2F_LIB") or os.path.join(_HERE, "libn2f.so")  # N2F_LIB: A/B variants

(N2F_OK, N2F_ERR_ARG, N2F_ERR_NONFINITE, N2F_ERR_CUDA, N2F_ERR_OOM, N2F_ERR_UNSUPPORTED,
 N2F_ERR_RANGE) = range(7)
N2F_RANGE_SLOTS = 36  # range guard: class * 9 + layer (include/n2f.h)
RANGE_CLASSES = ("act", "val_act", "grad", "weight")
N2F_F32, N2F_F64 = 0, 1
STOP_REASONS = {0: "patience", 1: "max_epochs", 2: "degenerate"}


class N2FConfig(C.Structure):
    _fields_ = [
        ("loss", C.c_int32),
        ("scheme", C.c_int32),
        ("lr", C.c_double),
        ("patience_epochs", C.c_int32),
        ("avg_window", C.c_int32),
        ("max_epochs", C.c_int32),
        ("conv_impl", C.c_int32),
        ("seed", C.c_uint64),
        ("use_graph", C.c_int32),
        ("reserved", C.c_int32 * 7),
    ]


class N2FResult(C.Structure):
    _fields_ = [
        ("epochs_run", C.c_int32),
        ("stop_reason", C.c_int32),
        ("vmin", C.c_double),
        ("vmax", C.c_double),
        ("best_score", C.c_double),
        ("val_history", C.POINTER(C.c_double)),
        ("train_loss", C.POINTER(C.c_double)),
        ("epoch_seconds", C.POINTER(C.c_double)),
        ("gpu_ms", C.c_double),
        ("kernel_launches", C.c_int64),
    ]


class N2FError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[n2f status {code}] {msg}")
        self.code = code
        self.msg = msg


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double
_FP = C.POINTER(C.c_float)

# name -> argtypes (all return int status unless listed in _RESTYPES)
SIGNATURES = {
    "n2f_last_error": [],
    "n2f_version": [],
    "n2f_create": [_I, _I, _I, C.POINTER(N2FConfig), C.POINTER(_P)],
    "n2f_destroy": [_P],
    "n2f_ctx_stream": [_P],
    "n2f_ctx_device_bytes": [_P],
    "n2f_fit_denoise_dev": [_P, _P, _I, _P, _P, C.POINTER(N2FResult)],
    "n2f_fit_denoise_host": [_P, _P, _I, _P, _P, C.POINTER(N2FResult)],
    "n2f_minmax": [_P, _I, _I64, _P, _P],
    "n2f_make_pairs": [_P, _I, _P, _I, _I, _D, _D, _I, _I, _P, _P, _P, _P, _P, _P],
    "n2f_init_layer": [C.c_uint64, _I, _I, _I, _I, _P, _P],
    "n2f_conv_fwd": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P],
    "n2f_conv_bwd": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P],
    "n2f_loss": [_P, _P, _P, _I64, _I, _P, _P],
    "n2f_adam": [_P, _P, _P, _P, _I64, _I, _D, _P],
    "n2f_validate_tail": [_P, _P, _P, _I64, _P, _P],
    "n2f_stop_replay": [_P, _I, _I, _P],
    "n2f_window_mean": [_P, _I, _I, _I, _I64, _D, _D, _P, _P],
    "n2f_ctx_prepare": [_P, _P, _I, _P, _I],
    "n2f_ctx_param_count": [_P, _P],
    "n2f_ctx_get_arena": [_P, _I, _P],
    "n2f_ctx_set_params": [_P, _P],
    "n2f_ctx_set_arena": [_P, _I, _P, _I],
    "n2f_ctx_step": [_P, _I, _P],
    "n2f_ctx_epoch": [_P, _P],
    "n2f_ctx_profile_epoch": [_P, _P, _P, _P],
    "n2f_ctx_validate": [_P, _P, _P],
    "n2f_ctx_get_pairs": [_P, _P, _P, _P, _P, _P],
    "n2f_sq_err_sum": [_P, _P, _I64, _P, _P],
    "n2f_psnr": [_P, _P, _I64, _D, _P, _P],
    "n2f_ssim": [_P, _P, _I, _I, _D, _D, _D, _P, _P],
    "n2f_device_count": [_P],
    "n2f_ctx_set_seed": [_P, C.c_uint64],
    "n2f_ctx_range_history": [_P, _P, _I, C.POINTER(C.c_int)],
    "n2f_ctx_check_guards": [_P, C.POINTER(C.c_int)],
}
_RESTYPES = {
    "n2f_last_error": C.c_char_p,
    "n2f_version": C.c_char_p,
    "n2f_ctx_stream": C.c_void_p,
    "n2f_ctx_device_bytes": C.c_size_t,
}

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load libn2f.so once; raise loudly if it is not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is not built; run `python -m paper_2108_10209_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def check(status: int) -> None:
    if status != N2F_OK:
        msg = load().n2f_last_error().decode(errors="replace")
        raise N2FError(status, msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr(a) -> int:
    """Raw address of a numpy array or a torch tensor."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
