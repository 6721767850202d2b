"""Host-side mirror of the reference trainer API, running on the B200 engine.

Same names, argument meaning, return types and error behaviour as the
reference module ``noise2fast.trainer`` (pkg/src/noise2fast/trainer.py):

* ``TrainConfig``            (trainer.py:29-51)  -- same fields, same checks
* ``DenoiseResult``          (trainer.py:69-75)
* ``train_single_channel``   (trainer.py:125-213) -- the hot path, one call
  into ``libn2f.so``: the whole fit (normalise, pairs, init, every epoch,
  validation, early stopping, window mean) runs on the GPU as one CUDA
  graph; the host only validates arguments and formats the result
* ``denoise_image``          (trainer.py:216-250) -- per (slice, channel)
  fan-out with ``derive_seed(config.seed, ch, sl)`` seeds

``install()`` rebinds ``noise2fast.trainer.train_single_channel`` (the module
global that ``denoise_image`` and the CLI jobs look up, trainer.py:241) so an
installed reference package runs on this engine.
"""

from __future__ import annotations

import contextlib
import dataclasses
import fcntl
import json
import os
import tempfile
import threading
import time
from dataclasses import dataclass

import numpy as np

from .imageio import ImageData  # noqa: F401  (re-exported; imaging.py:26)
from . import _lib
from ._lib import N2FConfig, N2FResult, STOP_REASONS, call, load

_LOSSES = ("bce", "mse")
_SCHEMES = ("checkerboard", "quad", "exact")
_M64 = 0xFFFFFFFFFFFFFFFF


@dataclass
class TrainConfig:
    loss: str = "bce"
    scheme: str = "checkerboard"
    lr: float = 0.001
    patience_epochs: int = 100
    avg_window: int = 100
    max_epochs: int = 20000
    seed: int = 0

    def __post_init__(self):
        if self.loss not in _LOSSES:
            raise ValueError(f"loss must be one of {_LOSSES}, got {self.loss!r}")
        if self.scheme not in _SCHEMES:
            raise ValueError(f"scheme must be one of {_SCHEMES}, got {self.scheme!r}")
        if self.lr <= 0:
            raise ValueError("lr must be > 0")
        if self.patience_epochs < 1:
            raise ValueError("patience_epochs must be >= 1")
        if self.avg_window < 1:
            raise ValueError("avg_window must be >= 1")
        if self.max_epochs < 1:
            raise ValueError("max_epochs must be >= 1")


@dataclass
class DenoiseResult:
    denoised: np.ndarray  # 2-D, original value scale, float64
    epochs_run: int
    val_history: list
    wall_time: float
    stop_reason: str  # "patience" | "max_epochs" | "degenerate"


# ---------------------------------------------------------------------------
# seeds (rng.py:20-39) -- integer SplitMix64, needed for denoise_image fan-out
# ---------------------------------------------------------------------------


def _mix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_seed(seed: int, *ids: int) -> int:
    acc = seed & _M64
    for i in ids:
        acc = _mix64(acc ^ (i & _M64))
    return acc


# ---------------------------------------------------------------------------
# engine contexts (one per process/device/shape/config, reused across images)
# ---------------------------------------------------------------------------


def _worker_ordinal() -> int:
    """0-based index of this process among a multiprocessing pool's workers
    (the reference CLI's spawn pool, cli.py:207-211), 0 outside a pool."""
    import multiprocessing as mp

    ident = getattr(mp.current_process(), "_identity", ())
    return ident[0] - 1 if ident else 0


def select_device(spec: str | None, ordinal: int, count: int) -> int:
    """GPU for this process: N2F_DEVICE=<k> pins device k; N2F_DEVICE=auto maps
    pool worker i to device i mod count (so ``--threads N`` on an N-GPU box
    runs one image per GPU at a time, BASELINE config 4); unset means 0."""
    if spec is None or spec == "":
        return 0
    if spec == "auto":
        if count < 1:
            raise RuntimeError("N2F_DEVICE=auto: no CUDA device visible")
        return ordinal % count
    return int(spec)


def _device_index() -> int:
    spec = os.environ.get("N2F_DEVICE")
    if spec != "auto":
        return select_device(spec, 0, 1)
    n = _lib.C.c_int()
    call("n2f_device_count", _lib.C.byref(n))
    return select_device(spec, _worker_ordinal(), n.value)


_lock_fds: dict[int, int] = {}


@contextlib.contextmanager
def _device_lock(device: int):
    """Inter-process lock per GPU around one fit of the public API.  Processes
    that share a GPU (the reference CLI's ``--threads N`` pool with fewer GPUs
    than workers) then take turns: one fit saturates a B200, so concurrent fits
    gain nothing, and two contexts time-slicing the persistent tcgen05 /
    while-graph kernels of a 512^2 fit were seen to stall for minutes."""
    fd = _lock_fds.get(device)
    if fd is None:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "all").replace(",", "_").replace("/", "_")
        path = os.path.join(tempfile.gettempdir(), f"n2f_b200_gpu_{vis}_{device}.lock")
        fd = os.open(path, os.O_CREAT | os.O_RDWR, 0o666)
        _lock_fds[device] = fd
    fcntl.flock(fd, fcntl.LOCK_EX)
    try:
        yield
    finally:
        fcntl.flock(fd, fcntl.LOCK_UN)


class Engine:
    """Owns one libn2f context: workspaces + the captured CUDA graph."""

    def __init__(self, height: int, width: int, config, device: int | None = None,
                 use_graph: bool = True):
        lib = load()
        self.height, self.width = int(height), int(width)
        self.device = _device_index() if device is None else int(device)
        cfg = N2FConfig()
        cfg.loss = _LOSSES.index(config.loss)
        cfg.scheme = _SCHEMES.index(config.scheme)
        cfg.lr = float(config.lr)
        cfg.patience_epochs = int(config.patience_epochs)
        cfg.avg_window = int(config.avg_window)
        cfg.max_epochs = int(config.max_epochs)
        cfg.conv_impl = 0  # tcgen05 FP16x3, the library's only implementation
        cfg.seed = int(config.seed) & _M64
        cfg.use_graph = 1 if use_graph else 0
        self.cfg = cfg
        self.max_epochs = int(config.max_epochs)
        h = _lib.C.c_void_p()
        call("n2f_create", self.device, self.height, self.width, _lib.C.byref(cfg), _lib.C.byref(h))
        self.handle = h
        self._lib = lib

    def close(self):
        if getattr(self, "handle", None):
            self._lib.n2f_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return self._lib.n2f_ctx_stream(self.handle) or 0

    @property
    def device_bytes(self) -> int:
        return int(self._lib.n2f_ctx_device_bytes(self.handle))

    def _result_struct(self):
        n = self.max_epochs
        hist = np.zeros(n, np.float64)
        losses = np.zeros(4 * n, np.float64)
        secs = np.zeros(n, np.float64)
        r = N2FResult()
        r.val_history = hist.ctypes.data_as(_lib.C.POINTER(_lib.C.c_double))
        r.train_loss = losses.ctypes.data_as(_lib.C.POINTER(_lib.C.c_double))
        r.epoch_seconds = secs.ctypes.data_as(_lib.C.POINTER(_lib.C.c_double))
        return r, hist, losses, secs

    def fit_host(self, image: np.ndarray, clean: np.ndarray | None = None):
        """Whole fit from host arrays (float32 or float64, C-contiguous)."""
        dtype = _lib.N2F_F64 if image.dtype == np.float64 else _lib.N2F_F32
        out = np.empty((self.height, self.width), np.float64)
        r, hist, losses, secs = self._result_struct()
        call("n2f_fit_denoise_host", self.handle, image.ctypes.data,
             dtype, clean.ctypes.data if clean is not None else None, out.ctypes.data,
             _lib.C.byref(r))
        n = r.epochs_run
        return out, r, hist[:n].copy(), losses[: 4 * n].reshape(n, 4).copy(), secs[:n].copy()

    def set_seed(self, seed: int) -> None:
        """Network seed of the next fit (TrainConfig.seed)."""
        self.cfg.seed = int(seed) & _M64
        call("n2f_ctx_set_seed", self.handle, self.cfg.seed)

    def params(self) -> np.ndarray:
        """The parameter arena (w0, b0, ..., w8, b8; weights K-major) on the host."""
        out = np.empty(self.param_count(), np.float32)
        call("n2f_ctx_get_arena", self.handle, 0, out.ctypes.data)
        return out

    def param_count(self) -> int:
        n = _lib.C.c_int64()
        call("n2f_ctx_param_count", self.handle, _lib.C.byref(n))
        return n.value

    def set_params(self, arena: np.ndarray) -> None:
        """Overwrite the parameters (resets Adam moments, step count and stop state)."""
        a = np.ascontiguousarray(arena, np.float32).reshape(-1)
        if a.size != self.param_count():
            raise ValueError(f"parameter arena has {a.size} values, the network has {self.param_count()}")
        call("n2f_ctx_set_params", self.handle, a.ctypes.data)

    def range_history(self) -> np.ndarray:
        """FP16x3 range guard record of the epochs run since the last init /
        set_params: [epochs, 4 classes (act, val_act, grad, weight), 9 layers]
        max |x * 2^e| of the fp16 operand pairs written (0 = none)."""
        buf = np.zeros((self.max_epochs, _lib.N2F_RANGE_SLOTS), np.float32)
        n = _lib.C.c_int()
        call("n2f_ctx_range_history", self.handle, buf.ctypes.data, self.max_epochs, _lib.C.byref(n))
        return buf[: n.value].reshape(n.value, 4, 9).copy()

    def save_checkpoint(self, path) -> None:
        """N2FW v1 checkpoint of the current parameters (model.py:143-152).
        The header's seed is the loaded checkpoint's, else this engine's."""
        from . import checkpoint

        seed = self.checkpoint_seed if self.checkpoint_seed is not None else self.cfg.seed
        checkpoint.save_checkpoint(self.params(), path, seed)

    checkpoint_seed = None

    def load_checkpoint(self, path) -> None:
        """Load an N2FW v1 checkpoint into this context (model.py:155-184)."""
        from . import checkpoint

        arena, seed, in_channels = checkpoint.load_checkpoint(path)
        if in_channels != 1:
            raise ValueError(f"checkpoint has in_channels={in_channels}; this engine fits "
                             "single-channel planes (in_channels=1)")
        self.set_params(arena)
        self.checkpoint_seed = int(seed)

    PROF_CLASSES = ("first_fwd", "conv_fwd", "head_loss", "wgrad", "dgrad", "first_wgrad", "adam",
                    "val_first", "val_conv", "val_head", "stop")

    def profile_epoch(self):
        """One more training epoch with CUDA events around every launch:
        (ms, flop, launches) arrays indexed [class, layer] (PROF_CLASSES x 9)."""
        n = len(self.PROF_CLASSES) * 9
        ms, fl = np.zeros(n), np.zeros(n)
        ln = np.zeros(n, np.int32)
        call("n2f_ctx_profile_epoch", self.handle, ms.ctypes.data, fl.ctypes.data, ln.ctypes.data)
        shape = (len(self.PROF_CLASSES), 9)
        return ms.reshape(shape), fl.reshape(shape), ln.reshape(shape)

    def fit_device(self, image_ptr: int, dtype: int, out_ptr: int, clean_ptr: int | None = None):
        """Whole fit on device-resident buffers (used by the bench's `value`)."""
        r = N2FResult()
        call("n2f_fit_denoise_dev", self.handle, image_ptr, dtype, clean_ptr, out_ptr,
             _lib.C.byref(r))
        return r


_cache_lock = threading.Lock()
_cache: dict = {}


def _engine_for(shape, config) -> Engine:
    # the seed is set per fit (n2f_ctx_set_seed): one context serves every
    # seed of a shape/config (denoise_image's per-channel seeds, CLI files)
    key = (shape, config.loss, config.scheme, float(config.lr), int(config.patience_epochs),
           int(config.avg_window), int(config.max_epochs), _device_index())
    with _cache_lock:
        eng = _cache.get(key)
        if eng is None:
            # keep one live context: large images own tens of GB of workspace
            for k in list(_cache):
                _cache.pop(k).close()
            eng = Engine(shape[0], shape[1], config)
            _cache[key] = eng
        eng.set_seed(config.seed)
        return eng


def release_engines() -> None:
    with _cache_lock:
        for k in list(_cache):
            _cache.pop(k).close()


# ---------------------------------------------------------------------------
# reference-facing API
# ---------------------------------------------------------------------------


def _write_telemetry(sink, record: dict) -> None:
    if sink is not None:
        sink.write(json.dumps(record) + "\n")


def train_single_channel(noisy, config, clean=None, telemetry=None, telemetry_tags=None) -> DenoiseResult:
    """Denoise one 2-D image by training a fresh network on it (on the GPU).

    Drop-in for ``noise2fast.trainer.train_single_channel`` (trainer.py:125-213):
    ``config`` may be this module's TrainConfig or the reference's.
    """
    t0 = time.perf_counter()
    arr = np.asarray(noisy)
    if arr.dtype not in (np.float32, np.float64):
        arr = np.asarray(arr, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"expected a 2-D image, got shape {arr.shape}")
    if arr.shape[0] < 4 or arr.shape[1] < 4:
        raise ValueError(f"image must be at least 4x4, got {arr.shape}")
    # checked here (before any engine work: a NaN image must not evict a
    # cached context, trainer.py:142-143); the device min/max scan re-checks
    if not np.isfinite(arr).all():
        raise ValueError("image contains non-finite values")
    clean_arr = None
    if config.scheme == "exact":
        if clean is None:
            raise ValueError("the exact scheme requires the clean ground-truth image")
        clean_arr = np.asarray(clean, dtype=np.float64)
        if clean_arr.shape != arr.shape:
            raise ValueError(f"clean shape {clean_arr.shape} != noisy shape {arr.shape}")
        arr = np.asarray(arr, dtype=np.float64)
    arr = np.ascontiguousarray(arr)
    if clean_arr is not None:
        clean_arr = np.ascontiguousarray(clean_arr)

    eng = _engine_for(arr.shape, config)
    wall0 = time.time()
    try:
        with _device_lock(eng.device):
            out, r, hist, losses, secs = eng.fit_host(arr, clean_arr)
    except _lib.N2FError as e:
        if e.code == _lib.N2F_ERR_NONFINITE:
            raise ValueError("image contains non-finite values") from None
        if e.code == _lib.N2F_ERR_ARG:
            raise ValueError(e.msg) from None
        if e.code == _lib.N2F_ERR_RANGE:
            # an fp16 operand pair would have overflowed: never return the NaN
            # image the fit would otherwise produce
            raise FloatingPointError(e.msg) from None
        raise
    reason = STOP_REASONS[r.stop_reason]
    if reason == "degenerate":
        return DenoiseResult(out, 0, [], time.perf_counter() - t0, "degenerate")
    tags = telemetry_tags or {}
    if telemetry is not None:
        for e in range(r.epochs_run):
            _write_telemetry(telemetry, {
                **tags,
                "epoch": e + 1,
                "train_loss_per_pair": [float(v) for v in losses[e]],
                "val_mse": float(hist[e]),
                "timestamp": wall0 + float(secs[e]),
            })
    return DenoiseResult(
        denoised=out,
        epochs_run=int(r.epochs_run),
        val_history=[float(v) for v in hist],
        wall_time=time.perf_counter() - t0,
        stop_reason=reason,
    )


def denoise_image(image, config, clean=None, telemetry=None):
    """Denoise every channel of every slice with independent runs (trainer.py:216-250)."""
    if not 1 <= image.channels <= 4:
        raise ValueError(f"expected 1-4 channels, got {image.channels}")
    if config.scheme == "exact":
        if clean is None:
            raise ValueError("the exact scheme requires the clean ground-truth image")
        if clean.samples.shape != image.samples.shape:
            raise ValueError("clean image layout differs from noisy image")
    out = np.empty_like(image.samples, dtype=np.float32)
    runs = []
    for sl in range(image.n_slices):
        for ch in range(image.channels):
            sub = dataclasses.replace(config, seed=derive_seed(config.seed, ch, sl))
            result = train_single_channel(
                image.samples[sl, :, :, ch],
                sub,
                clean=None if clean is None else clean.samples[sl, :, :, ch],
                telemetry=telemetry,
                telemetry_tags={"slice": sl, "channel": ch},
            )
            out[sl, :, :, ch] = result.denoised
            runs.append(result)
    return type(image)(out, image.bit_depth, image.data_range), runs


def install(metrics: bool = True) -> None:
    """Route the installed reference package's hot path through this engine.

    Rebinds the module global ``noise2fast.trainer.train_single_channel``
    (looked up at call time by ``denoise_image``, trainer.py:241, and hence by
    the CLI jobs, cli.py:147/175).  Spawned CLI workers: see INTEGRATION.md.
    """
    import noise2fast.trainer as ref_trainer

    ref_trainer.train_single_channel = train_single_channel
    if metrics:
        # benchmark-mode metrics (cli.py:113-139 looks them up on the module)
        import noise2fast.imaging as ref_imaging

        from . import metrics as m

        ref_imaging.psnr = m.psnr
        ref_imaging.ssim = m.ssim
