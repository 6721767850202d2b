"""B200-native Noise2Fast fit-and-denoise (drop-in for noise2fast.trainer's hot path).

The compute runs in hand-written sm_100a CUDA kernels behind the C ABI in
``include/n2f.h`` (``libn2f.so``); this package is the host-side mirror of the
reference's trainer interface.
"""

from .trainer import (  # noqa: F401
    DenoiseResult,
    Engine,
    ImageData,
    TrainConfig,
    denoise_image,
    derive_seed,
    install,
    release_engines,
    train_single_channel,
)

__all__ = [
    "DenoiseResult",
    "Engine",
    "ImageData",
    "TrainConfig",
    "denoise_image",
    "derive_seed",
    "install",
    "release_engines",
    "train_single_channel",
]
