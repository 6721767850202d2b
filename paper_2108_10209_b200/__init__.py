"""B200-native Noise2Fast fit-and-denoise (drop-in for noise2fast.trainer's hot path).

The compute runs in hand-written sm_100a CUDA kernels behind the C ABI in
``include/n2f.h`` (``libn2f.so``); this package is the host-side mirror of the
reference's trainer interface.
"""

from .imageio import ImageFormatError, from_plane, load_image, save_image  # noqa: F401
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
    "ImageFormatError",
    "TrainConfig",
    "denoise_image",
    "derive_seed",
    "from_plane",
    "install",
    "load_image",
    "release_engines",
    "save_image",
    "train_single_channel",
]
