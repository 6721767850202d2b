"""Image containers for the drop-in path: the decoded-image record that
``denoise_image`` consumes and the PNG / TIFF codecs around it (SURVEY.md §8
(f)#4; the reference's are ``imaging.py:26-88`` and ``imaging.py:98-163``).

Host-side only (Pillow does the container work, as in the reference); files
written here are byte-identical to the reference's for the same samples
(``tests/test_imageio.py`` checks that against the installed reference).

Layout: ``samples[slice, y, x, channel]`` float32.  ``bit_depth`` names the
container's sample type ("uint8", "uint16", "float32"); ``data_range`` is the
nominal range of integer data (255, 65535) or None for float data.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

_DEPTHS = {"uint8": (255.0, np.uint8), "uint16": (65535.0, np.uint16), "float32": (None, np.float32)}
# Pillow mode <-> (container, depth / channel count) accepted by the reference
_PNG_CHANNELS = {"L": 1, "RGB": 3}
_TIFF_DEPTH = {"L": "uint8", "I;16": "uint16", "F": "float32"}


class ImageFormatError(ValueError):
    """Unsupported or corrupt image file (imaging.py:22-23)."""


@dataclass
class ImageData:
    """Decoded image (imaging.py:26-62): float32 samples, (slices, h, w, channels)."""

    samples: np.ndarray
    bit_depth: str = "float32"
    data_range: float | None = 1.0

    def __post_init__(self):
        self.samples = np.asarray(self.samples, dtype=np.float32)
        if self.samples.ndim != 4:
            raise ValueError(f"samples must be (slices, h, w, channels), got shape {self.samples.shape}")
        if min(self.samples.shape) < 1:
            raise ValueError(f"empty image dimension: {self.samples.shape}")
        if self.bit_depth not in _DEPTHS:
            raise ValueError(f"unknown bit depth {self.bit_depth!r}")

    n_slices = property(lambda self: self.samples.shape[0])
    height = property(lambda self: self.samples.shape[1])
    width = property(lambda self: self.samples.shape[2])
    channels = property(lambda self: self.samples.shape[3])

    def plane(self, sl: int = 0, ch: int = 0) -> np.ndarray:
        return self.samples[sl, :, :, ch]


def from_plane(plane, bit_depth: str = "float32", data_range=None) -> ImageData:
    """One 2-D array as a one-slice, one-channel image (imaging.py:82-87)."""
    plane = np.asarray(plane, dtype=np.float32)
    if plane.ndim != 2:
        raise ValueError(f"expected 2-D plane, got {plane.shape}")
    return ImageData(plane[None, :, :, None], bit_depth, data_range)


def quantize(values: np.ndarray, bit_depth: str) -> np.ndarray:
    """Integer samples of a float plane: clamp to [0, range], then round half
    away from zero (imaging.py:127-130; values are non-negative after the clamp,
    so floor(x + 0.5) is that rounding)."""
    limit, dtype = _DEPTHS[bit_depth]
    if limit is None:
        return np.asarray(values, dtype=np.float32)
    return np.floor(np.clip(values, 0.0, limit) + 0.5).astype(dtype)


def load_image(path) -> ImageData:
    """Decode a PNG (8-bit gray / RGB) or TIFF (8/16-bit or float32 gray, any
    number of pages) file (imaging.py:98-124)."""
    from PIL import Image, ImageSequence

    path = Path(path)
    try:
        img = Image.open(path)
    except (OSError, ValueError) as exc:
        raise ImageFormatError(f"cannot read {path}: {exc}") from exc
    kind = path.suffix.lower()
    if kind == ".png":
        if img.mode not in _PNG_CHANNELS:
            raise ImageFormatError(f"{path}: PNG mode {img.mode!r} unsupported (L or RGB)")
        px = np.asarray(img, dtype=np.float32)
        return ImageData(px.reshape(1, px.shape[0], px.shape[1], -1), "uint8", 255.0)
    if kind in (".tif", ".tiff"):
        if img.mode not in _TIFF_DEPTH:
            raise ImageFormatError(f"{path}: TIFF mode {img.mode!r} unsupported (grayscale 8/16-bit or float32)")
        depth = _TIFF_DEPTH[img.mode]
        pages = np.stack([np.asarray(page, dtype=np.float32) for page in ImageSequence.Iterator(img)])
        return ImageData(pages[..., None], depth, _DEPTHS[depth][0])
    raise ImageFormatError(f"{path}: unsupported container (PNG or TIFF only)")


def save_image(img: ImageData, path) -> None:
    """Write an image; the extension picks the container (imaging.py:133-163).
    PNG and integer TIFF quantize (see ``quantize``); float32 TIFF is lossless."""
    from PIL import Image

    path = Path(path)
    kind = path.suffix.lower()
    if kind == ".png":
        if img.n_slices != 1:
            raise ImageFormatError("PNG cannot hold multi-slice stacks; use TIFF")
        if img.channels not in (1, 3):
            raise ImageFormatError(f"PNG supports 1 or 3 channels, got {img.channels}")
        px = quantize(img.samples[0], "uint8")
        Image.fromarray(px[:, :, 0] if img.channels == 1 else px).save(path)
    elif kind in (".tif", ".tiff"):
        if img.channels != 1:
            raise ImageFormatError("TIFF output is grayscale only; split channels first")
        if img.bit_depth == "float32":
            pages = [Image.fromarray(img.samples[i, :, :, 0], mode="F") for i in range(img.n_slices)]
        else:
            pages = [Image.fromarray(quantize(img.samples[i, :, :, 0], img.bit_depth))
                     for i in range(img.n_slices)]
        pages[0].save(path, save_all=len(pages) > 1, append_images=pages[1:])
    else:
        raise ImageFormatError(f"{path}: unsupported container (PNG or TIFF only)")
