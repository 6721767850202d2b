"""Weight checkpoints in the reference's ``N2FW`` format (model.py:143-184),
written from / read into the engine's parameter arena.

Layout (little endian): magic ``b"N2FW"``, version 1, in_channels,
n_layers (uint32 each); per layer the OIHW weight shape (4 x uint32); the
network seed (uint64); then per layer the float32 weights (OIHW) and bias.
The engine keeps weights K-major ``[cout][ky][kx][cin]``; the permutation to
OIHW is exact, so a checkpoint written here is byte-identical to the
reference's ``save_checkpoint`` of the same network and loads in
``noise2fast.model.load_checkpoint``.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"N2FW"  # model.py:22
VERSION = 1      # model.py:23
WIDTHS = (32, 32, 64, 64, 128, 128, 256, 256)  # model.py:20 CHANNEL_PLAN


def layer_shapes(in_channels: int = 1):
    """(cout, cin, k, k) OIHW shapes of the 8 3x3 layers and the 1x1 head."""
    shapes, prev = [], in_channels
    for c in WIDTHS:
        shapes.append((c, prev, 3, 3))
        prev = c
    shapes.append((1, prev, 1, 1))
    return shapes


def arena_to_layers(arena: np.ndarray, in_channels: int = 1):
    """Engine arena (w0, b0, ..., w8, b8; K-major weights) -> [(w_oihw, b)]."""
    out, off = [], 0
    for cout, cin, kh, kw in layer_shapes(in_channels):
        n = cout * kh * kw * cin
        w = arena[off: off + n].reshape(cout, kh, kw, cin).transpose(0, 3, 1, 2)
        off += n
        out.append((np.ascontiguousarray(w, np.float32), arena[off: off + cout].astype(np.float32)))
        off += cout
    if off != arena.size:
        raise ValueError(f"arena has {arena.size} values, the network {off}")
    return out


def layers_to_arena(layers) -> np.ndarray:
    parts = []
    for w, b in layers:
        parts += [np.ascontiguousarray(np.asarray(w, np.float32).transpose(0, 2, 3, 1)).ravel(),
                  np.asarray(b, np.float32).ravel()]
    return np.concatenate(parts)


def save_checkpoint(arena: np.ndarray, path, seed: int, in_channels: int = 1) -> None:
    """Write the engine arena as an N2FW v1 checkpoint (model.py:143-152)."""
    layers = arena_to_layers(np.asarray(arena, np.float32), in_channels)
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<III", VERSION, in_channels, len(layers)))
        for w, _ in layers:
            fh.write(struct.pack("<IIII", *w.shape))
        fh.write(struct.pack("<Q", int(seed) & 0xFFFFFFFFFFFFFFFF))
        for w, b in layers:
            fh.write(np.ascontiguousarray(w, dtype="<f4").tobytes())
            fh.write(np.ascontiguousarray(b, dtype="<f4").tobytes())


def load_checkpoint(path):
    """(engine arena, seed, in_channels) from an N2FW v1 file, with the
    reference's errors (model.py:155-162)."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != MAGIC:
            raise ValueError(f"not a weight checkpoint (bad magic {magic!r})")
        version, in_channels, n_layers = struct.unpack("<III", fh.read(12))
        if version != VERSION:
            raise ValueError(f"unsupported checkpoint version {version}")
        shapes = [struct.unpack("<IIII", fh.read(16)) for _ in range(n_layers)]
        (seed,) = struct.unpack("<Q", fh.read(8))
        if [tuple(s) for s in shapes] != layer_shapes(in_channels):
            raise ValueError(f"checkpoint layer shapes {shapes} are not the Noise2Fast network")
        layers = []
        for cout, cin, kh, kw in shapes:
            w = np.frombuffer(fh.read(4 * cout * cin * kh * kw), dtype="<f4").reshape(cout, cin, kh, kw)
            b = np.frombuffer(fh.read(4 * cout), dtype="<f4")
            layers.append((w, b))
    return layers_to_arena(layers), int(seed), int(in_channels)
