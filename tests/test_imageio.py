"""Image containers: the cases of the reference's
test_imaging.py:62-140 on this package's codecs, and byte-identity of the
written files against the installed reference (baseline/_ref) where present."""

import os
import sys

import numpy as np
import pytest

from paper_2108_10209_b200.imageio import (ImageData, ImageFormatError, from_plane, load_image,
                                            quantize, save_image)

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def test_float32_tiff_roundtrip_bitwise(tmp_path):
    rng = np.random.default_rng(0)
    img = from_plane((rng.standard_normal((20, 30)) * 300).astype(np.float32))
    save_image(img, tmp_path / "a.tiff")
    back = load_image(tmp_path / "a.tiff")
    assert back.bit_depth == "float32" and back.data_range is None
    assert np.array_equal(back.samples, img.samples)


def test_multipage_float_tiff_roundtrip(tmp_path):
    stack = np.random.default_rng(1).standard_normal((4, 12, 10, 1)).astype(np.float32)
    save_image(ImageData(stack, "float32", None), tmp_path / "stack.tif")
    back = load_image(tmp_path / "stack.tif")
    assert back.n_slices == 4 and np.array_equal(back.samples, stack)


def test_png_gray_and_rgb(tmp_path):
    from PIL import Image

    g = np.zeros((5, 5), np.uint8)
    g[2, 3] = 200
    Image.fromarray(g).save(tmp_path / "g.png")
    img = load_image(tmp_path / "g.png")
    assert (img.bit_depth, img.data_range, img.channels) == ("uint8", 255.0, 1)
    assert img.plane()[2, 3] == 200.0
    c = np.random.default_rng(2).integers(0, 256, (6, 7, 3)).astype(np.uint8)
    Image.fromarray(c).save(tmp_path / "c.png")
    rgb = load_image(tmp_path / "c.png")
    assert rgb.channels == 3 and (rgb.height, rgb.width) == (6, 7)
    save_image(rgb, tmp_path / "c2.png")
    assert np.array_equal(load_image(tmp_path / "c2.png").samples, rgb.samples)


def test_save_clamps_and_rounds_half_away(tmp_path):
    img = from_plane(np.array([[255.7, -3.0], [99.5, 100.4]], np.float32), "uint8", 255.0)
    save_image(img, tmp_path / "q.png")
    assert load_image(tmp_path / "q.png").plane().tolist() == [[255.0, 0.0], [100.0, 100.0]]
    assert quantize(np.array([0.5, 1.5, 2.5, 65535.4, 7e4]), "uint16").tolist() == [1, 2, 3, 65535, 65535]


def test_16bit_tiff_roundtrip(tmp_path):
    vals = np.random.default_rng(3).integers(0, 65536, (8, 9)).astype(np.float32)
    save_image(from_plane(vals, "uint16", 65535.0), tmp_path / "d.tif")
    back = load_image(tmp_path / "d.tif")
    assert back.bit_depth == "uint16" and back.data_range == 65535.0
    assert np.array_equal(back.plane(), vals)


def test_rejections(tmp_path):
    (tmp_path / "x.bmp").write_bytes(b"BM??")
    (tmp_path / "x.png").write_bytes(b"not a png")
    for name in ("x.bmp", "x.png", "missing.tif"):
        with pytest.raises(ImageFormatError):
            load_image(tmp_path / name)
    with pytest.raises(ImageFormatError):
        save_image(ImageData(np.zeros((2, 4, 4, 1), np.float32), "uint8", 255.0), tmp_path / "s.png")
    with pytest.raises(ImageFormatError):
        save_image(ImageData(np.zeros((1, 4, 4, 2), np.float32), "uint8", 255.0), tmp_path / "s.png")
    with pytest.raises(ImageFormatError):
        save_image(ImageData(np.zeros((1, 4, 4, 3), np.float32), "uint8", 255.0), tmp_path / "s.tif")
    with pytest.raises(ImageFormatError):
        save_image(from_plane(np.zeros((4, 4), np.float32)), tmp_path / "s.jpg")
    with pytest.raises(ValueError):
        ImageData(np.zeros((4, 4), np.float32))
    with pytest.raises(ValueError):
        ImageData(np.zeros((1, 4, 4, 1), np.float32), "int12")
    with pytest.raises(ValueError):
        from_plane(np.zeros((1, 4, 4)))


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "noise2fast")), reason="no baseline/_ref install")
def test_files_byte_identical_to_reference(tmp_path):
    """Same samples -> the same file bytes as the stock reference's save_image,
    and each side decodes the other's files to identical ImageData."""
    sys.path.insert(0, REF)
    try:
        from noise2fast import imaging as ref
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(5)
    cases = [
        ("f.tif", rng.standard_normal((3, 17, 9, 1)) * 40, "float32", None),
        ("u8.tif", rng.uniform(-20, 300, (2, 8, 11, 1)), "uint8", 255.0),
        ("u16.tiff", rng.uniform(-20, 70000, (1, 8, 11, 1)), "uint16", 65535.0),
        ("g.png", rng.uniform(-20, 300, (1, 13, 7, 1)), "uint8", 255.0),
        ("rgb.png", rng.uniform(-20, 300, (1, 13, 7, 3)), "uint8", 255.0),
    ]
    for name, samples, depth, rng_ in cases:
        samples = samples.astype(np.float32)
        mine, theirs = tmp_path / ("mine_" + name), tmp_path / ("ref_" + name)
        save_image(ImageData(samples, depth, rng_), mine)
        ref.save_image(ref.ImageData(samples, depth, rng_), theirs)
        assert mine.read_bytes() == theirs.read_bytes(), name
        a, b = load_image(theirs), ref.load_image(mine)
        assert (a.bit_depth, a.data_range) == (b.bit_depth, b.data_range)
        assert np.array_equal(a.samples, b.samples)
