"""tcgen05 plumbing checks: descriptor encodings for K-major and MN-major
SWIZZLE_128B operands and the tensor core's fp32->tf32 input conversion."""

import numpy as np
import pytest

from n2f_testutil import dev, empty, host

pytestmark = pytest.mark.gpu


def tf32_trunc(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32)


def tf32_round(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)


# modes: 0 K-major SWIZZLE_128B, 2 MN-major SWIZZLE_128B_BASE32B (mode 1, MN-major
# with 16-byte swizzle atoms, is not a valid tf32 operand layout: measured garbage)
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (2, 0), (0, 2), (2, 2)])
@pytest.mark.parametrize("n", [32, 128, 256])
def test_selftest_gemm(a_mn, b_mn, n):
    from paper_2108_10209_b200 import _lib

    rng = np.random.default_rng(n + 10 * a_mn + 100 * b_mn)
    a = rng.standard_normal((128, 32)).astype(np.float32)
    b = rng.standard_normal((n, 32)).astype(np.float32)
    da, db, dd = dev(a), dev(b), empty(128 * n)
    _lib.call("n2f_tc_selftest", da.data_ptr(), db.data_ptr(), dd.data_ptr(), n, a_mn, b_mn, None)
    d = host(dd).reshape(128, n)
    ref_t = tf32_trunc(a).astype(np.float64) @ tf32_trunc(b).astype(np.float64).T
    ref_r = tf32_round(a).astype(np.float64) @ tf32_round(b).astype(np.float64).T
    et, er = np.abs(d - ref_t).max(), np.abs(d - ref_r).max()
    print(f"a_mn={a_mn} b_mn={b_mn} n={n}: max|D-trunc|={et:.3e} max|D-round|={er:.3e}")
    assert min(et, er) < 1e-4 * np.abs(ref_t).max()


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (0, 2), (2, 2)])
@pytest.mark.parametrize("n", [64, 256])
def test_selftest_gemm_f16(a_mn, b_mn, n):
    """kind::f16 with fp16 operands: K-major SW128 (0), MN-major SW128 (1),
    MN-major SW64 (2, 32-element blocks)."""
    from paper_2108_10209_b200 import _lib

    rng = np.random.default_rng(7 + n + 3 * a_mn + b_mn)
    a = rng.standard_normal((128, 64)).astype(np.float16)
    b = rng.standard_normal((n, 64)).astype(np.float16)
    da, db, dd = dev(a.view(np.int16)), dev(b.view(np.int16)), empty(128 * n)
    _lib.call("n2f_tc_selftest_f16", da.data_ptr(), db.data_ptr(), dd.data_ptr(), n, a_mn, b_mn, None)
    d = host(dd).reshape(128, n)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    err = np.abs(d - ref).max() / np.abs(ref).max()
    print(f"f16 a_mn={a_mn} b_mn={b_mn} n={n}: rel err {err:.2e}")
    assert err < 1e-6


@pytest.mark.parametrize("n", [64, 128, 256])
def test_selftest_gemm_2sm(n):
    """cta_group::2 (cluster of 2 CTAs, M = 256): A split by rows, B by N halves."""
    from paper_2108_10209_b200 import _lib

    rng = np.random.default_rng(11 + n)
    a = rng.standard_normal((256, 64)).astype(np.float16)
    b = rng.standard_normal((n, 64)).astype(np.float16)
    da, db, dd = dev(a.view(np.int16)), dev(b.view(np.int16)), empty(256 * n)
    _lib.call("n2f_tc_selftest_2sm", da.data_ptr(), db.data_ptr(), dd.data_ptr(), n, None)
    d = host(dd).reshape(256, n)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    err = np.abs(d - ref).max() / np.abs(ref).max()
    print(f"2sm n={n}: rel err {err:.2e}")
    assert err < 1e-6


def test_split_operands_recover_fp32():
    """hi = tf32-truncated x, lo = x - hi: hi.hi + hi.lo + lo.hi ~ fp32 GEMM."""
    from paper_2108_10209_b200 import _lib

    rng = np.random.default_rng(1)
    a = rng.standard_normal((128, 32)).astype(np.float32)
    b = rng.standard_normal((64, 32)).astype(np.float32)
    ah, bh = tf32_trunc(a), tf32_trunc(b)
    al, bl = a - ah, b - bh
    out = np.zeros((128, 64))
    for x, y in ((ah, bh), (ah, bl), (al, bh)):
        dx, dy, dd = dev(x), dev(y), empty(128 * 64)
        _lib.call("n2f_tc_selftest", dx.data_ptr(), dy.data_ptr(), dd.data_ptr(), 64, 0, 0, None)
        out += host(dd).reshape(128, 64)
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    err = np.abs(out - exact).max() / np.abs(exact).max()
    one_pass = np.abs(tf32_round(a).astype(np.float64) @ tf32_round(b).astype(np.float64).T - exact).max()
    print(f"3xTF32 rel err {err:.2e}; 1-pass tf32 abs err {one_pass:.2e}")
    assert err < 2e-6
