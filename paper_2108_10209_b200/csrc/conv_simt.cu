// SIMT fp32 convolution kernels (forward, dgrad, wgrad) on NHWC activations.
//
// These restate the reference's fp32 conv (tensor.py:268-316: im2col + sgemm,
// col2im scatter for the input gradient) as implicit GEMMs with no im2col
// buffer.  They are the exact-fp32 path (fp32 products, fp32 accumulation in
// a different order than OpenBLAS) used for the small-channel layers, for
// the first layer (Cin = 1) and as the cross-check of the tcgen05 kernels.
//
//   forward : y[p][n] = epi( sum_{tap,c} x[p+d(tap)][c] * wk[n][tap][c] )
//   dgrad   : same kernel with wk = dgrad-transposed weights
//             wt[c][tap'][o] = w[o][8-tap'][c] and epi = ReLU mask of the
//             layer input (model.py:101-113 feeds grad_in * (pre>0) back)
//   wgrad   : dw[o][tap][c] = sum_p g[p][o] * x[p+d(tap)][c]  (deterministic
//             split over pixels: partial sums per split, reduced in fixed order)
#include "n2f_internal.cuh"
#include "tc_common.cuh"

namespace n2f {
namespace {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// 3x3 implicit GEMM, M = pixels (BM = 128), N = output channels, K = 9 * C.
// ---------------------------------------------------------------------------
template <int BN, int TM, int TN>
__global__ void __launch_bounds__(kThreads)
    k_conv3x3(const float* __restrict__ x, const float* __restrict__ wk,
              const float* __restrict__ bias, const float* __restrict__ mask,
              float* __restrict__ y, int H, int W, int C, int N, int epi) {
  constexpr int BM = 128, BK = 8, LDA = BM + 4, LDB = BN + 4;
  static_assert((BM / TM) * (BN / TN) == kThreads, "thread tile");
  __shared__ __align__(16) float As[2][BK][LDA];
  __shared__ __align__(16) float Bs[2][BK][LDB];

  const int tid = threadIdx.x;
  const int P = H * W;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;

  const int am = tid >> 1, ah = (tid & 1) * 4;
  const int ap = m0 + am;
  const bool avalid = ap < P;
  const int ay = avalid ? ap / W : 0;
  const int ax = avalid ? ap - ay * W : 0;
  const int bn = tid >> 1, bh = (tid & 1) * 4;
  const bool bload = bn < BN;
  const int cpt = C / BK;
  const int KB = 9 * cpt;

  float4 ra = make_float4(0.f, 0.f, 0.f, 0.f), rb = ra;
  auto load = [&](int kb) {
    const int tap = kb / cpt;
    const int c0 = (kb - tap * cpt) * BK;
    const int ky = tap / 3, kx = tap - 3 * (tap / 3);
    const int yy = ay + ky - 1, xx = ax + kx - 1;
    if (avalid && yy >= 0 && yy < H && xx >= 0 && xx < W)
      ra = __ldg(reinterpret_cast<const float4*>(x + (size_t)(yy * W + xx) * C + c0 + ah));
    else
      ra = make_float4(0.f, 0.f, 0.f, 0.f);
    if (bload)
      rb = __ldg(reinterpret_cast<const float4*>(wk + (size_t)(n0 + bn) * 9 * C + tap * C + c0 + bh));
  };
  auto store = [&](int buf) {
    As[buf][ah + 0][am] = ra.x;
    As[buf][ah + 1][am] = ra.y;
    As[buf][ah + 2][am] = ra.z;
    As[buf][ah + 3][am] = ra.w;
    if (bload) {
      Bs[buf][bh + 0][bn] = rb.x;
      Bs[buf][bh + 1][bn] = rb.y;
      Bs[buf][bh + 2][bn] = rb.z;
      Bs[buf][bh + 3][bn] = rb.w;
    }
  };

  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  load(0);
  store(0);
  __syncthreads();
  for (int kb = 0; kb < KB; ++kb) {
    const int cur = kb & 1;
    if (kb + 1 < KB) load(kb + 1);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        float4 v = *reinterpret_cast<const float4*>(&As[cur][k][ty * TM + i]);
        a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        float4 v = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * TN + j]);
        b[j] = v.x; b[j + 1] = v.y; b[j + 2] = v.z; b[j + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kb + 1 < KB) store(cur ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int p = m0 + ty * TM + i;
    if (p >= P) continue;
#pragma unroll
    for (int j = 0; j < TN; j += 4) {
      const int n = n0 + tx * TN + j;
      float4 v = make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
      if (epi == kEpiBiasRelu || epi == kEpiBias) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + n));
        v.x += bb.x; v.y += bb.y; v.z += bb.z; v.w += bb.w;
        if (epi == kEpiBiasRelu) {
          v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
        }
      } else if (epi == kEpiMask) {
        const float4 mk = __ldg(reinterpret_cast<const float4*>(mask + (size_t)p * N + n));
        v.x = mk.x > 0.f ? v.x : 0.f;
        v.y = mk.y > 0.f ? v.y : 0.f;
        v.z = mk.z > 0.f ? v.z : 0.f;
        v.w = mk.w > 0.f ? v.w : 0.f;
      }
      *reinterpret_cast<float4*>(y + (size_t)p * N + n) = v;
    }
  }
}

// ---------------------------------------------------------------------------
// First layer (Cin = 1): direct 3x3, one thread per (pixel, 8 output
// channels), one image row per grid row (no 64-bit index division).  The
// 9-tap sum order (fmaf over taps, then + bias) is the reference's im2col
// dot order (tensor.py:268-282).
// ---------------------------------------------------------------------------
template <int CPT>  // output channels per thread: 8 (the network, N % 8 == 0) or 1 (any N, fp32 out)
__global__ void __launch_bounds__(kThreads)
    k_conv_first(const float* __restrict__ x, const float* __restrict__ w,
                 const float* __restrict__ b, float* __restrict__ y, float* __restrict__ ylo, int H,
                 int W, int N, int relu, __half* __restrict__ yh16, __half* __restrict__ yl16,
                 float oscale) {
  // weights staged tap-major (ws[t][n]) so a thread's 8 channels of one tap
  // are two 16-byte smem loads
  __shared__ __align__(16) float ws[kMaxC * 9];
  __shared__ __align__(16) float bs[kMaxC];
  for (int i = threadIdx.x; i < N * 9; i += blockDim.x) ws[(i % 9) * N + i / 9] = w[i];
  for (int i = threadIdx.x; i < N; i += blockDim.x) bs[i] = b[i];
  __syncthreads();
  if constexpr (CPT == 1) {  // parity entry point for arbitrary N (fp32 output only)
    const int ppb = blockDim.x / N;
    const int n = threadIdx.x % N;
    const int px = blockIdx.x * ppb + threadIdx.x / N, py = blockIdx.y;
    if (px >= W || threadIdx.x >= ppb * N) return;
    float a = 0.f;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int yy = py + t / 3 - 1, xx = px + t % 3 - 1;
      const float xv = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(x + (int64_t)yy * W + xx) : 0.f;
      a = fmaf(xv, ws[t * N + n], a);
    }
    y[((int64_t)py * W + px) * N + n] = relu ? fmaxf(a + bs[n], 0.f) : a + bs[n];
    return;
  }
  const int nq = N >> 3, ppb = blockDim.x / nq;
  const int q = threadIdx.x % nq;
  const int px = blockIdx.x * ppb + threadIdx.x / nq, py = blockIdx.y;
  if (px >= W) return;
  float xv[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int yy = py + t / 3 - 1, xx = px + t % 3 - 1;
    xv[t] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(x + (int64_t)yy * W + xx) : 0.f;
  }
  float o[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = 0.f;
#pragma unroll
  for (int t = 0; t < 9; ++t) {  // per channel the same fmaf order over taps as before
    const float4 w0 = *reinterpret_cast<const float4*>(ws + t * N + 8 * q);
    const float4 w1 = *reinterpret_cast<const float4*>(ws + t * N + 8 * q + 4);
    const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = fmaf(xv[t], wv[j], o[j]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = relu ? fmaxf(o[j] + bs[8 * q + j], 0.f) : o[j] + bs[8 * q + j];
  const int64_t idx = ((int64_t)py * W + px) * N + 8 * q;
  if (y) {
    *reinterpret_cast<float4*>(y + idx) = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(y + idx + 4) = make_float4(o[4], o[5], o[6], o[7]);
  }
  if (yh16) {  // fp16 pair of y * oscale for the FP16 tcgen05 consumers
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      __half h0, l0, h1, l1;
      tc::split_f16(o[j] * oscale, h0, l0);
      tc::split_f16(o[j + 1] * oscale, h1, l1);
      hw[j / 2] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
      lw[j / 2] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
    }
    *reinterpret_cast<uint4*>(yh16 + idx) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(yl16 + idx) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  if (ylo) {  // tf32 residuals for a tcgen05 consumer
    float l[8], hh;
#pragma unroll
    for (int j = 0; j < 8; ++j) tc::split_tf32(o[j], hh, l[j]);
    *reinterpret_cast<float4*>(ylo + idx) = make_float4(l[0], l[1], l[2], l[3]);
    *reinterpret_cast<float4*>(ylo + idx + 4) = make_float4(l[4], l[5], l[6], l[7]);
  }
}

// ---------------------------------------------------------------------------
// wgrad: dw_part[s][o][k] = sum_{p in split s} g[p][o] * xg[p][k],  k = tap*C + c
// BM over o, BN over k, BP pixels per pipeline stage.
// ---------------------------------------------------------------------------
template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(kThreads)
    k_wgrad3x3(const float* __restrict__ g, const float* __restrict__ x, float* __restrict__ dw_part,
               float* __restrict__ db_part, int H, int W, int C, int NO, int chunk) {
  constexpr int BP = 8, LDG = BM + 4, LDX = BN + 4;
  constexpr int NG4 = BP * BM / 4, NX4 = BP * BN / 4;
  constexpr int PER = (NG4 + NX4 + kThreads - 1) / kThreads;
  static_assert((BM / TM) * (BN / TN) == kThreads, "thread tile");
  __shared__ __align__(16) float Gs[2][BP][LDG];
  __shared__ __align__(16) float Xs[2][BP][LDX];

  const int tid = threadIdx.x;
  const int P = H * W, K = 9 * C;
  const int o0 = blockIdx.x * BM, k0 = blockIdx.y * BN, s = blockIdx.z;
  const int pbeg = s * chunk;
  const int pend = min(P, pbeg + chunk);
  const int nstage = (max(pend - pbeg, 0) + BP - 1) / BP;

  float4 r[PER];
  auto load = [&](int st) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int f = tid + u * kThreads;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < NG4) {
        const int pp = f / (BM / 4), o4 = f - pp * (BM / 4);
        const int p = pbeg + st * BP + pp;
        if (p < pend) v = __ldg(reinterpret_cast<const float4*>(g + (size_t)p * NO + o0 + 4 * o4));
      } else if (f < NG4 + NX4) {
        const int e = f - NG4;
        const int pp = e / (BN / 4), k4 = e - pp * (BN / 4);
        const int p = pbeg + st * BP + pp;
        const int k = k0 + 4 * k4;
        if (p < pend && k < K) {
          const int tap = k / C, c = k - tap * C;
          const int py = p / W, px = p - py * W;
          const int yy = py + tap / 3 - 1, xx = px + tap % 3 - 1;
          if (yy >= 0 && yy < H && xx >= 0 && xx < W)
            v = __ldg(reinterpret_cast<const float4*>(x + (size_t)(yy * W + xx) * C + c));
        }
      }
      r[u] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int f = tid + u * kThreads;
      if (f < NG4) {
        const int pp = f / (BM / 4), o4 = f - pp * (BM / 4);
        *reinterpret_cast<float4*>(&Gs[buf][pp][4 * o4]) = r[u];
      } else if (f < NG4 + NX4) {
        const int e = f - NG4;
        const int pp = e / (BN / 4), k4 = e - pp * (BN / 4);
        *reinterpret_cast<float4*>(&Xs[buf][pp][4 * k4]) = r[u];
      }
    }
  };

  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  float acc[TM][TN];
  float bacc[TM];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    bacc[i] = 0.f;
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  }
  const bool do_bias = (blockIdx.y == 0) && (tx == 0) && (db_part != nullptr);

  if (nstage > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int st = 0; st < nstage; ++st) {
    const int cur = st & 1;
    if (st + 1 < nstage) load(st + 1);
#pragma unroll
    for (int pp = 0; pp < BP; ++pp) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        float4 v = *reinterpret_cast<const float4*>(&Gs[cur][pp][ty * TM + i]);
        a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        float4 v = *reinterpret_cast<const float4*>(&Xs[cur][pp][tx * TN + j]);
        b[j] = v.x; b[j + 1] = v.y; b[j + 2] = v.z; b[j + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        if (do_bias) bacc[i] += a[i];
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
    }
    if (st + 1 < nstage) store(cur ^ 1);
    __syncthreads();
  }

  float* dst = dw_part + (size_t)s * NO * K;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int o = o0 + ty * TM + i;
#pragma unroll
    for (int j = 0; j < TN; j += 4) {
      const int k = k0 + tx * TN + j;
      if (k < K)
        *reinterpret_cast<float4*>(dst + (size_t)o * K + k) =
            make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
    }
    if (do_bias) db_part[(size_t)s * NO + o] = bacc[i];
  }
}

// First-layer wgrad (Cin = 1): dw[o][tap], db[o]; 8 pixel lanes x 32 channels.
// First-layer wgrad (Cin = 1, NO = 32 output channels): warp = 32 channels,
// each warp walks 32-pixel row segments with a sliding 3x3 window of the
// input in registers (3 broadcast loads + one coalesced 128-byte gradient
// load per pixel).  Block partials [nsplit][NO * 9] / [nsplit][NO], warps
// combined in fixed order (deterministic).
constexpr int kFirstSeg = 32;
__global__ void __launch_bounds__(kThreads)
    k_wgrad_first(const float* __restrict__ g, const float* __restrict__ x,
                  float* __restrict__ dw_part, float* __restrict__ db_part, int H, int W, int upw) {
  constexpr int NO = 32;
  __shared__ float red[kThreads / 32][NO * 10];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int segs_x = (W + kFirstSeg - 1) / kFirstSeg;
  const int nunits = H * segs_x;
  const int gw = blockIdx.x * (kThreads / 32) + warp;
  float acc[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t] = 0.f;
  auto X = [&](int yy, int xx) {
    return (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(x + (int64_t)yy * W + xx) : 0.f;
  };
  const int u1 = min(nunits, (gw + 1) * upw);
  for (int u = gw * upw; u < u1; ++u) {
    const int py = u / segs_x, x0 = (u - py * segs_x) * kFirstSeg;
    const int x1 = min(W, x0 + kFirstSeg);
    float a0 = X(py - 1, x0 - 1), a1 = X(py - 1, x0);
    float b0 = X(py, x0 - 1), b1 = X(py, x0);
    float c0 = X(py + 1, x0 - 1), c1 = X(py + 1, x0);
    const float* gr = g + ((int64_t)py * W) * NO + lane;
#pragma unroll 4
    for (int px = x0; px < x1; ++px) {
      const float a2 = X(py - 1, px + 1), b2 = X(py, px + 1), c2 = X(py + 1, px + 1);
      const float gv = __ldg(gr + (int64_t)px * NO);
      acc[0] = fmaf(gv, a0, acc[0]);
      acc[1] = fmaf(gv, a1, acc[1]);
      acc[2] = fmaf(gv, a2, acc[2]);
      acc[3] = fmaf(gv, b0, acc[3]);
      acc[4] = fmaf(gv, b1, acc[4]);
      acc[5] = fmaf(gv, b2, acc[5]);
      acc[6] = fmaf(gv, c0, acc[6]);
      acc[7] = fmaf(gv, c1, acc[7]);
      acc[8] = fmaf(gv, c2, acc[8]);
      acc[9] += gv;
      a0 = a1; a1 = a2;
      b0 = b1; b1 = b2;
      c0 = c1; c1 = c2;
    }
  }
#pragma unroll
  for (int t = 0; t < 10; ++t) red[warp][t * NO + lane] = acc[t];
  __syncthreads();
  for (int i = threadIdx.x; i < NO * 10; i += kThreads) {
    float s = red[0][i];
#pragma unroll
    for (int k = 1; k < kThreads / 32; ++k) s += red[k][i];
    const int t = i / NO, o = i - t * NO;
    if (t < 9)
      dw_part[(int64_t)blockIdx.x * NO * 9 + o * 9 + t] = s;
    else
      db_part[(int64_t)blockIdx.x * NO + o] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
int conv3x3_simt(const float* x, const float* wk, const float* bias, const float* mask, float* y,
                 int h, int w, int cin, int cout, int epi, cudaStream_t st) {
  if (cin % 8 || cout % 32) return fail(N2F_ERR_ARG, "conv3x3_simt: cin %d cout %d", cin, cout);
  const int P = h * w;
  dim3 block(kThreads);
  if (cout % 128 == 0) {
    dim3 grid((P + 127) / 128, cout / 128);
    k_conv3x3<128, 8, 8><<<grid, block, 0, st>>>(x, wk, bias, mask, y, h, w, cin, cout, epi);
  } else if (cout % 64 == 0) {
    dim3 grid((P + 127) / 128, cout / 64);
    k_conv3x3<64, 8, 4><<<grid, block, 0, st>>>(x, wk, bias, mask, y, h, w, cin, cout, epi);
  } else {
    dim3 grid((P + 127) / 128, cout / 32);
    k_conv3x3<32, 4, 4><<<grid, block, 0, st>>>(x, wk, bias, mask, y, h, w, cin, cout, epi);
  }
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int conv_first_simt(const float* x, const float* w, const float* b, float* y, int h, int w_,
                    int cout, cudaStream_t st, int relu, float* ylo, void* yh16, void* yl16,
                    float oscale) {
  if (cout < 1 || cout > kMaxC) return fail(N2F_ERR_ARG, "conv_first: cout %d", cout);
  if (ylo && !y) return fail(N2F_ERR_ARG, "conv_first: tf32 residual needs y");
  if (h > 65535) return fail(N2F_ERR_ARG, "conv_first: height %d", h);
  if (cout % 8 == 0 && kThreads % (cout / 8) == 0) {
    const int ppb = kThreads / (cout / 8);
    k_conv_first<8><<<dim3((unsigned)((w_ + ppb - 1) / ppb), (unsigned)h), kThreads, 0, st>>>(
        x, w, b, y, ylo, h, w_, cout, relu, reinterpret_cast<__half*>(yh16),
        reinterpret_cast<__half*>(yl16), oscale);
  } else {
    if (!y || ylo || yh16) return fail(N2F_ERR_ARG, "conv_first: cout %d supports fp32 output only", cout);
    const int ppb = kThreads / cout;
    k_conv_first<1><<<dim3((unsigned)((w_ + ppb - 1) / ppb), (unsigned)h), kThreads, 0, st>>>(
        x, w, b, y, nullptr, h, w_, cout, relu, nullptr, nullptr, 1.f);
  }
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

// wgrad CTA tile (over cout x 9*cin) for a layer
static void wgrad_tile(int cout, int* bm, int* bn) {
  if (cout % 128 == 0) { *bm = 128; *bn = 128; }
  else if (cout % 64 == 0) { *bm = 64; *bn = 64; }
  else { *bm = 32; *bn = 128; }
}

int wgrad_nsplit(int64_t pixels, int cin, int cout) {
  // aim for ~4 waves of 256-thread CTAs over 148 SMs, >= 512 pixels per split
  int bm, bn;
  wgrad_tile(cout, &bm, &bn);
  const int64_t tiles =
      (cin == 1) ? 1 : (int64_t)((cout + bm - 1) / bm) * ((9 * cin + bn - 1) / bn);
  int64_t want = (4 * 148 + tiles - 1) / tiles;
  // the first layer's wgrad (k_wgrad_first): one block per ~256 pixels (8
  // warps x one 32-pixel segment: latency-bound, so many warps), at most 2048
  int64_t maxs = cin == 1 ? (pixels + 255) / 256 : (pixels + 511) / 512;
  if (cin == 1) want = 2048;
  int64_t n = want < maxs ? want : maxs;
  if (n < 1) n = 1;
  if (n > 1024) n = 1024;
  return (int)n;
}

int wgrad3x3_simt(const float* g, const float* x, float* dw_part, float* db_part, int h, int w,
                  int cin, int cout, int nsplit, cudaStream_t st) {
  const int P = h * w;
  int chunk = (P + nsplit - 1) / nsplit;
  chunk = (chunk + 7) / 8 * 8;
  const int K = 9 * cin;
  if (cin % 4 || cout % 32) return fail(N2F_ERR_ARG, "wgrad3x3_simt: cin %d cout %d", cin, cout);
  int bm, bn;
  wgrad_tile(cout, &bm, &bn);
  dim3 grid(cout / bm, (K + bn - 1) / bn, nsplit);
  if (bm == 128)
    k_wgrad3x3<128, 128, 8, 8><<<grid, kThreads, 0, st>>>(g, x, dw_part, db_part, h, w, cin, cout,
                                                          chunk);
  else if (bm == 64)
    k_wgrad3x3<64, 64, 4, 4><<<grid, kThreads, 0, st>>>(g, x, dw_part, db_part, h, w, cin, cout,
                                                        chunk);
  else
    k_wgrad3x3<32, 128, 4, 4><<<grid, kThreads, 0, st>>>(g, x, dw_part, db_part, h, w, cin, cout,
                                                         chunk);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int wgrad_first_simt(const float* g, const float* x, float* dw_part, float* db_part, int h, int w,
                     int cout, int nsplit, cudaStream_t st) {
  if (cout != 32) return fail(N2F_ERR_ARG, "wgrad_first: cout %d", cout);
  const int64_t nunits = (int64_t)h * ((w + kFirstSeg - 1) / kFirstSeg);
  const int64_t warps = (int64_t)nsplit * (kThreads / 32);
  const int upw = (int)((nunits + warps - 1) / warps);
  k_wgrad_first<<<nsplit, kThreads, 0, st>>>(g, x, dw_part, db_part, h, w, upw);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

}  // namespace n2f
