// First-layer (Cin = 1) kernels on NHWC activations: the L1 forward and the
// L1 weight gradient.  With one input channel the layer is K = 9: no GEMM
// shape for the tensor cores, and HBM/latency bound (132 B/px written by the
// forward), so both are direct CUDA-core kernels restating the reference's
// fp32 conv (tensor.py:268-316) in the im2col dot order.
//
//   forward : y[p][n] = relu( sum_tap x[p+d(tap)] * w[n][tap] + b[n] ), written
//             as the fp16 operand pair of y * 2^kExpAct for the L2 tcgen05
//             kernels (or fp32 for the parity entry point)
//   wgrad   : dw[o][tap] = sum_p g[p][o] * x[p+d(tap)], db[o] = sum_p g[p][o]
//             (deterministic split over pixels: partial sums per split,
//             reduced in fixed order by k_adam)
#include "n2f_internal.cuh"
#include "tc_common.cuh"

namespace n2f {
namespace {

constexpr int kThreads = 256;
constexpr int kFirstRows = 4;  // image rows per block of the first-layer forward

// ---------------------------------------------------------------------------
// First layer (Cin = 1): direct 3x3, one thread per (pixel, 8 output
// channels), one image row per grid row (no 64-bit index division).  The
// 9-tap sum order (fmaf over taps, then + bias) is the reference's im2col
// dot order (tensor.py:268-282).
// ---------------------------------------------------------------------------
template <int CPT>  // output channels per thread: 8 (the network, N % 8 == 0) or 1 (any N, fp32 out)
__global__ void __launch_bounds__(kThreads)
    k_conv_first(const float* __restrict__ x, const float* __restrict__ w,
                 const float* __restrict__ b, float* __restrict__ y, int H, int W, int N, int relu,
                 __half* __restrict__ yh16, __half* __restrict__ yl16, float oscale,
                 unsigned* __restrict__ amax) {
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
  // a block covers ppb pixels of kFirstRows consecutive rows (one weight
  // staging per kFirstRows rows)
  const int nq = N >> 3, ppb = blockDim.x / nq;
  const int q = threadIdx.x % nq;
  const int px = blockIdx.x * ppb + threadIdx.x / nq;
  const int py0 = blockIdx.y * kFirstRows, py1 = min(H, py0 + kFirstRows);
  unsigned mx = 0;
  if (px < W) {
    for (int py = py0; py < py1; ++py) {
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
      for (int t = 0; t < 9; ++t) {  // per channel the fmaf order over taps of the im2col dot
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
          const float a0 = o[j] * oscale, a1 = o[j + 1] * oscale;
          mx = max(mx, max(tc::range_bits(a0), tc::range_bits(a1)));
          tc::split_f16x2(a0, a1, hw[j / 2], lw[j / 2]);
        }
        *reinterpret_cast<uint4*>(yh16 + idx) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(yl16 + idx) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    }
  }
  if (yh16 && amax) tc::range_note(amax, mx);
}

// First-layer wgrad (Cin = 1, NO = 32 output channels): lane = output
// channel, a warp walks 32-pixel row segments.  Per segment it issues all 32
// coalesced 128-byte gradient rows at once (memory-level parallelism: the
// kernel streams 128 B/px of fp32 gradient and is HBM-bound), each lane loads
// one column of the three input rows of the 3x3 window (34 columns with the
// halo), and the window values reach the other lanes by shuffles.  Pixels of a
// segment are summed in x order, segments in unit order, warps in fixed
// order; block partials [nsplit][NO * 9] / [nsplit][NO] (deterministic).
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
    const int n = min(W - x0, kFirstSeg);
    const float* gr = g + ((int64_t)py * W + x0) * NO + lane;
    float gv[kFirstSeg];
#pragma unroll
    for (int i = 0; i < kFirstSeg; ++i) gv[i] = i < n ? __ldg(gr + i * NO) : 0.f;
    // window columns x0 - 1 + lane (and x0 + 31 + lane for lanes 0, 1)
    float r0[3], r1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      r0[d] = X(py + d - 1, x0 - 1 + lane);
      r1[d] = lane < 2 ? X(py + d - 1, x0 + 31 + lane) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kFirstSeg; ++i) {
      // x-window columns i, i + 1, i + 2 of the segment (pixel x0 + i)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          const int c = i + e;  // 0..33
          const float w = c < 32 ? __shfl_sync(0xffffffffu, r0[d], c)
                                 : __shfl_sync(0xffffffffu, r1[d], c - 32);
          acc[3 * d + e] = fmaf(gv[i], w, acc[3 * d + e]);
        }
      }
      acc[9] += gv[i];
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
int conv_first_simt(const float* x, const float* w, const float* b, float* y, int h, int w_,
                    int cout, cudaStream_t st, int relu, void* yh16, void* yl16, float oscale,
                    unsigned* amax) {
  if (cout < 1 || cout > kMaxC) return fail(N2F_ERR_ARG, "conv_first: cout %d", cout);
  if (h > 65535) return fail(N2F_ERR_ARG, "conv_first: height %d", h);
  if (cout % 8 == 0 && kThreads % (cout / 8) == 0) {
    const int ppb = kThreads / (cout / 8);
    k_conv_first<8><<<dim3((unsigned)((w_ + ppb - 1) / ppb), (unsigned)((h + kFirstRows - 1) / kFirstRows)),
                      kThreads, 0, st>>>(
        x, w, b, y, h, w_, cout, relu, reinterpret_cast<__half*>(yh16),
        reinterpret_cast<__half*>(yl16), oscale, amax);
  } else {
    if (!y || yh16) return fail(N2F_ERR_ARG, "conv_first: cout %d supports fp32 output only", cout);
    const int ppb = kThreads / cout;
    k_conv_first<1><<<dim3((unsigned)((w_ + ppb - 1) / ppb), (unsigned)h), kThreads, 0, st>>>(
        x, w, b, y, h, w_, cout, relu, nullptr, nullptr, 1.f, nullptr);
  }
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

// Pixel splits of the first-layer wgrad: one block per ~512 pixels (8 warps x
// two 32-pixel segments, each segment's 32 gradient rows in flight), <= 1024.
int wgrad_first_nsplit(int64_t pixels) {
  int64_t n = (pixels + 511) / 512;
  if (n < 1) n = 1;
  if (n > 1024) n = 1024;
  return (int)n;
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
