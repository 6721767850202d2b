// Image-quality metrics on the device (benchmark mode):
// PSNR and the mean SSIM with the 11x11 Gaussian window (sigma 1.5) over
// fully valid positions, both in f64 like the reference (imaging.py:251-311).
// HBM-bound stencils; block partials are reduced in a fixed order
// (deterministic).
#include <math.h>

#include <algorithm>

#include "n2f_internal.cuh"

namespace n2f {
namespace {

constexpr int kThreads = 256;
constexpr int kWin = 11;
constexpr int kTX = 32, kTY = 16;  // valid outputs per block
constexpr int kIX = kTX + kWin - 1, kIY = kTY + kWin - 1;

struct Win {
  double w[kWin];
};

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < kThreads / 32; ++k) s += red[k];
  return s;  // valid in thread 0
}

// Squared-error partials of (a - b) in f64 (imaging.py:249-263).
__global__ void __launch_bounds__(kThreads)
    k_sq_err(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
             double* __restrict__ part) {
  __shared__ double red[kThreads / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// SSIM map summed over one 32 x 16 tile of valid positions.  The window sums
// are separable: vertical 11-tap pass of a, b, a*a, b*b, a*b into smem, then
// the horizontal pass and the SSIM formula per output (imaging.py:266-311).
__global__ void __launch_bounds__(kThreads)
    k_ssim_tile(const double* __restrict__ a, const double* __restrict__ b, int H, int W, Win win,
                double c1, double c2, double* __restrict__ part) {
  __shared__ double sa[kIY][kIX], sb[kIY][kIX];
  __shared__ double v[5][kTY][kIX];
  __shared__ double red[kThreads / 32];
  const int ox0 = blockIdx.x * kTX, oy0 = blockIdx.y * kTY;  // valid-output origin
  for (int i = threadIdx.x; i < kIY * kIX; i += kThreads) {
    const int r = i / kIX, c = i - r * kIX;
    const int y = oy0 + r, x = ox0 + c;
    const bool in = y < H && x < W;
    sa[r][c] = in ? a[(int64_t)y * W + x] : 0.0;
    sb[r][c] = in ? b[(int64_t)y * W + x] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTY * kIX; i += kThreads) {
    const int r = i / kIX, c = i - r * kIX;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double p = sa[r + k][c], q = sb[r + k][c], wk = win.w[k];
      s0 += wk * p;
      s1 += wk * q;
      s2 += wk * (p * p);
      s3 += wk * (q * q);
      s4 += wk * (p * q);
    }
    v[0][r][c] = s0;
    v[1][r][c] = s1;
    v[2][r][c] = s2;
    v[3][r][c] = s3;
    v[4][r][c] = s4;
  }
  __syncthreads();
  const int HV = H - (kWin - 1), WV = W - (kWin - 1);
  double acc = 0.0;
  for (int i = threadIdx.x; i < kTY * kTX; i += kThreads) {
    const int r = i / kTX, c = i - r * kTX;
    if (oy0 + r >= HV || ox0 + c >= WV) continue;
    double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int l = 0; l < kWin; ++l) {
      const double wl = win.w[l];
#pragma unroll
      for (int q = 0; q < 5; ++q) m[q] += wl * v[q][r][c + l];
    }
    const double mu_a = m[0], mu_b = m[1];
    const double var_a = m[2] - mu_a * mu_a, var_b = m[3] - mu_b * mu_b;
    const double cov = m[4] - mu_a * mu_b;
    const double num = (2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2);
    const double den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2);
    acc += num / den;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = acc;
}

__global__ void k_sum_fixed(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[kThreads / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

struct DevBuf {
  double* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

Win gaussian_window() {  // imaging._gaussian_window(11, 1.5)
  Win w;
  const double half = (kWin - 1) / 2.0, sigma = 1.5;
  double sum = 0.0;
  for (int k = 0; k < kWin; ++k) {
    const double c = k - half;
    w.w[k] = exp(-(c * c) / (2.0 * sigma * sigma));
    sum += w.w[k];
  }
  for (int k = 0; k < kWin; ++k) w.w[k] /= sum;
  return w;
}

}  // namespace
}  // namespace n2f

using namespace n2f;

extern "C" {

int n2f_device_count(int* n) {
  if (!n) return fail(N2F_ERR_ARG, "n2f_device_count: null argument");
  *n = 0;
  N2F_CUDA(cudaGetDeviceCount(n));
  return N2F_OK;
}

int n2f_sq_err_sum(const double* a, const double* b, int64_t n, double* out, void* stream) {
  if (!a || !b || !out || n < 1) return fail(N2F_ERR_ARG, "n2f_sq_err_sum: bad argument");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nblk = (int)std::min<int64_t>(2 * 148 * 4, (n + kThreads - 1) / kThreads);
  DevBuf part, sum;
  N2F_CUDA(cudaMalloc(&part.p, nblk * sizeof(double)));
  N2F_CUDA(cudaMalloc(&sum.p, sizeof(double)));
  k_sq_err<<<nblk, kThreads, 0, st>>>(a, b, n, part.p);
  N2F_LAUNCH_CHECK();
  k_sum_fixed<<<1, kThreads, 0, st>>>(part.p, nblk, sum.p);
  N2F_LAUNCH_CHECK();
  N2F_CUDA(cudaMemcpyAsync(out, sum.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  N2F_CUDA(cudaStreamSynchronize(st));
  return N2F_OK;
}

int n2f_psnr(const double* a, const double* b, int64_t n, double data_range, double* out,
             void* stream) {
  if (!(data_range > 0)) return fail(N2F_ERR_ARG, "data_range must be positive");
  double s = 0.0;
  N2F_TRY(n2f_sq_err_sum(a, b, n, &s, stream));
  const double mse = s / (double)n;
  *out = mse == 0.0 ? INFINITY : 10.0 * log10(data_range * data_range / mse);
  return N2F_OK;
}

int n2f_ssim(const double* a, const double* b, int height, int width, double data_range, double k1,
             double k2, double* out, void* stream) {
  if (!a || !b || !out) return fail(N2F_ERR_ARG, "n2f_ssim: bad argument");
  if (height < kWin || width < kWin)
    return fail(N2F_ERR_ARG, "image (%d, %d) smaller than the 11x11 window", height, width);
  if (!(data_range > 0)) return fail(N2F_ERR_ARG, "data_range must be positive");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int HV = height - (kWin - 1), WV = width - (kWin - 1);
  const dim3 grid((WV + kTX - 1) / kTX, (HV + kTY - 1) / kTY);
  const int nblk = (int)(grid.x * grid.y);
  DevBuf part, sum;
  N2F_CUDA(cudaMalloc(&part.p, nblk * sizeof(double)));
  N2F_CUDA(cudaMalloc(&sum.p, sizeof(double)));
  const double c1 = (k1 * data_range) * (k1 * data_range), c2 = (k2 * data_range) * (k2 * data_range);
  k_ssim_tile<<<grid, kThreads, 0, st>>>(a, b, height, width, gaussian_window(), c1, c2, part.p);
  N2F_LAUNCH_CHECK();
  k_sum_fixed<<<1, kThreads, 0, st>>>(part.p, nblk, sum.p);
  N2F_LAUNCH_CHECK();
  double s = 0.0;
  N2F_CUDA(cudaMemcpyAsync(&s, sum.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  N2F_CUDA(cudaStreamSynchronize(st));
  *out = s / ((double)HV * (double)WV);
  return N2F_OK;
}

}  // extern "C"
