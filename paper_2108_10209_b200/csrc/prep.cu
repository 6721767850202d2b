// Input preparation kernels: min/max scan, normalisation, training-pair gather,
// He-uniform init from the counter RNG, dgrad weight transpose, partial reduce.
#include <stdarg.h>
#include <time.h>

#include "n2f_internal.cuh"

namespace n2f {

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_err;
thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
const std::string& error_text() { return g_err; }

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

double wall_seconds() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

namespace {

constexpr int kThreads = 256;
constexpr int kScanBlocks = 1184;  // 8 blocks per SM: the scan is HBM-bound

template <typename T>
__device__ __forceinline__ double load_as_double(const void* p, int64_t i) {
  return (double)reinterpret_cast<const T*>(p)[i];
}

__device__ __forceinline__ double load_img(const void* p, int dtype, int64_t i) {
  return dtype == N2F_F64 ? load_as_double<double>(p, i) : load_as_double<float>(p, i);
}

// min / max / non-finite count, stage 1 (per-block partials)
__device__ __forceinline__ void minmax_acc(double v, double& lo, double& hi, double& bad) {
  if (isfinite(v)) {
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  } else {
    bad += 1.0;
  }
}

// (min and max are exact in any order; the non-finite count is an exact
// integer: the result does not depend on the partition)
__global__ void __launch_bounds__(kThreads)
    k_minmax_part(const void* __restrict__ img, int dtype, int64_t n, double* __restrict__ part) {
  __shared__ double smin[kThreads], smax[kThreads], scnt[kThreads];
  double lo = INFINITY, hi = -INFINITY, bad = 0.0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  int64_t head = 0;  // elements before the 16-byte vector body
  if (dtype == N2F_F32 && (reinterpret_cast<uintptr_t>(img) & 15) == 0) {
    const float4* v4 = reinterpret_cast<const float4*>(img);
    const int64_t n4 = n / 4;
    for (int64_t i = tid; i < n4; i += nth) {
      const float4 v = __ldg(v4 + i);
      minmax_acc(v.x, lo, hi, bad);
      minmax_acc(v.y, lo, hi, bad);
      minmax_acc(v.z, lo, hi, bad);
      minmax_acc(v.w, lo, hi, bad);
    }
    head = n4 * 4;
  } else if (dtype == N2F_F64 && (reinterpret_cast<uintptr_t>(img) & 15) == 0) {
    const double2* v2 = reinterpret_cast<const double2*>(img);
    const int64_t n2 = n / 2;
    for (int64_t i = tid; i < n2; i += nth) {
      const double2 v = __ldg(v2 + i);
      minmax_acc(v.x, lo, hi, bad);
      minmax_acc(v.y, lo, hi, bad);
    }
    head = n2 * 2;
  }
  for (int64_t i = head + tid; i < n; i += nth) minmax_acc(load_img(img, dtype, i), lo, hi, bad);
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  scnt[threadIdx.x] = bad;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
      scnt[threadIdx.x] += scnt[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = smin[0];
    part[3 * blockIdx.x + 1] = smax[0];
    part[3 * blockIdx.x + 2] = scnt[0];
  }
}

__global__ void __launch_bounds__(kThreads)
    k_minmax_final(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  __shared__ double smin[kThreads], smax[kThreads], scnt[kThreads];
  double lo = INFINITY, hi = -INFINITY, bad = 0.0;
  for (int i = threadIdx.x; i < nparts; i += kThreads) {
    lo = fmin(lo, part[3 * i]);
    hi = fmax(hi, part[3 * i + 1]);
    bad += part[3 * i + 2];
  }
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  scnt[threadIdx.x] = bad;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
      scnt[threadIdx.x] += scnt[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = smin[0];
    out[1] = smax[0];
    out[2] = scnt[0];
  }
}

// (x - vmin) / (vmax - vmin) in f64, rounded once to f32 (imaging.py:204, trainer.py:163)
__device__ __forceinline__ float norm_value(double v, double vmin, double range) {
  return __double2float_rn(__ddiv_rn(__dsub_rn(v, vmin), range));
}

__global__ void __launch_bounds__(kThreads)
    k_normalize(const void* __restrict__ img, int dtype, int64_t n, const double* __restrict__ mm,
                float* __restrict__ norm) {
  const double vmin = mm[0], range = __dsub_rn(mm[1], mm[0]);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  int64_t head = 0;
  if (dtype == N2F_F32 && (reinterpret_cast<uintptr_t>(img) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(norm) & 15) == 0) {  // 16-byte loads and stores
    const float4* v4 = reinterpret_cast<const float4*>(img);
    float4* o4 = reinterpret_cast<float4*>(norm);
    const int64_t n4 = n / 4;
    for (int64_t i = tid; i < n4; i += nth) {
      const float4 v = __ldg(v4 + i);
      o4[i] = make_float4(norm_value(v.x, vmin, range), norm_value(v.y, vmin, range),
                          norm_value(v.z, vmin, range), norm_value(v.w, vmin, range));
    }
    head = n4 * 4;
  }
  for (int64_t i = head + tid; i < n; i += nth) norm[i] = norm_value(load_img(img, dtype, i), vmin, range);
}

__device__ __forceinline__ float clip01(float v, int clip) {
  return clip ? fminf(fmaxf(v, 0.f), 1.f) : v;
}

// One thread per 2x2 quad of the even-cropped image (downsample.py:45-66, 94-100, 141-164).
__global__ void __launch_bounds__(kThreads)
    k_pairs(const float* __restrict__ norm, const void* __restrict__ clean, int dtype,
            const double* __restrict__ mm, int H, int W, int scheme, int clip,
            float* __restrict__ pin, float* __restrict__ ptgt, int64_t plane) {
  const int hq = H / 2, wq = W / 2;  // quads of the even crop
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (int64_t)hq * wq) return;
  const int i = (int)(q / wq), j = (int)(q - (int64_t)i * wq);
  const int64_t r0 = (int64_t)(2 * i) * W + 2 * j, r1 = r0 + W;
  const float a = norm[r0], b = norm[r0 + 1], c = norm[r1], d = norm[r1 + 1];
  if (scheme == 1) {  // quad: TL=a TR=b BL=c; pairs (tl>tr) (tr>tl) (tl>bl) (bl>tl)
    const int64_t o = (int64_t)i * wq + j;
    pin[0 * plane + o] = a; ptgt[0 * plane + o] = clip01(b, clip);
    pin[1 * plane + o] = b; ptgt[1 * plane + o] = clip01(a, clip);
    pin[2 * plane + o] = a; ptgt[2 * plane + o] = clip01(c, clip);
    pin[3 * plane + o] = c; ptgt[3 * plane + o] = clip01(a, clip);
    return;
  }
  // up planes (H, W/2): rows 2i, 2i+1, col j.  left planes (H/2, W): row i, cols 2j, 2j+1
  const int64_t u0 = (int64_t)(2 * i) * wq + j, u1 = u0 + wq;
  const int64_t l0 = (int64_t)i * (2 * wq) + 2 * j, l1 = l0 + 1;  // row stride = even width
  // eu: a,d  ou: b,c  el: a,d  ol: c,b
  float eu0 = a, eu1 = d, ou0 = b, ou1 = c, el0 = a, el1 = d, ol0 = c, ol1 = b;
  pin[0 * plane + u0] = eu0; pin[0 * plane + u1] = eu1;
  pin[1 * plane + u0] = ou0; pin[1 * plane + u1] = ou1;
  pin[2 * plane + l0] = el0; pin[2 * plane + l1] = el1;
  pin[3 * plane + l0] = ol0; pin[3 * plane + l1] = ol1;
  float t_eu0 = eu0, t_eu1 = eu1, t_ou0 = ou0, t_ou1 = ou1;
  float t_el0 = el0, t_el1 = el1, t_ol0 = ol0, t_ol1 = ol1;
  if (scheme == 2) {  // exact: target = x_tgt - (s_tgt - s_in), fp32 (downsample.py:141-164)
    const double vmin = mm[0], range = __dsub_rn(mm[1], mm[0]);
    const float sa = norm_value(load_img(clean, dtype, r0), vmin, range);
    const float sb = norm_value(load_img(clean, dtype, r0 + 1), vmin, range);
    const float sc = norm_value(load_img(clean, dtype, r1), vmin, range);
    const float sd = norm_value(load_img(clean, dtype, r1 + 1), vmin, range);
    // s_eu: sa,sd  s_ou: sb,sc  s_el: sa,sd  s_ol: sc,sb
    t_ou0 = __fsub_rn(ou0, __fsub_rn(sb, sa)); t_ou1 = __fsub_rn(ou1, __fsub_rn(sc, sd));
    t_eu0 = __fsub_rn(eu0, __fsub_rn(sa, sb)); t_eu1 = __fsub_rn(eu1, __fsub_rn(sd, sc));
    t_ol0 = __fsub_rn(ol0, __fsub_rn(sc, sa)); t_ol1 = __fsub_rn(ol1, __fsub_rn(sb, sd));
    t_el0 = __fsub_rn(el0, __fsub_rn(sa, sc)); t_el1 = __fsub_rn(el1, __fsub_rn(sd, sb));
  }
  ptgt[0 * plane + u0] = clip01(t_ou0, clip); ptgt[0 * plane + u1] = clip01(t_ou1, clip);
  ptgt[1 * plane + u0] = clip01(t_eu0, clip); ptgt[1 * plane + u1] = clip01(t_eu1, clip);
  ptgt[2 * plane + l0] = clip01(t_ol0, clip); ptgt[2 * plane + l1] = clip01(t_ol1, clip);
  ptgt[3 * plane + l0] = clip01(t_el0, clip); ptgt[3 * plane + l1] = clip01(t_el1, clip);
}

// SplitMix64 output function (rng.py:20-28)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// He-uniform weights in [cout][ky][kx][cin] from the OIHW-ordered counter stream.
__global__ void __launch_bounds__(kThreads)
    k_init_layer(uint64_t key, double bound, int cin, int cout, int kk, float* __restrict__ w) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)cout * kk * cin;
  if (e >= total) return;
  const int c = (int)(e % cin);
  const int tap = (int)((e / cin) % kk);
  const int o = (int)(e / ((int64_t)cin * kk));
  const uint64_t idx = (uint64_t)o * cin * kk + (uint64_t)c * kk + tap;  // OIHW flat index
  const uint64_t bits = mix64(idx ^ key);
  const double u = (double)(bits >> 11) * 0x1.0p-53;
  // low + u * (high - low) with low = -bound, high = bound (rng.py:64)
  const double v = __dadd_rn(-bound, __dmul_rn(u, __dadd_rn(bound, bound)));
  w[e] = __double2float_rn(v);
}

__global__ void __launch_bounds__(kThreads)
    k_transpose_dgrad(const float* __restrict__ w, float* __restrict__ wt, int cin, int cout) {
  // wt[c][t'][o] = w[o][8-t'][c]
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)cout * 9 * cin;
  if (e >= total) return;
  const int o = (int)(e % cout);
  const int tp = (int)((e / cout) % 9);
  const int c = (int)(e / ((int64_t)cout * 9));
  wt[e] = w[((int64_t)o * 9 + (8 - tp)) * cin + c];
}

__global__ void __launch_bounds__(kThreads)
    k_reduce_partials(const float* __restrict__ part, float* __restrict__ out, int nsplit,
                      int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = part[i];
  for (int k = 1; k < nsplit; ++k) s += part[(int64_t)k * n + i];
  out[i] = s;
}

inline unsigned nblocks(int64_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }

}  // namespace

// ---- internal launchers used by the engine ---------------------------------
int launch_minmax(const void* img, int dtype, int64_t n, double* part, double* out3,
                  cudaStream_t st) {
  k_minmax_part<<<kScanBlocks, kThreads, 0, st>>>(img, dtype, n, part);
  k_minmax_final<<<1, kThreads, 0, st>>>(part, kScanBlocks, out3);
  ++g_launches;
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}
size_t minmax_scratch_doubles() { return 3 * kScanBlocks; }

int launch_pairs(const void* img, int dtype, const void* clean, const double* mm, int H, int W,
                 int scheme, int clip, float* norm, float* pin, float* ptgt, int64_t plane,
                 cudaStream_t st) {
  const int64_t n = (int64_t)H * W;
  k_normalize<<<nblocks(n) < 2048 ? nblocks(n) : 2048, kThreads, 0, st>>>(img, dtype, n, mm, norm);
  const int64_t nq = (int64_t)(H / 2) * (W / 2);
  N2F_LAUNCH_CHECK();
  if (nq > 0) {
    k_pairs<<<nblocks(nq), kThreads, 0, st>>>(norm, clean, dtype, mm, H, W, scheme, clip, pin, ptgt,
                                              plane);
    N2F_LAUNCH_CHECK();
  }
  return N2F_OK;
}

uint64_t layer_key(uint64_t seed, int layer) {
  const uint64_t lseed = mix64(seed ^ (uint64_t)layer);  // derive_seed(seed, layer)
  return mix64(lseed);                                   // CounterRng key
}

int launch_init_layer(uint64_t seed, int layer, int cin, int cout, int k, float* w,
                      cudaStream_t st) {
  const int kk = k * k;
  const double bound = sqrt(6.0 / (double)(cin * kk));
  const int64_t total = (int64_t)cout * kk * cin;
  k_init_layer<<<nblocks(total), kThreads, 0, st>>>(layer_key(seed, layer), bound, cin, cout, kk, w);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int transpose_dgrad_weights(const float* w, float* wt, int cin, int cout, cudaStream_t st) {
  const int64_t total = (int64_t)cout * 9 * cin;
  k_transpose_dgrad<<<nblocks(total), kThreads, 0, st>>>(w, wt, cin, cout);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int reduce_partials(const float* part, float* out, int nsplit, int64_t n, cudaStream_t st) {
  k_reduce_partials<<<nblocks(n), kThreads, 0, st>>>(part, out, nsplit, n);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

}  // namespace n2f
