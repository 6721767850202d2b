// Training-loop kernels: multi-tensor Adam with fused deterministic split-K
// reduction, the device-side early-stopping state machine (with the FP16x3
// range guard), the output window mean, and the standalone loss / validation
// tail of the parity entry points (the engine fuses both into the L8
// epilogue, conv_tc.cu).
#include "n2f_internal.cuh"
#include "tc_common.cuh"
#include "loss_dev.cuh"
#include "train.cuh"

namespace n2f {
namespace {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// Multi-tensor Adam (tensor.py:125-141) with the split-K gradient reduction
// fused in, and the derived operand copies.  Each block reduces one (tensor,
// column chunk, row slab) rectangle of the [nsplit][n] partials: rl row lanes
// x cw columns, every lane summing its rows in a fixed order, lanes combined
// in a fixed order; tensors with several slabs park slab sums in scratch and
// the last-arriving block of the chunk adds them in slab order (the result
// does not depend on block scheduling: deterministic).  Then Adam with
// NumPy-2 semantics: every Python-float scalar is rounded to fp32 first and
// each operation is rounded separately (no FMA contraction).
// ---------------------------------------------------------------------------
constexpr int kAdamRowsPerLane = 16;
// One element's Adam update (NumPy-2 fp32 semantics, tensor.py:125-141) in
// registers, plus the scattered fp16 pair of the dgrad-transposed weight;
// m, v, p and the forward fp16 pair are stored by the caller.  rmax: max
// |p * 2^kExpW| of the pairs written (range guard).
__device__ __forceinline__ void adam_elem(const AdamArgs& args, const AdamTensor& T, int64_t j,
                                          float g, float bc1, float bc2, float& m, float& v, float& p,
                                          __half& h16, __half& l16, unsigned& rmax) {
  m = __fmul_rn(m, args.beta1);
  m = __fadd_rn(m, __fmul_rn(args.one_minus_beta1, g));
  v = __fmul_rn(v, args.beta2);
  v = __fadd_rn(v, __fmul_rn(args.one_minus_beta2, __fmul_rn(g, g)));
  const float mh = __fdiv_rn(m, bc1);
  const float vh = __fdiv_rn(v, bc2);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(args.lr, mh), __fadd_rn(__fsqrt_rn(vh), args.eps)));
  if (T.want16) {  // p * 2^kExpW
    const float a = __fmul_rn(p, args.wscale);
    rmax = max(rmax, tc::range_bits(a));
    tc::split_f16(a, h16, l16);
  }
  if (T.wt || T.wth16) {  // wt[c][8-tap][o] = w[o][tap][c]
    const int jj = (int)j;
    // cin is a power of two in the network (shift); 9 is a compile-time divisor
    const int r = T.cin_log2 >= 0 ? jj >> T.cin_log2 : jj / T.cin;
    const int cc = jj - r * T.cin;
    const int o = r / 9;
    const int tap = r - 9 * o;
    const int64_t q = ((int64_t)cc * 9 + (8 - tap)) * T.cout + o;
    if (T.wt) T.wt[q] = p;
    if (T.wth16) {
      T.wth16[q] = h16;
      T.wtl16[q] = l16;
    }
  }
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

__global__ void __launch_bounds__(kThreads)
    k_adam(AdamArgs args, const int* __restrict__ step_counter, int fixed_t) {
  __shared__ float red[kThreads];
  __shared__ int last;
  const int blk = blockIdx.x;
  int tl = 0, th = args.ntensors - 1;  // the tensor owning this block (binary search)
  while (tl < th) {
    const int mid = (tl + th + 1) >> 1;
    if (blk >= args.t[mid].blk0)
      tl = mid;
    else
      th = mid - 1;
  }
  const AdamTensor& T = args.t[tl];
  const int local = blk - T.blk0;
  if (T.vec == 4) {
    // wide tensors with <= 16 split rows: 4 columns per thread, every row of
    // partials in flight as float4 loads, then the update on a float4 of
    // moments / parameters (same per-element arithmetic and sum order)
    const int64_t j4 = ((int64_t)local * kThreads + threadIdx.x) * 4;
    if (j4 >= T.n) return;
    const int64_t i4 = T.off + j4;
    float4 m4 = *reinterpret_cast<const float4*>(args.m + i4);
    float4 v4 = *reinterpret_cast<const float4*>(args.v + i4);
    float4 p4 = *reinterpret_cast<const float4*>(args.p + i4);
    const float* __restrict__ part = T.part + j4;
    float4 x[kAdamRowsPerLane];
#pragma unroll
    for (int q = 0; q < kAdamRowsPerLane; ++q)
      x[q] = q < T.nsplit ? __ldg(reinterpret_cast<const float4*>(part + (int64_t)q * T.n))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 g4 = x[0];
#pragma unroll
    for (int q = 1; q < kAdamRowsPerLane; ++q) {
      if (q < T.nsplit) {
        g4.x += x[q].x;
        g4.y += x[q].y;
        g4.z += x[q].z;
        g4.w += x[q].w;
      }
    }
    const int t = step_counter ? *step_counter : fixed_t;
    const int ti = (t < args.table_len ? t : args.table_len) - 1;
    const float bc1 = args.bc1[ti], bc2 = args.bc2[ti];
    float* mv = &m4.x;
    float* vv = &v4.x;
    float* pv = &p4.x;
    const float* gv = &g4.x;
    __half h[4], l[4];
    unsigned rmax = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) adam_elem(args, T, j4 + e, gv[e], bc1, bc2, mv[e], vv[e], pv[e], h[e], l[e], rmax);
    *reinterpret_cast<float4*>(args.m + i4) = m4;
    *reinterpret_cast<float4*>(args.v + i4) = v4;
    *reinterpret_cast<float4*>(args.p + i4) = p4;
    if (T.want16) {
      *reinterpret_cast<uint2*>(args.phi16 + i4) = make_uint2(pack_h2(h[0], h[1]), pack_h2(h[2], h[3]));
      *reinterpret_cast<uint2*>(args.plo16 + i4) = make_uint2(pack_h2(l[0], l[1]), pack_h2(l[2], l[3]));
      if (T.amax) tc::range_note(T.amax, rmax);
    }
    return;
  }
  const int chunk = local / T.ns, slab = local - chunk * T.ns;
  const int cw = T.cw, rl = T.rl;
  const int c = threadIdx.x % cw, r = threadIdx.x / cw;
  const int64_t j = (int64_t)chunk * cw + c;
  const bool colok = j < T.n;
  const int rb = slab * kAdamRowsPerLane * rl;
  const int re = min(T.nsplit, rb + kAdamRowsPerLane * rl);
  // the Adam lanes fetch their moments and parameter while the partials load
  const int64_t i = T.off + j;
  const bool upd = r == 0 && colok;
  float m = 0.f, v = 0.f, p = 0.f;
  if (upd && T.ns == 1) {
    m = args.m[i];
    v = args.v[i];
    p = args.p[i];
  }
  float s = 0.f;
  if (colok) {
    // all (<= 16) partial rows of this lane in flight at once, then summed
    // in row order
    const float* __restrict__ part = T.part + j + (int64_t)(rb + r) * T.n;
    const int64_t stride = (int64_t)rl * T.n;
    const int nr = (re - rb - r + rl - 1) / rl;
    float x[kAdamRowsPerLane];
#pragma unroll
    for (int q = 0; q < kAdamRowsPerLane; ++q) x[q] = q < nr ? __ldg(part + q * stride) : 0.f;
    s = x[0];
#pragma unroll
    for (int q = 1; q < kAdamRowsPerLane; ++q)
      if (q < nr) s += x[q];
  }
  float g = s;
  if (rl > 1) {
    red[threadIdx.x] = s;
    __syncthreads();
    if (r == 0)
      for (int k = 1; k < rl; ++k) g += red[k * cw + c];
  }
  if (T.ns > 1) {
    if (r == 0 && colok) args.scratch[T.scr0 + (int64_t)slab * T.n + j] = g;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int prev = atomicAdd(args.counters + T.cnt0 + chunk, 1);
      last = prev == T.ns - 1;
      if (last) args.counters[T.cnt0 + chunk] = 0;  // self-reset for the next launch
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (r == 0 && colok) {
      const float* sc = args.scratch + T.scr0 + j;
      g = __ldcg(sc);
      for (int q = 1; q < T.ns; ++q) g += __ldcg(sc + (int64_t)q * T.n);
    }
  }
  if (!upd) return;
  if (T.ns > 1) {
    m = args.m[i];
    v = args.v[i];
    p = args.p[i];
  }
  const int t = step_counter ? *step_counter : fixed_t;
  const int ti = (t < args.table_len ? t : args.table_len) - 1;
  const float bc1 = args.bc1[ti], bc2 = args.bc2[ti];
  __half h16, l16;
  unsigned rmax = 0;
  adam_elem(args, T, j, g, bc1, bc2, m, v, p, h16, l16, rmax);
  args.m[i] = m;
  args.v[i] = v;
  args.p[i] = p;
  if (T.want16) {  // the forward operand pair of the tcgen05 kernels
    args.phi16[i] = h16;
    args.plo16[i] = l16;
    if (T.amax) tc::range_note(T.amax, rmax);
  }
}

// ---------------------------------------------------------------------------
// Dgrad-transposed weight pairs: one block per (layer, tap, 32 output x 32
// input channels) tile; reads rows of 32 consecutive input channels and
// writes rows of 32 consecutive output channels (64-byte segments both ways)
// through a shared-memory tile, for the hi and lo parts.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_transpose_pairs(TransposePairs t) {
  __shared__ unsigned short sh[2][32][33];
  const int b = blockIdx.x;
  int li = 1;
  while (li < 7 && b >= t.tile0[li + 1]) ++li;
  const int cin = t.cin[li], cout = t.cout[li];
  const int ctiles = (cin + 31) / 32, otiles = (cout + 31) / 32;
  int r = b - t.tile0[li];
  const int tap = r / (ctiles * otiles);
  r -= tap * ctiles * otiles;
  const int ob = r / ctiles, cb = r - ob * ctiles;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const unsigned short* whi = reinterpret_cast<const unsigned short*>(t.whi + t.off[li]);
  const unsigned short* wlo = reinterpret_cast<const unsigned short*>(t.wlo + t.off[li]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int o = ob * 32 + ty + 8 * k, c = cb * 32 + tx;
    if (o < cout && c < cin) {
      const int64_t i = ((int64_t)o * 9 + tap) * cin + c;
      sh[0][ty + 8 * k][tx] = __ldg(whi + i);
      sh[1][ty + 8 * k][tx] = __ldg(wlo + i);
    }
  }
  __syncthreads();
  unsigned short* thi = reinterpret_cast<unsigned short*>(t.thi[li]);
  unsigned short* tlo = reinterpret_cast<unsigned short*>(t.tlo[li]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = cb * 32 + ty + 8 * k, o = ob * 32 + tx;
    if (o < cout && c < cin) {
      const int64_t q = ((int64_t)c * 9 + (8 - tap)) * cout + o;
      thi[q] = sh[0][tx][ty + 8 * k];
      tlo[q] = sh[1][tx][ty + 8 * k];
    }
  }
}

// ---------------------------------------------------------------------------
// End-of-epoch bookkeeping (trainer.py:78-94): reduce the validation and loss
// partials in fixed order, record history, strict-improvement patience rule,
// and drive the graph's while-condition.  Range guard: the epoch's
// per-(class, layer) max |x * 2^e| slots move into range_hist[epoch] and are
// reset; a slot at or above kRangeLimit (or a non-finite score) stops the fit
// with N2F_STOP_RANGE instead of training on through inf/NaN operands.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
    k_stop(DevState* __restrict__ st, const double* __restrict__ part_se, int n_se, double pv,
           const double* __restrict__ part_loss, int n_loss, Pt4 pt,
           double* __restrict__ val_hist, double* __restrict__ loss_hist,
           unsigned long long* __restrict__ time_hist, int patience, int max_epochs,
           unsigned* __restrict__ range_cur, float* __restrict__ range_hist,
           cudaGraphConditionalHandle handle, int use_handle) {
  __shared__ double red[kThreads];
  __shared__ int bad_slot;
  if (threadIdx.x == 0) bad_slot = kRangeSlots;
  __syncthreads();
  if (range_cur && threadIdx.x < kRangeSlots) {
    const unsigned b = range_cur[threadIdx.x];
    range_cur[threadIdx.x] = 0u;
    if (range_hist) range_hist[(int64_t)st->epoch * kRangeSlots + threadIdx.x] = __uint_as_float(b);
    if (b >= __float_as_uint(kRangeLimit)) atomicMin(&bad_slot, (int)threadIdx.x);
  }
  double s = 0.0;
  for (int i = threadIdx.x; i < n_se; i += kThreads) s += part_se[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double score = red[0] / pv;
  __syncthreads();
  double losses[4];
  for (int q = 0; q < 4; ++q) {
    double l = 0.0;
    for (int i = threadIdx.x; i < n_loss; i += kThreads) l += part_loss[q * n_loss + i];
    red[threadIdx.x] = l;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    losses[q] = red[0] / pt.v[q];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  const int e = st->epoch;  // 0-based index of this epoch
  val_hist[e] = score;
  for (int q = 0; q < 4; ++q) loss_hist[4 * e + q] = losses[q];
  time_hist[e] = now;
  st->epoch = e + 1;
  if (score < st->best) {
    st->best = score;
    st->since = 0;
    st->best_epoch = e + 1;
  } else {
    st->since += 1;
  }
  int go = 1;
  if (bad_slot < kRangeSlots || !isfinite(score)) {
    st->stopped = 1;
    st->stop_reason = N2F_STOP_RANGE;
    st->range_slot = bad_slot < kRangeSlots ? bad_slot : -1;
    st->range_val = bad_slot < kRangeSlots ? range_hist ? range_hist[(int64_t)e * kRangeSlots + bad_slot]
                                                        : kRangeLimit
                                           : (float)score;
    go = 0;
  } else if (st->since >= patience) {
    st->stopped = 1;
    st->stop_reason = N2F_STOP_PATIENCE;
    go = 0;
  } else if (e + 1 >= max_epochs) {
    st->stopped = 1;
    st->stop_reason = N2F_STOP_MAX_EPOCHS;
    go = 0;
  }
  if (use_handle) cudaGraphSetConditional(handle, go);
}

// Mean of the buffered outputs in epoch order (sequential fp32 adds, then
// / fl32(n)), mapped back with f64 (x * (vmax - vmin) + vmin)
// (trainer.py:104-109, imaging.py:208-211).
__global__ void __launch_bounds__(kThreads)
    k_window_mean(const float* __restrict__ ring, int64_t plane, int window,
                  const DevState* __restrict__ st, int n_arg, int first_arg,
                  const double* __restrict__ mm, double vmin_arg, double vmax_arg,
                  double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= plane) return;
  int n = n_arg, first = first_arg;
  if (st) {
    n = st->epoch < window ? st->epoch : window;
    first = (st->epoch - n) % window;
  }
  const double vmin = mm ? mm[0] : vmin_arg;
  const double vmax = mm ? mm[1] : vmax_arg;
  auto slot = [&](int k) { return __ldg(ring + (int64_t)((first + k) % window) * plane + p); };
  float acc = slot(0);
  int k = 1;
  for (; k + 3 < n; k += 4) {  // four loads in flight, added in epoch order
    const float a0 = slot(k), a1 = slot(k + 1), a2 = slot(k + 2), a3 = slot(k + 3);
    acc = __fadd_rn(acc, a0);
    acc = __fadd_rn(acc, a1);
    acc = __fadd_rn(acc, a2);
    acc = __fadd_rn(acc, a3);
  }
  for (; k < n; ++k) acc = __fadd_rn(acc, slot(k));
  const float mean = __fdiv_rn(acc, (float)n);
  out[p] = __dadd_rn(__dmul_rn((double)mean, __dsub_rn(vmax, vmin)), vmin);
}

// Standalone loss on logits (parity entry point).
__global__ void __launch_bounds__(kThreads)
    k_loss(const float* __restrict__ z, const float* __restrict__ t, float* __restrict__ grad,
           int64_t n, int loss, double* __restrict__ part) {
  __shared__ double red[kThreads];
  const float nf = (float)n;
  const float two_over_n = (float)(2.0 / (double)n);
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float elem;
    grad[i] = loss_grad(z[i], t[i], loss, nf, two_over_n, &elem);
    s += elem;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(kThreads)
    k_val_tail(const float* __restrict__ z, const float* __restrict__ norm, float* __restrict__ out,
               int64_t n, double* __restrict__ part) {
  __shared__ double red[kThreads];
  const float tiny = __int_as_float(1), top = __int_as_float(0x3f7fffff);
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float o = fminf(fmaxf(sigmoid_ref(z[i]), tiny), top);
    out[i] = o;
    const double d = (double)o - (double)norm[i];
    s += d * d;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_sum_parts(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

__global__ void k_reset_state(DevState* st) {
  if (threadIdx.x == 0) {
    st->epoch = 0;
    st->step = 0;
    st->since = 0;
    st->stopped = 0;
    st->stop_reason = N2F_STOP_MAX_EPOCHS;
    st->best_epoch = 0;
    st->best = INFINITY;
    st->range_slot = -1;
    st->range_val = 0.f;
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    st->t0 = now;
  }
}

}  // namespace

// ---- launchers ---------------------------------------------------------------
void adam_plan(AdamArgs& a) {
  int blk = 0, cnt = 0;
  int64_t scr = 0;
  for (int q = 0; q < a.ntensors; ++q) {
    AdamTensor& T = a.t[q];
    const int ns_rows = T.nsplit < 1 ? 1 : T.nsplit;
    int rl = 1;
    while (rl < 32 && ns_rows > kAdamRowsPerLane * rl) rl <<= 1;
    T.rl = rl;
    T.cin_log2 = -1;
    for (int b = 0; b < 31; ++b)
      if (T.cin == (1 << b)) T.cin_log2 = b;
    // float4 columns: one row lane, 16-byte aligned rows and arena offset
    T.vec = (rl == 1 && T.n % 4 == 0 && T.off % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(T.part) & 15) == 0) ? 4 : 1;
    T.cw = kThreads * T.vec / rl;
    T.ns = (ns_rows + kAdamRowsPerLane * rl - 1) / (kAdamRowsPerLane * rl);
    T.nchunk = (int)((T.n + T.cw - 1) / T.cw);
    T.blk0 = blk;
    blk += T.nchunk * T.ns;
    T.cnt0 = cnt;
    T.scr0 = scr;
    if (T.ns > 1) {
      cnt += T.nchunk;
      scr += (int64_t)T.ns * T.n;
    }
  }
  a.nblocks = blk;
  a.cnt_total = cnt;
  a.scr_total = scr;
}

int launch_adam(const AdamArgs& args, const int* step_counter, int fixed_t, cudaStream_t st) {
  if (args.nblocks < 1) return fail(N2F_ERR_ARG, "launch_adam: no plan (adam_plan)");
  if (args.cnt_total && (!args.scratch || !args.counters))
    return fail(N2F_ERR_ARG, "launch_adam: plan needs scratch and counters");
  k_adam<<<(unsigned)args.nblocks, kThreads, 0, st>>>(args, step_counter, fixed_t);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int launch_transpose_pairs(const TransposePairs& t, cudaStream_t st) {
  k_transpose_pairs<<<(unsigned)t.tile0[8], 256, 0, st>>>(t);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int launch_stop(DevState* dst, const double* part_se, int n_se, double pv, const double* part_loss,
                int n_loss, const double pt[4], double* val_hist, double* loss_hist,
                unsigned long long* time_hist, int patience, int max_epochs, unsigned* range_cur,
                float* range_hist, cudaGraphConditionalHandle handle, int use_handle,
                cudaStream_t st) {
  Pt4 ptv{{pt[0], pt[1], pt[2], pt[3]}};
  k_stop<<<1, kThreads, 0, st>>>(dst, part_se, n_se, pv, part_loss, n_loss, ptv, val_hist, loss_hist,
                                 time_hist, patience, max_epochs, range_cur, range_hist, handle,
                                 use_handle);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int launch_window_mean(const float* ring, int64_t plane, int window, const DevState* dst, int n,
                       int first, const double* mm, double vmin, double vmax, double* out,
                       cudaStream_t st) {
  k_window_mean<<<(unsigned)((plane + kThreads - 1) / kThreads), kThreads, 0, st>>>(
      ring, plane, window, dst, n, first, mm, vmin, vmax, out);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int launch_loss(const float* z, const float* t, float* grad, int64_t n, int loss, double* part,
                int nblk, double* sum_out, cudaStream_t st) {
  k_loss<<<nblk, kThreads, 0, st>>>(z, t, grad, n, loss, part);
  k_sum_parts<<<1, 32, 0, st>>>(part, nblk, sum_out);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int launch_val_tail(const float* z, const float* norm, float* out, int64_t n, double* part, int nblk,
                    double* sum_out, cudaStream_t st) {
  k_val_tail<<<nblk, kThreads, 0, st>>>(z, norm, out, n, part);
  k_sum_parts<<<1, 32, 0, st>>>(part, nblk, sum_out);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int launch_reset_state(DevState* dst, cudaStream_t st) {
  k_reset_state<<<1, 32, 0, st>>>(dst);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

}  // namespace n2f
