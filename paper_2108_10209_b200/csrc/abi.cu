// Per-kernel C-ABI entry points (include/n2f.h) used by the parity suite.
// They run the same device kernels the engine runs, on caller-owned device
// buffers; scratch is allocated per call (test path, not the hot loop).
#include <math.h>

#include <vector>

#include "n2f_internal.cuh"
#include "train.cuh"

using namespace n2f;

namespace {

struct Scratch {
  std::vector<void*> ptrs;
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  int get(T** out, size_t count) {
    void* p = nullptr;
    N2F_CUDA(cudaMalloc(&p, count * sizeof(T) < 16 ? 16 : count * sizeof(T)));
    ptrs.push_back(p);
    *out = reinterpret_cast<T*>(p);
    return N2F_OK;
  }
};

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Test-only 1x1 convolution kernels (the engine fuses the 1x1 head).
__global__ void k_conv1x1_fwd(const float* __restrict__ x, const float* __restrict__ w,
                              const float* __restrict__ b, float* __restrict__ y, int64_t P, int cin,
                              int cout, int relu) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P * cout) return;
  const int64_t p = e / cout;
  const int o = (int)(e - p * cout);
  float a = 0.f;
  for (int c = 0; c < cin; ++c) a = fmaf(x[p * cin + c], w[(int64_t)o * cin + c], a);
  a += b[o];
  y[e] = relu ? fmaxf(a, 0.f) : a;
}

__global__ void k_conv1x1_dx(const float* __restrict__ g, const float* __restrict__ w,
                             const float* __restrict__ mask, float* __restrict__ dx, int64_t P,
                             int cin, int cout) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P * cin) return;
  const int64_t p = e / cin;
  const int c = (int)(e - p * cin);
  float a = 0.f;
  for (int o = 0; o < cout; ++o) a = fmaf(g[p * cout + o], w[(int64_t)o * cin + c], a);
  dx[e] = (mask && !(mask[e] > 0.f)) ? 0.f : a;
}

__global__ void k_conv1x1_dw(const float* __restrict__ g, const float* __restrict__ x,
                             float* __restrict__ dw, float* __restrict__ db, int64_t P, int cin,
                             int cout) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)cout * (cin + 1)) return;
  const int o = (int)(e / (cin + 1));
  const int c = (int)(e - (int64_t)o * (cin + 1));
  float a = 0.f;
  for (int64_t p = 0; p < P; ++p) a += g[p * cout + o] * (c < cin ? x[p * cin + c] : 1.f);
  if (c < cin) {
    if (dw) dw[(int64_t)o * cin + c] = a;
  } else if (db) {
    db[o] = a;
  }
}

unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

// Tensor-core operand (fp16 pair of x * 2^exp) of an fp32 device tensor
// (scratch-owned).
int make_operand(Scratch& s, const float* x, int64_t n, int exp, TcOperand* op, cudaStream_t st) {
  uint16_t *hi, *lo;
  N2F_TRY(s.get(&hi, (size_t)n));
  N2F_TRY(s.get(&lo, (size_t)n));
  N2F_TRY(split_f16(x, hi, lo, exp, n, st));
  *op = {hi, lo, exp};
  return N2F_OK;
}

int check_impl(int impl) {
  if (impl != kImplAuto && impl != kImplTcF16)
    return fail(N2F_ERR_UNSUPPORTED, "conv impl %d: this library implements only tcgen05 FP16x3 (0/3)",
                impl);
  return N2F_OK;
}

}  // namespace

extern "C" {

int n2f_minmax(const void* image, int dtype, int64_t n, double* out3, void* stream) {
  if (!image || !out3 || n < 1) return fail(N2F_ERR_ARG, "n2f_minmax: bad argument");
  Scratch s;
  double *part, *mm;
  N2F_TRY(s.get(&part, minmax_scratch_doubles()));
  N2F_TRY(s.get(&mm, 4));
  N2F_TRY(launch_minmax(image, dtype, n, part, mm, S(stream)));
  N2F_CUDA(cudaMemcpyAsync(out3, mm, 3 * sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  return N2F_OK;
}

int n2f_make_pairs(const void* image, int dtype, const void* clean, int height, int width,
                   double vmin, double vmax, int scheme, int clip_targets, float* norm,
                   float* pair_in, float* pair_tgt, int ph[4], int pw[4], void* stream) {
  if (!image || !norm || !pair_in || !pair_tgt || height < 2 || width < 2)
    return fail(N2F_ERR_ARG, "n2f_make_pairs: bad argument");
  if (scheme == 2 && !clean) return fail(N2F_ERR_ARG, "exact scheme needs the clean image");
  const int He = height & ~1, We = width & ~1;
  int64_t plane;
  if (scheme == 1) {
    for (int k = 0; k < 4; ++k) { ph[k] = He / 2; pw[k] = We / 2; }
    plane = (int64_t)(He / 2) * (We / 2);
  } else {
    ph[0] = ph[1] = He; pw[0] = pw[1] = We / 2;
    ph[2] = ph[3] = He / 2; pw[2] = pw[3] = We;
    plane = (int64_t)He * (We / 2);
  }
  Scratch s;
  double* mm;
  N2F_TRY(s.get(&mm, 4));
  const double h[2] = {vmin, vmax};
  N2F_CUDA(cudaMemcpyAsync(mm, h, sizeof h, cudaMemcpyHostToDevice, S(stream)));
  N2F_TRY(launch_pairs(image, dtype, clean, mm, height, width, scheme, clip_targets, norm, pair_in,
                       pair_tgt, plane, S(stream)));
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  return N2F_OK;
}

int n2f_init_layer(uint64_t seed, int layer, int cin, int cout, int k, float* w, void* stream) {
  if (!w || cin < 1 || cout < 1 || (k != 1 && k != 3)) return fail(N2F_ERR_ARG, "n2f_init_layer");
  N2F_TRY(launch_init_layer(seed, layer, cin, cout, k, w, S(stream)));
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  return N2F_OK;
}

int n2f_conv_fwd(const float* x, const float* w, const float* b, float* y, int h, int wd, int cin,
                 int cout, int k, int relu, int impl, void* stream) {
  if (!x || !w || !b || !y || h < 1 || wd < 1) return fail(N2F_ERR_ARG, "n2f_conv_fwd");
  N2F_TRY(check_impl(impl));
  const int64_t P = (int64_t)h * wd;
  if (k == 1) {
    k_conv1x1_fwd<<<nb(P * cout), 256, 0, S(stream)>>>(x, w, b, y, P, cin, cout, relu);
    N2F_LAUNCH_CHECK();
  } else if (k == 3 && cin == 1) {
    N2F_TRY(conv_first_simt(x, w, b, y, h, wd, cout, S(stream), relu));
  } else if (k == 3 && tc_supported(cin, cout)) {
    static Scratch s;  // kept alive across async calls on an explicit stream
    for (void* q : s.ptrs) cudaFree(q);
    s.ptrs.clear();
    TcOperand ox, ow;
    N2F_TRY(make_operand(s, x, P * cin, kExpAct, &ox, S(stream)));
    N2F_TRY(make_operand(s, w, (int64_t)cout * 9 * cin, kExpW, &ow, S(stream)));
    ConvTcPlan pl;
    N2F_TRY(conv_tc_plan(&pl, ox, ow, h, wd, cin, cout));
    N2F_TRY(conv_tc_plan_out(&pl, y, nullptr, nullptr, 1.f));
    N2F_TRY(conv_tc_launch(pl, b, nullptr, nullptr, relu ? kEpiBiasRelu : kEpiBias, S(stream)));
  } else {
    return fail(N2F_ERR_UNSUPPORTED, "conv_fwd: unsupported shape cin=%d cout=%d k=%d", cin, cout, k);
  }
  if (!stream) N2F_CUDA(cudaStreamSynchronize(S(stream)));  // async on an explicit stream
  return N2F_OK;
}

int n2f_conv_bwd(const float* g, const float* x, const float* w, const float* mask, float* dx,
                 float* dw, float* db, int h, int wd, int cin, int cout, int k, int impl,
                 void* stream) {
  if (!g || h < 1 || wd < 1) return fail(N2F_ERR_ARG, "n2f_conv_bwd");
  N2F_TRY(check_impl(impl));
  const int64_t P = (int64_t)h * wd;
  Scratch s;
  if (k == 1) {
    if (dx) {
      k_conv1x1_dx<<<nb(P * cin), 256, 0, S(stream)>>>(g, w, mask, dx, P, cin, cout);
      N2F_LAUNCH_CHECK();
    }
    if (dw || db) {
      k_conv1x1_dw<<<nb((int64_t)cout * (cin + 1)), 256, 0, S(stream)>>>(g, x, dw, db, P, cin, cout);
      N2F_LAUNCH_CHECK();
    }
    N2F_CUDA(cudaStreamSynchronize(S(stream)));
    return N2F_OK;
  }
  if (k != 3) return fail(N2F_ERR_UNSUPPORTED, "conv_bwd: k=%d", k);
  if (dx && !tc_supported(cout, cin))
    return fail(N2F_ERR_UNSUPPORTED, "conv_bwd dgrad: cin %d cout %d", cin, cout);
  if (dw && !(cin == 1 && cout == 32) && !tc_supported(cin, cout))
    return fail(N2F_ERR_UNSUPPORTED, "conv_bwd wgrad: cin %d cout %d", cin, cout);
  // db: the column sums of g ([P][cout]) -- the fixed-order partial reduction
  // with one "split" per pixel (inside the engine they come from the dgrad /
  // head epilogues and the first-layer wgrad)
  if (db) N2F_TRY(reduce_partials(g, db, (int)P, cout, S(stream)));
  if (dw && cin == 1) {
    const int ns = wgrad_first_nsplit(P);
    float *pw, *pb;
    N2F_TRY(s.get(&pw, (size_t)ns * cout * 9));
    N2F_TRY(s.get(&pb, (size_t)ns * cout));
    N2F_TRY(wgrad_first_simt(g, x, pw, pb, h, wd, cout, ns, S(stream)));
    N2F_TRY(reduce_partials(pw, dw, ns, (int64_t)cout * 9, S(stream)));
  } else if (dw) {
    const int nst = wgrad_tc_nsplit(cin, cout, h, wd);
    float* ptc;
    N2F_TRY(s.get(&ptc, (size_t)nst * cout * 9 * cin));
    TcOperand ox, og;
    N2F_TRY(make_operand(s, x, P * cin, kExpAct, &ox, S(stream)));
    N2F_TRY(make_operand(s, g, P * cout, kExpAct, &og, S(stream)));
    WgradTcPlan pl;
    N2F_TRY(wgrad_tc_plan(&pl, ox, og, h, wd, cin, cout, nst));
    N2F_TRY(wgrad_tc_launch(pl, ptc, S(stream)));
    N2F_TRY(reduce_partials(ptc, dw, nst, (int64_t)cout * 9 * cin, S(stream)));
  }
  if (dx) {
    float* wt;
    N2F_TRY(s.get(&wt, (size_t)cout * 9 * cin));
    N2F_TRY(transpose_dgrad_weights(w, wt, cin, cout, S(stream)));
    TcOperand og, owt, omask;
    N2F_TRY(make_operand(s, g, P * cout, kExpAct, &og, S(stream)));
    N2F_TRY(make_operand(s, wt, (int64_t)cout * 9 * cin, kExpW, &owt, S(stream)));
    const void* mk = nullptr;
    if (mask) {  // the epilogue tests the sign of the fp16 hi tensor of the layer input
      N2F_TRY(make_operand(s, mask, P * cin, kExpAct, &omask, S(stream)));
      mk = omask.hi;
    }
    ConvTcPlan pl;
    N2F_TRY(conv_tc_plan(&pl, og, owt, h, wd, cout, cin));
    N2F_TRY(conv_tc_plan_out(&pl, dx, nullptr, nullptr, 1.f));
    N2F_TRY(conv_tc_launch(pl, nullptr, mk, nullptr, mask ? kEpiMask : kEpiNone, S(stream)));
  }
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  return N2F_OK;
}

int n2f_loss(const float* z, const float* t, float* grad, int64_t n, int loss, double* loss_out,
             void* stream) {
  if (!z || !t || !grad || n < 1 || (loss != 0 && loss != 1)) return fail(N2F_ERR_ARG, "n2f_loss");
  Scratch s;
  double *part, *sum;
  const int nblk = 296;
  N2F_TRY(s.get(&part, nblk));
  N2F_TRY(s.get(&sum, 1));
  N2F_TRY(launch_loss(z, t, grad, n, loss, part, nblk, sum, S(stream)));
  double hs = 0.0;
  N2F_CUDA(cudaMemcpyAsync(&hs, sum, 8, cudaMemcpyDeviceToHost, S(stream)));
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  if (loss_out) *loss_out = hs / (double)n;
  return N2F_OK;
}

int n2f_adam(float* p, const float* g, float* m, float* v, int64_t n, int t, double lr,
             void* stream) {
  if (!p || !g || !m || !v || n < 1 || t < 1) return fail(N2F_ERR_ARG, "n2f_adam");
  Scratch s;
  float* tab;
  N2F_TRY(s.get(&tab, 2));
  const float h[2] = {(float)(1.0 - pow(0.9, (double)t)), (float)(1.0 - pow(0.999, (double)t))};
  N2F_CUDA(cudaMemcpyAsync(tab, h, sizeof h, cudaMemcpyHostToDevice, S(stream)));
  AdamArgs a{};
  a.ntensors = 1;
  a.total = n;
  a.p = p;
  a.m = m;
  a.v = v;
  a.bc1 = tab;
  a.bc2 = tab + 1;
  a.table_len = 1;
  a.beta1 = 0.9f;
  a.one_minus_beta1 = (float)(1.0 - 0.9);
  a.beta2 = 0.999f;
  a.one_minus_beta2 = (float)(1.0 - 0.999);
  a.lr = (float)lr;
  a.eps = 1e-8f;
  a.t[0].off = 0;
  a.t[0].n = n;
  a.t[0].part = g;
  a.t[0].nsplit = 1;
  a.t[0].wt = nullptr;
  adam_plan(a);
  N2F_TRY(launch_adam(a, nullptr, 1, S(stream)));
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  return N2F_OK;
}

int n2f_validate_tail(const float* z, const float* norm, float* out, int64_t n, double* score,
                      void* stream) {
  if (!z || !norm || !out || n < 1) return fail(N2F_ERR_ARG, "n2f_validate_tail");
  Scratch s;
  double *part, *sum;
  const int nblk = 296;
  N2F_TRY(s.get(&part, nblk));
  N2F_TRY(s.get(&sum, 1));
  N2F_TRY(launch_val_tail(z, norm, out, n, part, nblk, sum, S(stream)));
  double hs = 0.0;
  N2F_CUDA(cudaMemcpyAsync(&hs, sum, 8, cudaMemcpyDeviceToHost, S(stream)));
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  if (score) *score = hs / (double)n;
  return N2F_OK;
}

int n2f_stop_replay(const double* scores, int n, int patience, int* stop_epoch) {
  if (!scores || n < 0 || patience < 1 || !stop_epoch) return fail(N2F_ERR_ARG, "n2f_stop_replay");
  Scratch s;
  DevState* st;
  double *se, *loss, *vh, *lh;
  unsigned long long* th;
  N2F_TRY(s.get(&st, 1));
  N2F_TRY(s.get(&se, n > 0 ? n : 1));
  N2F_TRY(s.get(&loss, 4));
  N2F_TRY(s.get(&vh, n > 0 ? n : 1));
  N2F_TRY(s.get(&lh, 4 * (n > 0 ? n : 1)));
  N2F_TRY(s.get(&th, n > 0 ? n : 1));
  N2F_CUDA(cudaMemset(loss, 0, 4 * sizeof(double)));
  if (n > 0) N2F_CUDA(cudaMemcpy(se, scores, n * sizeof(double), cudaMemcpyHostToDevice));
  N2F_TRY(launch_reset_state(st, 0));
  const double pt[4] = {1, 1, 1, 1};
  *stop_epoch = -1;
  for (int e = 0; e < n; ++e) {
    // max_epochs beyond the sequence so only the patience rule can stop it
    N2F_TRY(launch_stop(st, se + e, 1, 1.0, loss, 1, pt, vh, lh, th, patience, n + 1, nullptr, nullptr, 0, 0, 0));
    DevState h;
    N2F_CUDA(cudaMemcpy(&h, st, sizeof h, cudaMemcpyDeviceToHost));
    if (h.stopped) {
      *stop_epoch = e + 1;
      break;
    }
  }
  return N2F_OK;
}

int n2f_window_mean(const float* ring, int n_slots, int first_slot, int n, int64_t plane,
                    double vmin, double vmax, double* out, void* stream) {
  if (!ring || !out || n < 1 || n > n_slots || first_slot < 0 || first_slot >= n_slots)
    return fail(N2F_ERR_ARG, "n2f_window_mean");
  N2F_TRY(launch_window_mean(ring, plane, n_slots, nullptr, n, first_slot, nullptr, vmin, vmax, out,
                             S(stream)));
  N2F_CUDA(cudaStreamSynchronize(S(stream)));
  return N2F_OK;
}

}  // extern "C"
