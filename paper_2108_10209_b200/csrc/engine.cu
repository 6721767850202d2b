// The per-image fit-and-denoise engine: context (workspaces sized once per
// image shape), one training epoch as a fixed kernel sequence, the whole loop
// as ONE CUDA graph with a device-driven while node, and the C-ABI entry
// points of include/n2f.h that drive it.
//
// Hot path restated (reference trainer.py:125-213):
//   normalise + 4 training pairs        -> prep.cu (bit-exact)
//   build_network (He-uniform, seeded)   -> prep.cu k_init_layer (bit-exact)
//   per epoch: 4 x [fwd L1..L8, fused head+loss+head-bwd, wgrad/dgrad L8..L1,
//              Adam], full-res validation fwd + head, stop-state update
//   finalize: window mean + denormalise  -> train.cu k_window_mean (bit-exact)
#include <math.h>
#include <string.h>

#include <vector>

#include "n2f_internal.cuh"
#include "train.cuh"

using namespace n2f;

struct n2f_ctx {
  int device = 0;
  int H = 0, W = 0;
  n2f_config cfg{};
  cudaStream_t stream = nullptr;

  // geometry
  int ph[4]{}, pw[4]{};
  int64_t plane = 0;  // elements of one training plane
  int64_t Pt = 0;     // pixels per training pair (identical for the 4 pairs)
  int64_t Pv = 0;     // validation pixels (H*W)

  // device buffers: each allocation is bracketed by guard bytes (a fixed
  // pattern checked by n2f_ctx_check_guards -- the out-of-bounds-write check
  // that runs everywhere, compute-sanitizer being unavailable on the GPU pool)
  std::vector<void*> allocs;     // base pointers (guard included)
  std::vector<size_t> alloc_bytes;  // payload bytes of each
  size_t bytes = 0;
  void* img = nullptr;    // staging input (H*W f64)
  void* clean = nullptr;  // staging clean image (exact scheme)
  double* mm = nullptr;   // {vmin, vmax, nonfinite}
  double* mm_part = nullptr;
  float* norm = nullptr;  // H*W f32
  float* pin = nullptr;   // 4 planes
  float* ptgt = nullptr;  // 4 planes
  float* params = nullptr;
  float* m = nullptr;
  float* v = nullptr;
  int64_t poff[2 * kLayers]{};  // tensor offsets in the arena (w0,b0,w1,b1,...)
  int64_t pnum[2 * kLayers]{};
  int64_t ptotal = 0;
  float* wt[kLayers]{};  // dgrad-transposed weights (layers 1..7), fp32 master copy
  float* z = nullptr;     // logits of the last training step
  float* gB = nullptr;    // L1 dgrad output (fp32: the first-layer wgrad input)
  float* ring = nullptr;
  int nsplit0 = 0;  // pixel splits of the first-layer wgrad
  float* part_w[kLayers]{};
  float* part_b[kLayers]{};
  int nblk_head = 0, nblk_val = 0;
  double* part_loss = nullptr;  // [4][nblk_head]
  double* part_se = nullptr;    // [nblk_val]
  DevState* dstate = nullptr;
  int* step_counter = nullptr;
  double* val_hist = nullptr;
  double* loss_hist = nullptr;
  unsigned long long* time_hist = nullptr;
  float* bc1 = nullptr;
  float* bc2 = nullptr;
  int table_len = 0;
  double* out_stage = nullptr;  // H*W f64 for the host API
  unsigned* range_cur = nullptr;  // [kRangeSlots] this epoch's max |x * 2^e| (float bits)
  float* range_hist = nullptr;    // [max_epochs][kRangeSlots]

  // host pinned mirrors
  double* h_mm = nullptr;
  DevState* h_state = nullptr;

  // graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t epoch_launches = 0;  // kernels in one captured epoch body

  // tcgen05 FP16x3 operands: fp16 (hi, lo) pairs of the scaled tensors;
  // activations and weights carry 2^kExpAct / 2^kExpW, gradients 2^exp_g
  // (see setup)
  int exp_g = 0;
  __half* w16[2] = {};            // hi, lo arenas (same layout as params)
  __half* wt16[2][kLayers] = {};  // dgrad-transposed pairs
  __half* act16[2][kLayers] = {}; // layer outputs 0..6
  __half* g16[2][2] = {};         // [A/B][hi/lo] gradient ping-pong
  __half* v16[2][2] = {};         // [A/B][hi/lo] validation ping-pong
  uint32_t* mbits[kLayers] = {};  // bit-packed ReLU masks of the tcgen05 forward outputs (L2..L7)
  ConvTcPlan fwd_plan[2][kLayers]{};
  ConvTcPlan dgrad_plan[2][kLayers]{};
  ConvTcPlan val_plan[kLayers]{};
  WgradTcPlan wgrad_plan[2][kLayers]{};
  AdamArgs adam_sc[2]{};  // per training-plane shape class
  TransposePairs tpose{};  // Adam's forward weight pairs -> dgrad-transposed pairs
  // profiling
  struct Mark {
    int cls, li;
    double flop;
    cudaEvent_t a, b;
  };
  bool prof = false;
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  int wsplit[2][kLayers]{};
  int last_sc = 0;  // shape class of the last enqueued step (parity readback)
};

namespace {

constexpr size_t kGuardBytes = 256;
constexpr int kGuardByte = 0xA5;

template <typename T>
int dalloc(n2f_ctx* c, T** p, size_t count) {
  void* q = nullptr;
  const size_t b = count * sizeof(T);
  const size_t pb = (b + 255) / 256 * 256;  // payload rounded to the guard alignment
  N2F_CUDA(cudaMalloc(&q, pb + 2 * kGuardBytes));
  c->allocs.push_back(q);
  c->alloc_bytes.push_back(pb);
  c->bytes += b;
  uint8_t* base = reinterpret_cast<uint8_t*>(q);
  N2F_CUDA(cudaMemset(base, kGuardByte, kGuardBytes));
  N2F_CUDA(cudaMemset(base + kGuardBytes + pb, kGuardByte, kGuardBytes));
  *p = reinterpret_cast<T*>(base + kGuardBytes);
  return N2F_OK;
}

const float* W_(n2f_ctx* c, int li) { return c->params + c->poff[2 * li]; }
const float* B_(n2f_ctx* c, int li) { return c->params + c->poff[2 * li + 1]; }
unsigned* RS_(n2f_ctx* c, int cls, int li) { return c->range_cur + cls * kLayers + li; }

// training-plane shape class of pair k (checkerboard: up pairs 0,1 vs left 2,3)
int shape_class(const n2f_ctx* c, int k) {
  return (c->ph[k] == c->ph[0] && c->pw[k] == c->pw[0]) ? 0 : 1;
}

// ---- per-kernel-class profiling (CUDA events around each launch, host loop)
enum ProfClass {
  kPFirst = 0, kPFwd, kPHead, kPWgrad, kPDgrad, kPWgradFirst, kPAdam, kPValFirst, kPValConv,
  kPHeadVal, kPStop, kPClasses
};

cudaEvent_t prof_event(n2f_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

// Run `call` (returns a status); when profiling, bracket it with events and
// charge the algorithmic FLOPs to (class, layer).
#define PROF(cls, li, flop, call)                                   \
  do {                                                              \
    cudaEvent_t a_ = nullptr;                                       \
    if (c->prof) {                                                  \
      a_ = prof_event(c);                                           \
      cudaEventRecord(a_, c->stream);                               \
    }                                                               \
    N2F_TRY(call);                                                  \
    if (c->prof) {                                                  \
      cudaEvent_t b_ = prof_event(c);                               \
      cudaEventRecord(b_, c->stream);                               \
      c->marks.push_back({(int)(cls), (int)(li), (double)(flop), a_, b_}); \
    }                                                               \
  } while (0)

double conv_flop(int64_t P, int li) { return 2.0 * P * kCout[li] * kKsz[li] * kKsz[li] * kCin[li]; }

// One training step on pair k (model.forward / _loss_and_grad / backward /
// apply_gradients, model.py:72-120, trainer.py:184-190): L1 forward, L2..L8
// forward on the tensor cores (L8 with the L9 head, loss and head backward
// fused), then per layer L8..L2 the wgrad (split-K partials) and the masked
// dgrad (whose epilogue also writes the bias-gradient column sums of the
// layer below), the L1 wgrad, and Adam (reducing every partial in fixed order).
int enqueue_step(n2f_ctx* c, int k) {
  cudaStream_t st = c->stream;
  const int sc = shape_class(c, k);
  c->last_sc = sc;
  const int h = c->ph[k], w = c->pw[k];
  const int64_t P = (int64_t)h * w;
  const float* x0 = c->pin + k * c->plane;
  const float* tgt = c->ptgt + k * c->plane;
  PROF(kPFirst, 0, conv_flop(P, 0),
       conv_first_simt(x0, W_(c, 0), B_(c, 0), nullptr, h, w, kCout[0], st, 1, c->act16[0][0],
                       c->act16[1][0], ldexpf(1.f, kExpAct), RS_(c, kRangeAct, 0)));
  for (int li = 1; li < 7; ++li)
    PROF(kPFwd, li, conv_flop(P, li),
         conv_tc_launch(c->fwd_plan[sc][li], B_(c, li), nullptr, nullptr, kEpiBiasRelu, st));
  HeadTrainArgs ht{W_(c, 8), B_(c, 8), tgt, c->z, c->part_w[8], c->part_b[8],
                   c->part_loss + (int64_t)k * c->nblk_head, c->step_counter, c->cfg.loss,
                   (float)P, (float)(2.0 / (double)P)};
  PROF(kPFwd, 7, conv_flop(P, 7) + 6.0 * P * kMaxC,
       conv_tc_launch_head_train(c->fwd_plan[sc][7], B_(c, 7), c->part_b[7], ht, st));
  for (int li = 7; li >= 1; --li) {
    PROF(kPWgrad, li, conv_flop(P, li), wgrad_tc_launch(c->wgrad_plan[sc][li], c->part_w[li], st));
    const void* mask = c->mbits[li - 1] ? (const void*)c->mbits[li - 1] : (const void*)c->act16[0][li - 1];
    PROF(kPDgrad, li, conv_flop(P, li),
         conv_tc_launch(c->dgrad_plan[sc][li], nullptr, mask, li > 1 ? c->part_b[li - 1] : nullptr,
                        kEpiMask, st));
  }
  PROF(kPWgradFirst, 0, conv_flop(P, 0),
       wgrad_first_simt(c->gB, x0, c->part_w[0], c->part_b[0], h, w, kCout[0], c->nsplit0, st));
  PROF(kPAdam, 0, 0.0, launch_adam(c->adam_sc[sc], c->step_counter, 0, st));
  PROF(kPAdam, 1, 0.0, launch_transpose_pairs(c->tpose, st));
  return N2F_OK;
}

// Full-resolution validation (trainer.validate -> model.predict, trainer.py:97-101,
// model.py:123-140): forward with the head fused into L8 (sigmoid, clip, ring
// slot, squared-error partials).
int enqueue_validate(n2f_ctx* c) {
  cudaStream_t st = c->stream;
  PROF(kPValFirst, 0, conv_flop(c->Pv, 0),
       conv_first_simt(c->norm, W_(c, 0), B_(c, 0), nullptr, c->H, c->W, kCout[0], st, 1,
                       c->v16[0][0], c->v16[0][1], ldexpf(1.f, kExpAct), RS_(c, kRangeValAct, 0)));
  for (int li = 1; li < 7; ++li)
    PROF(kPValConv, li, conv_flop(c->Pv, li),
         conv_tc_launch(c->val_plan[li], B_(c, li), nullptr, nullptr, kEpiBiasRelu, st));
  HeadValArgs hv{W_(c, 8), B_(c, 8), c->norm, c->ring, c->dstate, c->cfg.avg_window, c->part_se};
  PROF(kPValConv, 7, conv_flop(c->Pv, 7) + 2.0 * c->Pv * kMaxC,
       conv_tc_launch_head_val(c->val_plan[7], B_(c, 7), hv, st));
  return N2F_OK;
}

int enqueue_epoch(n2f_ctx* c, int use_handle) {
  for (int k = 0; k < 4; ++k) N2F_TRY(enqueue_step(c, k));
  N2F_TRY(enqueue_validate(c));
  const double pt[4] = {(double)c->Pt, (double)c->Pt, (double)c->Pt, (double)c->Pt};
  PROF(kPStop, 0, 0.0,
       launch_stop(c->dstate, c->part_se, c->nblk_val, (double)c->Pv, c->part_loss, c->nblk_head,
                   pt, c->val_hist, c->loss_hist, c->time_hist, c->cfg.patience_epochs,
                   c->cfg.max_epochs, c->range_cur, c->range_hist, c->handle, use_handle,
                   c->stream));
  return N2F_OK;
}

int build_graph(n2f_ctx* c) {
  N2F_CUDA(cudaGraphCreate(&c->graph, 0));
  N2F_CUDA(cudaGraphConditionalHandleCreate(&c->handle, c->graph, 1, cudaGraphCondAssignDefault));
  // cudaGraphNodeParams has a deleted default constructor (union member);
  // build it in zeroed raw storage.
  alignas(cudaGraphNodeParams) unsigned char raw[sizeof(cudaGraphNodeParams)];
  memset(raw, 0, sizeof raw);
  cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(raw);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = c->handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  N2F_CUDA(cudaGraphAddNode(&node, c->graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  N2F_CUDA(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
  const int64_t before = g_launches;
  int s = enqueue_epoch(c, 1);
  c->epoch_launches = g_launches - before;
  g_launches = before;  // captured, not executed
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->stream, &captured);
  if (s != N2F_OK) return s;
  N2F_CUDA(e);
  N2F_CUDA(cudaGraphInstantiate(&c->exec, c->graph, 0));
  return N2F_OK;
}

// Reduction plan of an Adam descriptor (k_adam sums the split-K partials
// itself) plus its slab scratch and self-resetting arrival counters.
int plan_adam(n2f_ctx* c, AdamArgs& a) {
  adam_plan(a);
  a.scratch = nullptr;
  a.counters = nullptr;
  if (a.scr_total) N2F_TRY(dalloc(c, &a.scratch, (size_t)a.scr_total));
  if (a.cnt_total) {
    N2F_TRY(dalloc(c, &a.counters, (size_t)a.cnt_total));
    N2F_CUDA(cudaMemset(a.counters, 0, (size_t)a.cnt_total * sizeof(int)));
  }
  return N2F_OK;
}

int setup(n2f_ctx* c) {
  N2F_CUDA(cudaSetDevice(c->device));
  N2F_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  N2F_CUDA(cudaEventCreate(&c->ev0));
  N2F_CUDA(cudaEventCreate(&c->ev1));
  const int H = c->H, W = c->W;
  const int He = H & ~1, We = W & ~1;
  if (c->cfg.scheme == 1) {
    for (int k = 0; k < 4; ++k) { c->ph[k] = He / 2; c->pw[k] = We / 2; }
    c->plane = (int64_t)(He / 2) * (We / 2);
  } else {
    c->ph[0] = c->ph[1] = He; c->pw[0] = c->pw[1] = We / 2;
    c->ph[2] = c->ph[3] = He / 2; c->pw[2] = c->pw[3] = We;
    c->plane = (int64_t)He * (We / 2);
  }
  c->Pt = c->plane;
  c->Pv = (int64_t)H * W;

  N2F_TRY(dalloc(c, reinterpret_cast<double**>(&c->img), c->Pv));
  if (c->cfg.scheme == 2) N2F_TRY(dalloc(c, reinterpret_cast<double**>(&c->clean), c->Pv));
  N2F_TRY(dalloc(c, &c->mm, 4));
  N2F_TRY(dalloc(c, &c->mm_part, minmax_scratch_doubles()));
  N2F_TRY(dalloc(c, &c->norm, c->Pv));
  N2F_TRY(dalloc(c, &c->pin, 4 * c->plane));
  N2F_TRY(dalloc(c, &c->ptgt, 4 * c->plane));

  int64_t off = 0;
  for (int li = 0; li < kLayers; ++li) {
    c->poff[2 * li] = off;
    c->pnum[2 * li] = (int64_t)kCout[li] * kKsz[li] * kKsz[li] * kCin[li];
    off += c->pnum[2 * li];
    c->poff[2 * li + 1] = off;
    c->pnum[2 * li + 1] = kCout[li];
    off += kCout[li];
  }
  c->ptotal = off;
  N2F_TRY(dalloc(c, &c->params, off));
  N2F_TRY(dalloc(c, &c->m, off));
  N2F_TRY(dalloc(c, &c->v, off));
  for (int li = 1; li < 8; ++li) N2F_TRY(dalloc(c, &c->wt[li], c->pnum[2 * li]));
  // layer outputs live as fp16 operand pairs (below) and the L9 head is fused
  // into L8's epilogue; the only fp32 layer buffer is the L1 dgrad output
  N2F_TRY(dalloc(c, &c->z, c->Pt));
  N2F_TRY(dalloc(c, &c->gB, c->Pt * kCout[0]));
  N2F_TRY(dalloc(c, &c->ring, (int64_t)c->cfg.avg_window * c->Pv));
  N2F_TRY(dalloc(c, &c->range_cur, kRangeSlots));
  N2F_CUDA(cudaMemset(c->range_cur, 0, kRangeSlots * sizeof(unsigned)));
  N2F_TRY(dalloc(c, &c->range_hist, (int64_t)c->cfg.max_epochs * kRangeSlots));

  // split-K partial buffers: the bias gradient of layer li (1..6) is a
  // per-tile column sum written by the dgrad of layer li+1, L8's by the fused
  // head; weight gradients use the tcgen05 wgrad's split count
  c->nsplit0 = wgrad_first_nsplit(c->Pt);
  const int tiles[2] = {conv_tc_tiles(c->ph[0], c->pw[0]), conv_tc_tiles(c->ph[2], c->pw[2])};
  const int max_tiles = tiles[0] > tiles[1] ? tiles[0] : tiles[1];
  for (int sc = 0; sc < 2; ++sc)
    for (int li = 1; li < 8; ++li)
      c->wsplit[sc][li] = wgrad_tc_nsplit(kCin[li], kCout[li], c->ph[2 * sc], c->pw[2 * sc]);
  for (int li = 0; li < kLayers; ++li) {
    int64_t nb, nw;
    if (li == 0) {
      nb = nw = c->nsplit0;
    } else if (li == 8) {  // fused head: per-tile db9, per-(tile, warp group) dW9
      nb = max_tiles;
      nw = 4 * (int64_t)max_tiles;
    } else {
      nb = max_tiles;
      nw = c->wsplit[0][li] > c->wsplit[1][li] ? c->wsplit[0][li] : c->wsplit[1][li];
    }
    N2F_TRY(dalloc(c, &c->part_w[li], nw * c->pnum[2 * li]));
    N2F_TRY(dalloc(c, &c->part_b[li], nb * c->pnum[2 * li + 1]));
  }
  // gradient scale: |dL/dz| <= 1/P per pixel, so 2^ceil(log2 P) lifts the
  // head gradient to O(1); kExpAct more keeps small entries out of the
  // fp16 subnormal range
  int lg = 0;
  while ((int64_t(1) << lg) < c->Pt) ++lg;
  c->exp_g = lg + kExpAct;
  for (int q = 0; q < 2; ++q) {
    N2F_TRY(dalloc(c, &c->w16[q], c->ptotal));
    for (int li = 1; li < 8; ++li) N2F_TRY(dalloc(c, &c->wt16[q][li], c->pnum[2 * li]));
    for (int li = 0; li < 7; ++li) N2F_TRY(dalloc(c, &c->act16[q][li], c->Pt * kCout[li]));
    for (int ab = 0; ab < 2; ++ab) {
      N2F_TRY(dalloc(c, &c->g16[ab][q], c->Pt * kMaxC));
      N2F_TRY(dalloc(c, &c->v16[ab][q], c->Pv * kMaxC));
    }
  }
  // operand pairs of layer li's input activation, its weights (forward and
  // dgrad-transposed) and the gradient buffer A (ab 0) or B (ab 1)
  auto act_op = [&](int li) { return TcOperand{c->act16[0][li], c->act16[1][li], kExpAct}; };
  auto w_op = [&](int li) {
    const int64_t o = c->poff[2 * li];
    return TcOperand{c->w16[0] + o, c->w16[1] + o, kExpW};
  };
  auto wt_op = [&](int li) { return TcOperand{c->wt16[0][li], c->wt16[1][li], kExpW}; };
  auto g_op = [&](int ab) { return TcOperand{c->g16[ab][0], c->g16[ab][1], c->exp_g}; };
  auto v_op = [&](int ab) { return TcOperand{c->v16[ab][0], c->v16[ab][1], kExpAct}; };
  const float sa = ldexpf(1.f, kExpAct), sg = ldexpf(1.f, c->exp_g);
  // the tcgen05 forward outputs (L2..L7) also emit their ReLU mask bit-packed
  // for the dgrad above them: one word per 32 channels and pixel instead of
  // re-reading the fp16 activation as the mask (dgrad L4 -17 %; the L2 dgrad
  // reads the L1 activation: emitting bits from the first-layer kernel cost
  // more there than the dgrad gained)
  for (int li = 1; li < 7; ++li) N2F_TRY(dalloc(c, &c->mbits[li], c->Pt * (kCout[li] / 32)));
  for (int sc = 0; sc < 2; ++sc) {
    const int h = c->ph[2 * sc], w = c->pw[2 * sc];
    for (int li = 1; li < 8; ++li) {
      // forward: outputs are the next layer's operand pair; L8 (head fused)
      // writes the L8 gradient pair (the dgrad/wgrad input)
      ConvTcPlan& fp = c->fwd_plan[sc][li];
      N2F_TRY(conv_tc_plan(&fp, act_op(li - 1), w_op(li), h, w, kCin[li], kCout[li]));
      if (li == 7) {
        N2F_TRY(conv_tc_plan_out(&fp, nullptr, c->g16[0][0], c->g16[0][1], sg));
        N2F_TRY(conv_tc_plan_range(&fp, RS_(c, kRangeGrad, 7)));
      } else {
        N2F_TRY(conv_tc_plan_out(&fp, nullptr, c->act16[0][li], c->act16[1][li], sa));
        N2F_TRY(conv_tc_plan_range(&fp, RS_(c, kRangeAct, li)));
      }
      if (c->mbits[li]) N2F_TRY(conv_tc_plan_maskbits(&fp, c->mbits[li], 0));
      // dgrad: reads gradient buffer ab (L8's is A, the head output), writes
      // the other; L1's output feeds the first-layer wgrad in fp32
      const int ab = (li & 1) ? 0 : 1;
      ConvTcPlan& dp = c->dgrad_plan[sc][li];
      N2F_TRY(conv_tc_plan(&dp, g_op(ab), wt_op(li), h, w, kCout[li], kCin[li]));
      const int nb = 1 - ab;
      if (li == 1) {
        N2F_TRY(conv_tc_plan_out(&dp, c->gB, nullptr, nullptr, sg));
      } else {
        N2F_TRY(conv_tc_plan_out(&dp, nullptr, c->g16[nb][0], c->g16[nb][1], sg));
        N2F_TRY(conv_tc_plan_range(&dp, RS_(c, kRangeGrad, li - 1)));
      }
      if (c->mbits[li - 1]) N2F_TRY(conv_tc_plan_maskbits(&dp, nullptr, 1));
      N2F_TRY(wgrad_tc_plan(&c->wgrad_plan[sc][li], act_op(li - 1), g_op(ab), h, w, kCin[li],
                            kCout[li], c->wsplit[sc][li]));
    }
  }
  for (int li = 1; li < 8; ++li) {
    const int ab = (li & 1) ? 0 : 1;  // L1 writes vA; layer li reads vA when li is odd
    ConvTcPlan& vp = c->val_plan[li];
    N2F_TRY(conv_tc_plan(&vp, v_op(ab), w_op(li), c->H, c->W, kCin[li], kCout[li]));
    if (li == 7) {
      N2F_TRY(conv_tc_plan_out(&vp, nullptr, nullptr, nullptr, sa));  // fused head
    } else {
      N2F_TRY(conv_tc_plan_out(&vp, nullptr, c->v16[1 - ab][0], c->v16[1 - ab][1], sa));
      N2F_TRY(conv_tc_plan_range(&vp, RS_(c, kRangeValAct, li)));
    }
  }
  // the fused heads write one loss / squared-error partial per tile
  c->nblk_head = max_tiles;
  c->nblk_val = c->val_plan[7].tiles;
  N2F_TRY(dalloc(c, &c->part_loss, 4 * (int64_t)c->nblk_head));
  N2F_TRY(dalloc(c, &c->part_se, c->nblk_val));
  // a shape class with fewer tiles leaves its tail of the loss partials at 0
  N2F_CUDA(cudaMemset(c->part_loss, 0, 4 * (size_t)c->nblk_head * sizeof(double)));
  N2F_TRY(dalloc(c, &c->dstate, 1));
  N2F_TRY(dalloc(c, &c->step_counter, 1));
  N2F_TRY(dalloc(c, &c->val_hist, c->cfg.max_epochs));
  N2F_TRY(dalloc(c, &c->loss_hist, 4 * (int64_t)c->cfg.max_epochs));
  N2F_TRY(dalloc(c, &c->time_hist, c->cfg.max_epochs));
  N2F_TRY(dalloc(c, &c->out_stage, c->Pv));

  // Adam bias-correction table: fl32(1 - beta^t) with Python's pow semantics;
  // beyond ~17.3k steps both saturate to 1.0f, so the table is capped.
  int64_t steps = 4 * (int64_t)c->cfg.max_epochs;
  c->table_len = (int)(steps < 32768 ? steps : 32768);
  std::vector<float> t1(c->table_len), t2(c->table_len);
  for (int t = 1; t <= c->table_len; ++t) {
    t1[t - 1] = (float)(1.0 - pow(0.9, (double)t));
    t2[t - 1] = (float)(1.0 - pow(0.999, (double)t));
  }
  if (steps > c->table_len && (t1.back() != 1.0f || t2.back() != 1.0f))
    return fail(N2F_ERR_ARG, "bias-correction table did not saturate");
  N2F_TRY(dalloc(c, &c->bc1, c->table_len));
  N2F_TRY(dalloc(c, &c->bc2, c->table_len));
  N2F_CUDA(cudaMemcpy(c->bc1, t1.data(), t1.size() * 4, cudaMemcpyHostToDevice));
  N2F_CUDA(cudaMemcpy(c->bc2, t2.data(), t2.size() * 4, cudaMemcpyHostToDevice));

  AdamArgs a{};
  a.ntensors = 2 * kLayers;
  a.total = c->ptotal;
  a.p = c->params;
  a.m = c->m;
  a.v = c->v;
  a.bc1 = c->bc1;
  a.bc2 = c->bc2;
  a.table_len = c->table_len;
  a.beta1 = 0.9f;
  a.one_minus_beta1 = (float)(1.0 - 0.9);
  a.beta2 = 0.999f;
  a.one_minus_beta2 = (float)(1.0 - 0.999);
  a.lr = (float)c->cfg.lr;
  a.eps = 1e-8f;
  a.phi16 = c->w16[0];
  a.plo16 = c->w16[1];
  a.wscale = ldexpf(1.f, kExpW);
  for (int li = 0; li < kLayers; ++li) {
    for (int q = 0; q < 2; ++q) {
      AdamTensor& T = a.t[2 * li + q];
      T.off = c->poff[2 * li + q];
      T.n = c->pnum[2 * li + q];
      T.part = q == 0 ? c->part_w[li] : c->part_b[li];
      T.wt = nullptr;
      T.cin = kCin[li];
      T.cout = kCout[li];
    }
  }
  // tcgen05 weights (layers 1..7): Adam also writes their forward fp16 pairs
  // from the same registers; the dgrad-transposed pairs follow in one tiled
  // transpose launch (coalesced, instead of 2-byte scattered stores)
  for (int li = 1; li < 8; ++li) {
    AdamTensor& T = a.t[2 * li];
    T.want16 = 1;
    T.amax = RS_(c, kRangeWeight, li);
    T.wth16 = nullptr;
    T.wtl16 = nullptr;
  }
  {
    TransposePairs& tp = c->tpose;
    tp.whi = c->w16[0];
    tp.wlo = c->w16[1];
    int tiles = 0;
    for (int li = 1; li < 8; ++li) {
      tp.thi[li] = c->wt16[0][li];
      tp.tlo[li] = c->wt16[1][li];
      tp.off[li] = c->poff[2 * li];
      tp.cin[li] = kCin[li];
      tp.cout[li] = kCout[li];
      tp.tile0[li] = tiles;
      tiles += 9 * ((kCin[li] + 31) / 32) * ((kCout[li] + 31) / 32);
    }
    tp.tile0[8] = tiles;
  }
  // split counts per shape class: bias gradients of layers 1..7 are per-tile
  // column sums (dgrad epilogue of the layer above; L8's from the head), the
  // head's partials come from the fused L8 epilogue
  for (int sc = 0; sc < 2; ++sc) {
    AdamArgs& as = c->adam_sc[sc];
    as = a;
    as.t[0].nsplit = as.t[1].nsplit = c->nsplit0;
    for (int li = 1; li <= 7; ++li) {
      as.t[2 * li].nsplit = c->wsplit[sc][li];
      as.t[2 * li + 1].nsplit = li == 7 ? c->fwd_plan[sc][7].tiles : c->dgrad_plan[sc][li + 1].tiles;
    }
    as.t[16].nsplit = 4 * c->fwd_plan[sc][7].tiles;
    as.t[17].nsplit = c->fwd_plan[sc][7].tiles;
    N2F_TRY(plan_adam(c, as));
  }

  N2F_CUDA(cudaMallocHost(&c->h_mm, 4 * sizeof(double)));
  N2F_CUDA(cudaMallocHost(&c->h_state, sizeof(DevState)));
  if (c->cfg.use_graph) N2F_TRY(build_graph(c));
  return N2F_OK;
}

// minmax + checks; returns N2F_OK and sets *degenerate
int prepare_input(n2f_ctx* c, const void* image, int dtype, const void* clean, int* degenerate) {
  cudaStream_t st = c->stream;
  N2F_TRY(launch_minmax(image, dtype, c->Pv, c->mm_part, c->mm, st));
  N2F_CUDA(cudaMemcpyAsync(c->h_mm, c->mm, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  N2F_CUDA(cudaStreamSynchronize(st));
  if (c->h_mm[2] != 0.0) return fail(N2F_ERR_NONFINITE, "image contains non-finite values");
  *degenerate = c->h_mm[0] == c->h_mm[1];
  if (*degenerate) return N2F_OK;
  N2F_TRY(launch_pairs(image, dtype, clean, c->mm, c->H, c->W, c->cfg.scheme, c->cfg.loss == 0,
                       c->norm, c->pin, c->ptgt, c->plane, st));
  return N2F_OK;
}

// Derived operand copies of the weights (dgrad-transposed fp32 copy and the
// fp16 pairs of both layouts).  Adam keeps them current after every step;
// this refreshes them after init / set_params, and resets the range slots so
// the first epoch's record starts with these weights.
int refresh_derived(n2f_ctx* c) {
  N2F_CUDA(cudaMemsetAsync(c->range_cur, 0, kRangeSlots * sizeof(unsigned), c->stream));
  for (int li = 1; li < 8; ++li) {
    const int64_t o = c->poff[2 * li], n = c->pnum[2 * li];
    unsigned* slot = RS_(c, kRangeWeight, li);
    N2F_TRY(transpose_dgrad_weights(c->params + o, c->wt[li], kCin[li], kCout[li], c->stream));
    N2F_TRY(split_f16(c->params + o, c->w16[0] + o, c->w16[1] + o, kExpW, n, c->stream, slot));
    N2F_TRY(split_f16(c->wt[li], c->wt16[0][li], c->wt16[1][li], kExpW, n, c->stream, slot));
  }
  return N2F_OK;
}

int init_network(n2f_ctx* c) {
  cudaStream_t st = c->stream;
  for (int li = 0; li < kLayers; ++li)
    N2F_TRY(launch_init_layer(c->cfg.seed, li, kCin[li], kCout[li], kKsz[li],
                              c->params + c->poff[2 * li], st));
  for (int li = 0; li < kLayers; ++li)
    N2F_CUDA(cudaMemsetAsync(c->params + c->poff[2 * li + 1], 0, c->pnum[2 * li + 1] * 4, st));
  N2F_TRY(refresh_derived(c));
  N2F_CUDA(cudaMemsetAsync(c->m, 0, c->ptotal * 4, st));
  N2F_CUDA(cudaMemsetAsync(c->v, 0, c->ptotal * 4, st));
  N2F_CUDA(cudaMemsetAsync(c->step_counter, 0, sizeof(int), st));
  N2F_TRY(launch_reset_state(c->dstate, st));
  return N2F_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
namespace {

__global__ void k_to_f64(const void* __restrict__ src, int dtype, int64_t n, double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = dtype == N2F_F64 ? reinterpret_cast<const double*>(src)[i]
                              : (double)reinterpret_cast<const float*>(src)[i];
}

size_t dtype_size(int dtype) { return dtype == N2F_F64 ? 8 : 4; }

int check_cfg(const n2f_config* cfg) {
  if (!cfg) return fail(N2F_ERR_ARG, "null config");
  if (cfg->loss != 0 && cfg->loss != 1) return fail(N2F_ERR_ARG, "loss must be bce(0) or mse(1)");
  if (cfg->scheme < 0 || cfg->scheme > 2) return fail(N2F_ERR_ARG, "scheme must be 0..2");
  if (!(cfg->lr > 0)) return fail(N2F_ERR_ARG, "lr must be > 0");
  if (cfg->patience_epochs < 1) return fail(N2F_ERR_ARG, "patience_epochs must be >= 1");
  if (cfg->avg_window < 1) return fail(N2F_ERR_ARG, "avg_window must be >= 1");
  if (cfg->max_epochs < 1) return fail(N2F_ERR_ARG, "max_epochs must be >= 1");
  return N2F_OK;
}

const char* range_class_name(int cls) {
  switch (cls) {
    case kRangeAct: return "training activation";
    case kRangeValAct: return "validation activation";
    case kRangeGrad: return "gradient";
    default: return "weight";
  }
}

// The fit stopped on the range guard (k_stop): N2F_ERR_RANGE naming the slot.
int range_error(const n2f_ctx* c, const DevState& s) {
  if (s.range_slot < 0)
    return fail(N2F_ERR_RANGE, "non-finite validation score %g at epoch %d (FP16x3 range guard)",
                (double)s.range_val, s.epoch);
  return fail(N2F_ERR_RANGE,
              "FP16x3 range guard: %s of layer %d reached max |x * 2^e| = %g (limit %g) at epoch %d; "
              "the fp16 operand split would overflow",
              range_class_name(s.range_slot / kLayers), s.range_slot % kLayers + 1,
              (double)s.range_val, (double)kRangeLimit, s.epoch);
}

int run_loop(n2f_ctx* c) {
  if (c->cfg.use_graph) {
    N2F_CUDA(cudaGraphLaunch(c->exec, c->stream));
    return N2F_OK;
  }
  for (int e = 0; e < c->cfg.max_epochs; ++e) {
    N2F_TRY(enqueue_epoch(c, 0));
    N2F_CUDA(cudaMemcpyAsync(c->h_state, c->dstate, sizeof(DevState), cudaMemcpyDeviceToHost,
                             c->stream));
    N2F_CUDA(cudaStreamSynchronize(c->stream));
    if (c->h_state->stopped) break;
  }
  return N2F_OK;
}

}  // namespace

extern "C" {

const char* n2f_last_error(void) {
  return error_text().c_str();
}

const char* n2f_version(void) { return "n2f-b200 0.1 (sm_100a)"; }

int n2f_create(int device, int height, int width, const n2f_config* cfg, n2f_ctx** out) {
  if (!out) return fail(N2F_ERR_ARG, "null out");
  *out = nullptr;
  N2F_TRY(check_cfg(cfg));
  if (height < 4 || width < 4)
    return fail(N2F_ERR_ARG, "image must be at least 4x4, got (%d, %d)", height, width);
  if (cfg->conv_impl != kImplAuto && cfg->conv_impl != kImplTcF16)
    return fail(N2F_ERR_UNSUPPORTED,
                "conv_impl %d: this library implements only tcgen05 FP16x3 (0 = auto, 3)",
                cfg->conv_impl);
  n2f_ctx* c = new n2f_ctx();
  c->device = device;
  c->H = height;
  c->W = width;
  c->cfg = *cfg;
  int s = setup(c);
  if (s != N2F_OK) {
    n2f_destroy(c);
    return s;
  }
  *out = c;
  return N2F_OK;
}

int n2f_destroy(n2f_ctx* c) {
  if (!c) return N2F_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->exec) cudaGraphExecDestroy(c->exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  for (void* p : c->allocs) cudaFree(p);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->h_mm) cudaFreeHost(c->h_mm);
  if (c->h_state) cudaFreeHost(c->h_state);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return N2F_OK;
}

void* n2f_ctx_stream(n2f_ctx* c) { return c ? (void*)c->stream : nullptr; }
size_t n2f_ctx_device_bytes(n2f_ctx* c) { return c ? c->bytes : 0; }

int n2f_fit_denoise_dev(n2f_ctx* c, const void* image, int dtype, const void* clean, double* out,
                        n2f_result* res) {
  if (!c || !image || !out || !res) return fail(N2F_ERR_ARG, "null argument");
  if (dtype != N2F_F32 && dtype != N2F_F64) return fail(N2F_ERR_ARG, "dtype");
  if (c->cfg.scheme == 2 && !clean)
    return fail(N2F_ERR_ARG, "the exact scheme requires the clean ground-truth image");
  N2F_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  N2F_CUDA(cudaEventRecord(c->ev0, st));
  const int64_t launches0 = g_launches;
  int degenerate = 0;
  N2F_TRY(prepare_input(c, image, dtype, clean, &degenerate));
  res->vmin = c->h_mm[0];
  res->vmax = c->h_mm[1];
  if (degenerate) {
    k_to_f64<<<256, 256, 0, st>>>(image, dtype, c->Pv, out);
    N2F_LAUNCH_CHECK();
    N2F_CUDA(cudaEventRecord(c->ev1, st));
    N2F_CUDA(cudaStreamSynchronize(st));
    res->epochs_run = 0;
    res->stop_reason = N2F_STOP_DEGENERATE;
    res->best_score = INFINITY;
    res->kernel_launches = g_launches - launches0;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    res->gpu_ms = ms;
    return N2F_OK;
  }
  N2F_TRY(init_network(c));
  N2F_TRY(run_loop(c));
  N2F_TRY(launch_window_mean(c->ring, c->Pv, c->cfg.avg_window, c->dstate, 0, 0, c->mm, 0, 0, out,
                             st));
  N2F_CUDA(cudaEventRecord(c->ev1, st));
  N2F_CUDA(cudaMemcpyAsync(c->h_state, c->dstate, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  N2F_CUDA(cudaStreamSynchronize(st));
  const int ne = c->h_state->epoch;
  res->epochs_run = ne;
  res->kernel_launches =
      g_launches - launches0 + (c->cfg.use_graph ? (int64_t)ne * c->epoch_launches : 0);
  res->stop_reason = c->h_state->stop_reason;
  res->best_score = c->h_state->best;
  if (res->val_history)
    N2F_CUDA(cudaMemcpy(res->val_history, c->val_hist, ne * sizeof(double), cudaMemcpyDeviceToHost));
  if (res->train_loss)
    N2F_CUDA(cudaMemcpy(res->train_loss, c->loss_hist, 4 * ne * sizeof(double),
                        cudaMemcpyDeviceToHost));
  if (res->epoch_seconds && ne > 0) {
    std::vector<unsigned long long> t(ne);
    N2F_CUDA(cudaMemcpy(t.data(), c->time_hist, ne * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost));
    for (int e = 0; e < ne; ++e) res->epoch_seconds[e] = 1e-9 * (double)(t[e] - c->h_state->t0);
  }
  float ms = 0.f;
  N2F_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  res->gpu_ms = ms;
  if (c->h_state->stop_reason == N2F_STOP_RANGE) return range_error(c, *c->h_state);
  return N2F_OK;
}

int n2f_fit_denoise_host(n2f_ctx* c, const void* image, int dtype, const void* clean, double* out,
                         n2f_result* res) {
  if (!c || !image || !out || !res) return fail(N2F_ERR_ARG, "null argument");
  if (dtype != N2F_F32 && dtype != N2F_F64) return fail(N2F_ERR_ARG, "dtype");
  N2F_CUDA(cudaSetDevice(c->device));
  const size_t nb = c->Pv * dtype_size(dtype);
  N2F_CUDA(cudaMemcpyAsync(c->img, image, nb, cudaMemcpyHostToDevice, c->stream));
  const void* dclean = nullptr;
  if (clean) {
    if (!c->clean) return fail(N2F_ERR_ARG, "clean image given but scheme is not exact");
    N2F_CUDA(cudaMemcpyAsync(c->clean, clean, nb, cudaMemcpyHostToDevice, c->stream));
    dclean = c->clean;
  }
  N2F_TRY(n2f_fit_denoise_dev(c, c->img, dtype, dclean, c->out_stage, res));
  N2F_CUDA(cudaMemcpyAsync(out, c->out_stage, c->Pv * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  return N2F_OK;
}

// ---- step-level debug/parity entry points ----------------------------------
int n2f_ctx_prepare(n2f_ctx* c, const void* image, int dtype, const void* clean, int init_from_seed) {
  if (!c || !image) return fail(N2F_ERR_ARG, "null argument");
  N2F_CUDA(cudaSetDevice(c->device));
  const size_t nb = c->Pv * dtype_size(dtype);
  N2F_CUDA(cudaMemcpy(c->img, image, nb, cudaMemcpyHostToDevice));
  const void* dclean = nullptr;
  if (clean && c->clean) {
    N2F_CUDA(cudaMemcpy(c->clean, clean, nb, cudaMemcpyHostToDevice));
    dclean = c->clean;
  }
  int degenerate = 0;
  N2F_TRY(prepare_input(c, c->img, dtype, dclean, &degenerate));
  if (degenerate) return fail(N2F_ERR_ARG, "degenerate image");
  if (init_from_seed) N2F_TRY(init_network(c));
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  return N2F_OK;
}

int n2f_ctx_param_count(n2f_ctx* c, int64_t* n) {
  if (!c || !n) return fail(N2F_ERR_ARG, "null argument");
  *n = c->ptotal;
  return N2F_OK;
}

// which: 0 = params, 1 = adam m, 2 = adam v, 3 = gradients of the last step
int n2f_ctx_get_arena(n2f_ctx* c, int which, float* host) {
  if (!c || !host) return fail(N2F_ERR_ARG, "null argument");
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  if (which <= 2) {
    const float* src = which == 0 ? c->params : which == 1 ? c->m : c->v;
    N2F_CUDA(cudaMemcpy(host, src, c->ptotal * 4, cudaMemcpyDeviceToHost));
    return N2F_OK;
  }
  float* tmp = nullptr;
  N2F_CUDA(cudaMalloc(&tmp, c->ptotal * 4));
  const AdamArgs& args = c->adam_sc[c->last_sc];
  for (int q = 0; q < 2 * kLayers; ++q) {
    const AdamTensor& T = args.t[q];
    int s = reduce_partials(T.part, tmp + T.off, T.nsplit, T.n, c->stream);
    if (s != N2F_OK) {
      cudaFree(tmp);
      return s;
    }
  }
  cudaError_t e = cudaMemcpyAsync(host, tmp, c->ptotal * 4, cudaMemcpyDeviceToHost, c->stream);
  cudaStreamSynchronize(c->stream);
  cudaFree(tmp);
  N2F_CUDA(e);
  return N2F_OK;
}

// Network seed for the next fit's initialisation (model.py:46-65): the only
// per-image setting that is not baked into the workspaces or the captured
// graph, so one context serves every seed (denoise_image, CLI per-file seeds).
int n2f_ctx_set_seed(n2f_ctx* c, uint64_t seed) {
  if (!c) return fail(N2F_ERR_ARG, "null ctx");
  c->cfg.seed = seed;
  return N2F_OK;
}

// Overwrite params (engine layout) and reset Adam moments/step and stop state.
int n2f_ctx_set_params(n2f_ctx* c, const float* host) {
  if (!c || !host) return fail(N2F_ERR_ARG, "null argument");
  N2F_CUDA(cudaMemcpy(c->params, host, c->ptotal * 4, cudaMemcpyHostToDevice));
  N2F_TRY(refresh_derived(c));
  N2F_CUDA(cudaMemsetAsync(c->m, 0, c->ptotal * 4, c->stream));
  N2F_CUDA(cudaMemsetAsync(c->v, 0, c->ptotal * 4, c->stream));
  N2F_CUDA(cudaMemsetAsync(c->step_counter, 0, sizeof(int), c->stream));
  N2F_TRY(launch_reset_state(c->dstate, c->stream));
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  return N2F_OK;
}

// Overwrite one arena (0 params, 1 Adam m, 2 Adam v) and the Adam step count
// (t of the NEXT step is step+1), leaving everything else untouched.
int n2f_ctx_set_arena(n2f_ctx* c, int which, const float* host, int step) {
  if (!c || which < 0 || which > 2) return fail(N2F_ERR_ARG, "bad argument");
  if (host) {
    float* dst = which == 0 ? c->params : which == 1 ? c->m : c->v;
    N2F_CUDA(cudaMemcpy(dst, host, c->ptotal * 4, cudaMemcpyHostToDevice));
    if (which == 0) N2F_TRY(refresh_derived(c));
  }
  if (step >= 0) N2F_CUDA(cudaMemcpy(c->step_counter, &step, sizeof(int), cudaMemcpyHostToDevice));
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  return N2F_OK;
}

int n2f_ctx_step(n2f_ctx* c, int pair, float* logits_host) {
  if (!c || pair < 0 || pair > 3) return fail(N2F_ERR_ARG, "bad pair");
  N2F_TRY(enqueue_step(c, pair));
  if (logits_host)
    N2F_CUDA(cudaMemcpyAsync(logits_host, c->z, c->Pt * 4, cudaMemcpyDeviceToHost, c->stream));
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  return N2F_OK;
}

// One epoch with CUDA events around every launch (host loop, same stream):
// per (kernel class, layer) total device ms, algorithmic FLOPs and launch
// counts, arrays of N2F_PROF_CLASSES x 9.  Continues the current training.
int n2f_ctx_profile_epoch(n2f_ctx* c, double* ms, double* flop, int* launches) {
  if (!c || !ms || !flop || !launches) return fail(N2F_ERR_ARG, "null argument");
  c->marks.clear();
  c->ev_used = 0;
  c->prof = true;
  int s = enqueue_epoch(c, 0);
  c->prof = false;
  if (s != N2F_OK) return s;
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < kPClasses * kLayers; ++i) {
    ms[i] = 0.0;
    flop[i] = 0.0;
    launches[i] = 0;
  }
  for (const auto& m : c->marks) {
    float t = 0.f;
    N2F_CUDA(cudaEventElapsedTime(&t, m.a, m.b));
    const int i = m.cls * kLayers + m.li;
    ms[i] += t;
    flop[i] += m.flop;
    launches[i] += 1;
  }
  return N2F_OK;
}

int n2f_ctx_epoch(n2f_ctx* c, int* stopped) {
  if (!c) return fail(N2F_ERR_ARG, "null ctx");
  N2F_TRY(enqueue_epoch(c, 0));
  N2F_CUDA(cudaMemcpyAsync(c->h_state, c->dstate, sizeof(DevState), cudaMemcpyDeviceToHost,
                           c->stream));
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  if (stopped) *stopped = c->h_state->stopped;
  if (c->h_state->stop_reason == N2F_STOP_RANGE) return range_error(c, *c->h_state);
  return N2F_OK;
}

// Guard bytes around every context allocation still hold their pattern (no
// kernel wrote past either end of a buffer); *n_bad = corrupted guards.
int n2f_ctx_check_guards(n2f_ctx* c, int* n_bad) {
  if (!c || !n_bad) return fail(N2F_ERR_ARG, "bad argument");
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<uint8_t> h(kGuardBytes);
  int bad = 0;
  for (size_t i = 0; i < c->allocs.size(); ++i) {
    const uint8_t* base = reinterpret_cast<const uint8_t*>(c->allocs[i]);
    for (int side = 0; side < 2; ++side) {
      const uint8_t* g = side ? base + kGuardBytes + c->alloc_bytes[i] : base;
      N2F_CUDA(cudaMemcpy(h.data(), g, kGuardBytes, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < kGuardBytes; ++k)
        if (h[k] != (uint8_t)kGuardByte) {
          ++bad;
          break;
        }
    }
  }
  *n_bad = bad;
  return N2F_OK;
}

// Per-epoch range-guard maxima of the epochs run since the last reset
// (init / set_params): [n][N2F_RANGE_SLOTS] floats.
int n2f_ctx_range_history(n2f_ctx* c, float* host, int max_rows, int* n_rows) {
  if (!c || !host || max_rows < 0 || !n_rows) return fail(N2F_ERR_ARG, "bad argument");
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  DevState s;
  N2F_CUDA(cudaMemcpy(&s, c->dstate, sizeof s, cudaMemcpyDeviceToHost));
  const int n = s.epoch < max_rows ? s.epoch : max_rows;
  if (n > 0)
    N2F_CUDA(cudaMemcpy(host, c->range_hist, (size_t)n * kRangeSlots * sizeof(float),
                        cudaMemcpyDeviceToHost));
  *n_rows = n;
  return N2F_OK;
}

// Validation output of the current net (slot of the current epoch) + score.
int n2f_ctx_validate(n2f_ctx* c, float* out_host, double* score) {
  if (!c) return fail(N2F_ERR_ARG, "null ctx");
  N2F_TRY(enqueue_validate(c));
  N2F_CUDA(cudaMemcpyAsync(c->h_state, c->dstate, sizeof(DevState), cudaMemcpyDeviceToHost,
                           c->stream));
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  const int slot = c->h_state->epoch % c->cfg.avg_window;
  if (out_host)
    N2F_CUDA(cudaMemcpy(out_host, c->ring + (int64_t)slot * c->Pv, c->Pv * 4,
                        cudaMemcpyDeviceToHost));
  if (score) {
    std::vector<double> p(c->nblk_val);
    N2F_CUDA(cudaMemcpy(p.data(), c->part_se, p.size() * 8, cudaMemcpyDeviceToHost));
    double s = 0.0;
    for (double q : p) s += q;
    *score = s / (double)c->Pv;
  }
  return N2F_OK;
}

// Training planes (4 inputs then 4 targets) and the f32 normalised image.
int n2f_ctx_get_pairs(n2f_ctx* c, float* pin, float* ptgt, float* norm, int* ph, int* pw) {
  if (!c) return fail(N2F_ERR_ARG, "null ctx");
  N2F_CUDA(cudaStreamSynchronize(c->stream));
  if (pin) N2F_CUDA(cudaMemcpy(pin, c->pin, 4 * c->plane * 4, cudaMemcpyDeviceToHost));
  if (ptgt) N2F_CUDA(cudaMemcpy(ptgt, c->ptgt, 4 * c->plane * 4, cudaMemcpyDeviceToHost));
  if (norm) N2F_CUDA(cudaMemcpy(norm, c->norm, c->Pv * 4, cudaMemcpyDeviceToHost));
  for (int k = 0; k < 4; ++k) {
    if (ph) ph[k] = c->ph[k];
    if (pw) pw[k] = c->pw[k];
  }
  return N2F_OK;
}

}  // extern "C"
