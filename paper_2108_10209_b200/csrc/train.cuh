// Device-side state and launchers of the training-loop kernels (train.cu).
#pragma once
#include <cuda_fp16.h>

#include "n2f_internal.cuh"

namespace n2f {

// Early-stopping state (trainer.py:54-66), resident on the device.
struct DevState {
  int epoch;        // completed epochs
  int step;         // unused (Adam t lives in its own counter)
  int since;        // epochs since the last strict improvement
  int stopped;
  int stop_reason;
  int best_epoch;
  double best;
  unsigned long long t0;  // %globaltimer at the start of the fit
  int range_slot;         // N2F_STOP_RANGE: class * 9 + layer of the slot over the limit (-1: score)
  float range_val;        //   and its max |x * 2^e| (or the non-finite score)
};

// The 1x1 head (L9) fused into the epilogue of the last 3x3 convolution
// (FP16x3 path): training = logits, loss, dloss/dz, the L8 gradient pair and
// per-tile partials of dW9 / db9 / loss; validation = sigmoid, clip, ring slot
// and per-tile squared-error partials.
struct HeadTrainArgs {
  const float* w9;
  const float* b9;
  const float* tgt;
  float* zout;
  float* part_w9;      // [tiles * 4][256] (one row per 32-pixel warp group)
  float* part_b9;      // [tiles]
  double* part_loss;   // [tiles]
  int* step_counter;   // Adam t, incremented once per step
  int loss;
  float nf, two_over_n;
};
struct HeadValArgs {
  const float* w9;
  const float* b9;
  const float* norm;
  float* ring;
  const DevState* st;
  int window;
  double* part_se;  // [tiles]
};

// L8 forward with the head fused (FP16 dy plan, N = 256; conv_tc.cu).  The
// training variant writes the L8 gradient pair through the plan's outputs and
// the bias gradient of L8 into colsum ([tiles][256]).
int conv_tc_launch_head_train(const ConvTcPlan& pl, const float* bias, float* colsum,
                              const HeadTrainArgs& ht, cudaStream_t st);
int conv_tc_launch_head_val(const ConvTcPlan& pl, const float* bias, const HeadValArgs& hv,
                            cudaStream_t st);

struct Pt4 {
  double v[4];
};

struct AdamTensor {
  int64_t off;        // offset in the parameter arena
  int64_t n;          // elements
  const float* part;  // [nsplit][n] gradient partials
  int nsplit;
  float* wt;          // optional dgrad-transposed copy (3x3 weights), else null
  int want16;         // write the fp16 pair of p * wscale into AdamArgs::phi16/plo16
  unsigned* amax;     // range-guard slot of those pairs (or null)
  __half* wth16;      // optional fp16 pair of the dgrad-transposed copy (scaled)
  __half* wtl16;
  int cin, cout;
  // reduction plan (adam_plan): rl row lanes x cw columns per block, ns row
  // slabs of <= 16 rl partial rows (slab sums combined by the last block of a
  // column chunk through scratch + an arrival counter), blocks [blk0, ...)
  int rl, cw, ns, nchunk, blk0, cnt0;
  int vec;  // 4: float4 columns per thread (one row lane, aligned), else 1
  int cin_log2;  // log2(cin) when cin is a power of two, else -1
  int64_t scr0;
};

constexpr int kMaxTensors = 18;

struct AdamArgs {
  AdamTensor t[kMaxTensors];
  int ntensors;
  int64_t total;
  float* p;
  __half* phi16;  // fp16 pair arenas (same layout as p), for tensors with want16
  __half* plo16;
  float wscale;   // 2^kExpW
  float* m;
  float* v;
  const float* bc1;  // fl32(1 - beta1^t), t = 1..table_len
  const float* bc2;
  int table_len;
  float beta1, one_minus_beta1, beta2, one_minus_beta2, lr, eps;
  int nblocks;         // set by adam_plan
  int64_t scr_total;   // floats of slab scratch the plan needs
  int cnt_total;       // arrival counters the plan needs (zeroed once; self-resetting)
  float* scratch;
  int* counters;
};

// The dgrad-transposed fp16 weight pairs wt[c][8-tap][o] = w[o][tap][c] of
// the tcgen05 layers, rebuilt from the forward pairs after every Adam step
// by one tiled (coalesced) launch over all layers.
struct TransposePairs {
  const __half* whi;  // forward pair arenas (AdamArgs::phi16 / plo16 layout)
  const __half* wlo;
  __half* thi[kLayers];
  __half* tlo[kLayers];
  int64_t off[kLayers];  // weight offset of layer li in the arena
  int cin[kLayers], cout[kLayers];
  int tile0[kLayers + 1];  // first 32 x 32 tile of layer li (layers 1..7), tile0[8] = total
};
int launch_transpose_pairs(const TransposePairs& t, cudaStream_t st);

// Fill the reduction plan of every tensor (needs t[].n / nsplit) and the
// scratch / counter sizes; the caller allocates scratch and zeroed counters.
void adam_plan(AdamArgs& a);

int launch_adam(const AdamArgs& args, const int* step_counter, int fixed_t, cudaStream_t st);
int launch_stop(DevState* dst, const double* part_se, int n_se, double pv, const double* part_loss,
                int n_loss, const double pt[4], double* val_hist, double* loss_hist,
                unsigned long long* time_hist, int patience, int max_epochs, unsigned* range_cur,
                float* range_hist, cudaGraphConditionalHandle handle, int use_handle,
                cudaStream_t st);
int launch_window_mean(const float* ring, int64_t plane, int window, const DevState* dst, int n,
                       int first, const double* mm, double vmin, double vmax, double* out,
                       cudaStream_t st);
int launch_loss(const float* z, const float* t, float* grad, int64_t n, int loss, double* part,
                int nblk, double* sum_out, cudaStream_t st);
int launch_val_tail(const float* z, const float* norm, float* out, int64_t n, double* part, int nblk,
                    double* sum_out, cudaStream_t st);
int launch_reset_state(DevState* dst, cudaStream_t st);

// prep.cu
int launch_minmax(const void* img, int dtype, int64_t n, double* part, double* out3,
                  cudaStream_t st);
size_t minmax_scratch_doubles();
int launch_pairs(const void* img, int dtype, const void* clean, const double* mm, int H, int W,
                 int scheme, int clip, float* norm, float* pin, float* ptgt, int64_t plane,
                 cudaStream_t st);
int launch_init_layer(uint64_t seed, int layer, int cin, int cout, int k, float* w,
                      cudaStream_t st);

}  // namespace n2f
