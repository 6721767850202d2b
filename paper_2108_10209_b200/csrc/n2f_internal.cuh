// Internal declarations shared by the libn2f translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/n2f.h"

namespace n2f {

// ---- error plumbing ---------------------------------------------------------
void set_error(const std::string& msg);
const std::string& error_text();
int fail(int code, const char* fmt, ...);

// On failure the runtime's (non-sticky) last-error slot is cleared too, so a
// failed allocation is not reported again by the next launch check.
#define N2F_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      (void)cudaGetLastError();                                                          \
      return ::n2f::fail(e_ == cudaErrorMemoryAllocation ? N2F_ERR_OOM : N2F_ERR_CUDA,   \
                         "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                         __LINE__);                                                      \
    }                                                                                    \
  } while (0)

#define N2F_TRY(call)            \
  do {                           \
    int s_ = (call);             \
    if (s_ != N2F_OK) return s_; \
  } while (0)

// Every launcher calls this once per kernel it launched (it also counts the
// launches, so the engine can report how many of its kernels a fit ran).
extern thread_local int64_t g_launches;
#define N2F_LAUNCH_CHECK()  \
  do {                      \
    ++::n2f::g_launches;    \
    N2F_CUDA(cudaGetLastError()); \
  } while (0)

// ---- network geometry (reference model.py:20, 36-43) ------------------------
constexpr int kLayers = 9;
constexpr int kCin[kLayers] = {1, 32, 32, 64, 64, 128, 128, 256, 256};
constexpr int kCout[kLayers] = {32, 32, 64, 64, 128, 128, 256, 256, 1};
constexpr int kKsz[kLayers] = {3, 3, 3, 3, 3, 3, 3, 3, 1};
constexpr int kMaxC = 256;

// ---- conv implementation ------------------------------------------------------
// n2f_config::conv_impl: the product library has ONE implementation, tcgen05
// FP16x3 (0 = auto = 3); anything else is N2F_ERR_UNSUPPORTED.
enum ConvImpl { kImplAuto = 0, kImplTcF16 = 3 };
// power-of-two operand scales of the FP16 split (activations, weights);
// gradients use ceil(log2(pixels)) + kExpAct (see engine.cu setup)
constexpr int kExpAct = 8, kExpW = 8;

// ---- FP16x3 range guard (see tc_common.cuh range_note) ----------------------
// One slot per (tensor class, layer) holds max |x * 2^e| (as ordered float
// bits) of every operand pair written during the current epoch; the stop
// kernel moves the slots into a per-epoch history and stops the fit with
// N2F_STOP_RANGE when one reaches kRangeLimit (or is non-finite).
enum RangeClass { kRangeAct = 0, kRangeValAct = 1, kRangeGrad = 2, kRangeWeight = 3, kRangeClasses = 4 };
constexpr int kRangeSlots = kRangeClasses * kLayers;
constexpr float kRangeLimit = 32768.f;  // 2^15: one binade of headroom below fp16's 65504

// Epilogue modes of the 3x3 implicit GEMM.
enum Epi { kEpiBiasRelu = 0, kEpiMask = 1, kEpiBias = 2, kEpiNone = 3 };

// First-layer kernels (first_layer.cu).  conv_first: fp32 output y and/or the
// fp16 pair of y * oscale (yh16/yl16), amax = range slot of that pair.
int conv_first_simt(const float* x, const float* w, const float* b, float* y, int h, int w_,
                    int cout, cudaStream_t st, int relu = 1, void* yh16 = nullptr,
                    void* yl16 = nullptr, float oscale = 1.f, unsigned* amax = nullptr);
int wgrad_first_simt(const float* g, const float* x, float* dw_part, float* db_part, int h, int w,
                     int cout, int nsplit, cudaStream_t st);
int wgrad_first_nsplit(int64_t pixels);

// tcgen05 kernels (conv_tc.cu).  A plan holds the TMA descriptors of one
// (input buffer, weight buffer, shape) combination; it is built once and
// launched many times (graph-capturable: maps are kernel parameters).
// A tensor-core operand: the fp16 pair (hi, lo) of x * 2^exp.
struct TcOperand {
  const void* hi;
  const void* lo;
  int exp;
};
struct ConvTcPlan {
  CUtensorMap mx, mxl, mw, mwl;
  CUtensorMap my, myh, myl;  // outputs (conv_tc_plan_out): fp32, fp16 hi / lo
  int omask;                 // which outputs exist (1 y, 2 hi, 4 lo)
  float oscale;              // FP16 pair = fp16 split of y * oscale
  uint32_t* mbits_out;       // bit-packed ReLU mask of the output ([px][N/32]), or null
  int mask_bits;             // the launch's `mask` is such a bit mask (else fp16 values)
  unsigned* amax;            // range-guard slot of the pair output, or null
  float* y;                  // the same outputs as raw pointers
  void* yhi;
  void* ylo;
  int H, W, C, N, grid;
  float unscale;  // 2^-(exp_x + exp_w)
  int tiles;      // 16 x 8 pixel CTA tiles = rows of the colsum output
};
bool tc_supported(int cin, int cout);
int conv_tc_plan(ConvTcPlan* pl, const TcOperand& x, const TcOperand& w, int H, int W, int C, int N);
// Outputs (bound once per plan): y fp32 (may be null) and/or the fp16 pair of
// y * oscale into yhi/ylo (either may be null).  mask at launch: the fp16 hi
// tensor of the layer input (ReLU mask), or a bit mask (conv_tc_plan_maskbits).
int conv_tc_plan_out(ConvTcPlan* pl, float* y, void* yhi, void* ylo, float oscale);
// Wide layers (N >= 64): the forward can emit its ReLU mask bit-packed, the
// dgrad can consume one (call after conv_tc_plan_out).
int conv_tc_plan_maskbits(ConvTcPlan* pl, uint32_t* mbits_out, int mask_bits_in);
int conv_tc_plan_range(ConvTcPlan* pl, unsigned* amax);
int conv_tc_launch(const ConvTcPlan& pl, const float* bias, const void* mask, float* colsum, int epi,
                   cudaStream_t st);
int conv_tc_tiles(int H, int W);  // ConvTcPlan::tiles of an H x W plan
struct WgradTcPlan {
  CUtensorMap mx, mxl, mg, mgl;
  int H, W, C, N, mblocks, nsplit;
  float unscale;
  int xblk;   // activation blocks of an M block loaded as one 4-D box (C % 128 == 0)
  int cs;     // CTAs per cluster (2: pairs of M blocks, cta_group::2)
  int gridx;  // CTAs along M (mblocks rounded up to a multiple of cs)
  int seg;    // pixels per K stage (32 pairs; 64 or 128 single CTAs)
};
int wgrad_tc_nsplit(int cin, int cout, int H, int W);
int wgrad_tc_plan(WgradTcPlan* pl, const TcOperand& x, const TcOperand& g, int H, int W, int C,
                  int N, int nsplit);
int wgrad_tc_launch(const WgradTcPlan& pl, float* part, cudaStream_t st);
int split_f16(const float* x, void* hi, void* lo, int exp2, int64_t n, cudaStream_t st,
              unsigned* amax = nullptr);

// utility kernels (prep.cu / train.cu)
int reduce_partials(const float* part, float* out, int nsplit, int64_t n, cudaStream_t st);
int transpose_dgrad_weights(const float* w, float* wt, int cin, int cout, cudaStream_t st);

double wall_seconds();

}  // namespace n2f
