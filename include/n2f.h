/*
 * n2f.h -- C ABI of the B200-native Noise2Fast fit-and-denoise engine (libn2f.so).
 *
 * This is the drop-in boundary for the reference's per-image hot path
 * `noise2fast.trainer.train_single_channel` (reference
 * pkg/src/noise2fast/trainer.py:125-213).  The reference is pure Python, so
 * its "FFI" is the Python call itself; the Python mirror in
 * paper_2108_10209_b200/trainer.py binds these symbols with ctypes and keeps
 * the reference's signature, errors and return type.
 *
 * Conventions: plain pointers and sizes only; every function returns an
 * n2f_status (0 == OK) and n2f_last_error() gives the message.  One context
 * per (process, device, image shape, config); contexts are not thread-safe
 * (the reference is single-threaded per run).
 * `stream` arguments are cudaStream_t passed as void* (NULL = context stream).
 */
#ifndef N2F_H
#define N2F_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum n2f_status {
  N2F_OK = 0,
  N2F_ERR_ARG = 1,        /* bad argument (maps to ValueError)            */
  N2F_ERR_NONFINITE = 2,  /* image contains NaN/Inf (trainer.py:142-143)  */
  N2F_ERR_CUDA = 3,       /* CUDA runtime/driver failure                   */
  N2F_ERR_OOM = 4,        /* device allocation failed                      */
  N2F_ERR_UNSUPPORTED = 5, /* config value not implemented                 */
  N2F_ERR_RANGE = 6        /* an FP16x3 operand left fp16's range (see the
                              range guard below); the fit was stopped      */
} n2f_status;

/* TrainConfig (trainer.py:29-51). loss: 0 = "bce", 1 = "mse";
 * scheme: 0 = "checkerboard", 1 = "quad", 2 = "exact". */
typedef struct n2f_config {
  int32_t loss;
  int32_t scheme;
  double lr;
  int32_t patience_epochs;
  int32_t avg_window;
  int32_t max_epochs;
  int32_t conv_impl;      /* 0 = auto (= 3) or 3 = tcgen05 FP16x3, the only implementation;
                             any other value is N2F_ERR_UNSUPPORTED */
  uint64_t seed;
  int32_t use_graph;      /* 1 = whole loop in one CUDA graph (while node), 0 = host loop */
  int32_t reserved[7];
} n2f_config;

/* stop_reason codes (trainer.py:74) */
enum { N2F_STOP_PATIENCE = 0, N2F_STOP_MAX_EPOCHS = 1, N2F_STOP_DEGENERATE = 2,
       N2F_STOP_RANGE = 3 /* internal: the fit returns N2F_ERR_RANGE */ };

/* Per-image outcome (DenoiseResult, trainer.py:69-75).  The optional history
 * buffers are HOST arrays supplied by the caller, each sized for max_epochs
 * entries (train_loss: 4 per epoch); they may be NULL. */
typedef struct n2f_result {
  int32_t epochs_run;
  int32_t stop_reason;
  double vmin, vmax;          /* NormParams of the input                       */
  double best_score;
  double* val_history;        /* [max_epochs]     f64 validation MSE           */
  double* train_loss;         /* [4*max_epochs]   per-pair training loss       */
  double* epoch_seconds;      /* [max_epochs]     device time since start (s)  */
  double gpu_ms;              /* device time of the whole fit (CUDA events)    */
  int64_t kernel_launches;    /* libn2f kernels executed by the fit            */
} n2f_result;

typedef struct n2f_ctx n2f_ctx;

/* dtype codes for image buffers */
enum { N2F_F32 = 0, N2F_F64 = 1 };

const char* n2f_last_error(void);
const char* n2f_version(void);

/* ---- context lifecycle (workspaces sized once per H x W; no allocation in the loop) */
int n2f_create(int device, int height, int width, const n2f_config* cfg, n2f_ctx** out);
int n2f_destroy(n2f_ctx* ctx);
void* n2f_ctx_stream(n2f_ctx* ctx);
size_t n2f_ctx_device_bytes(n2f_ctx* ctx);

/* ---- whole fit-and-denoise (trainer.train_single_channel) ------------------
 * image: H*W samples (dtype N2F_F32/N2F_F64), row-major.  out: H*W f64, the
 * denoised image on the input's value scale (or the input itself, copied, for
 * a degenerate constant image).  clean: only for scheme "exact" (same dtype).
 * *_dev variants take device pointers; *_host variants take host pointers and
 * include the host<->device copies. */
int n2f_fit_denoise_dev(n2f_ctx* ctx, const void* image, int dtype, const void* clean,
                        double* out, n2f_result* res);
int n2f_fit_denoise_host(n2f_ctx* ctx, const void* image, int dtype, const void* clean,
                         double* out, n2f_result* res);

/* ---- per-kernel entry points used by the parity suite (device pointers) ---- */

/* min/max/nonfinite of an H*W image; out3 (host): {vmin, vmax, n_nonfinite}.
 * (imaging.normalize_plane, imaging.py:190-205) */
int n2f_minmax(const void* image, int dtype, int64_t n, double* out3, void* stream);

/* normalise + training-pair gather (imaging.py:190-205, downsample.py:45-164).
 * norm: H*W f32; pair_in/pair_tgt: 4 planes each of the pair shape, written as
 * 4 consecutive planes of plane_elems; returns each pair's (h,w) in ph/pw. */
int n2f_make_pairs(const void* image, int dtype, const void* clean, int height, int width,
                   double vmin, double vmax, int scheme, int clip_targets, float* norm,
                   float* pair_in, float* pair_tgt, int ph[4], int pw[4], void* stream);

/* He-uniform init of one conv layer in the engine's [cout][ky][kx][cin] layout
 * from the counter stream CounterRng(derive_seed(seed, layer)) (model.py:46-65). */
int n2f_init_layer(uint64_t seed, int layer, int cin, int cout, int k, float* w_kmajor,
                   void* stream);

/* conv forward (+bias, +ReLU when relu != 0), NHWC activations:
 * x [h*w][cin], w [cout][k][k][cin], y [h*w][cout] (tensor.py:490-506).
 * Runs the engine's kernels: 3x3 with cin % 32 == 0 and cout in {32, 64,
 * 128, 256} on the tcgen05 FP16x3 kernel (operands split at the engine's
 * scales), 3x3 with cin == 1 on the first-layer kernel, and 1x1 (the head,
 * fused into the L8 epilogue inside the engine) on a direct kernel; other
 * shapes return N2F_ERR_UNSUPPORTED.  impl: 0 or 3. */
int n2f_conv_fwd(const float* x, const float* w, const float* b, float* y, int h, int wd,
                 int cin, int cout, int k, int relu, int impl, void* stream);

/* conv backward (tensor.py:509-530): g is the gradient at the pre-activation
 * [h*w][cout]; dx [h*w][cin] = conv^T(g) masked by (mask > 0) when mask != NULL;
 * dw [cout][k][k][cin], db [cout].  Any of dx/dw/db may be NULL to skip it.
 * Same kernels and shape rules as n2f_conv_fwd (dgrad: the tcgen05 kernel
 * with cout % 32 == 0 and cin in {32, 64, 128, 256}; dw: tcgen05 wgrad, or
 * the first-layer wgrad for cin == 1 and cout == 32). */
int n2f_conv_bwd(const float* g, const float* x, const float* w, const float* mask, float* dx,
                 float* dw, float* db, int h, int wd, int cin, int cout, int k, int impl,
                 void* stream);

/* loss at the logits (tensor.py:164-193, trainer.py:112-117): grad [n] and
 * mean loss (host double). loss: 0 = bce, 1 = mse-through-sigmoid. */
int n2f_loss(const float* z, const float* t, float* grad, int64_t n, int loss, double* loss_out,
             void* stream);

/* Adam on n fp32 params, step t >= 1 (tensor.py:125-141), bitwise-faithful. */
int n2f_adam(float* p, const float* g, float* m, float* v, int64_t n, int t, double lr,
             void* stream);

/* predict tail: sigmoid + clip to (0,1) open range (model.py:136-140) and f64
 * MSE against norm (trainer.py:97-101). score: host double. */
int n2f_validate_tail(const float* z, const float* norm, float* out, int64_t n, double* score,
                      void* stream);

/* stop rule replay over a score sequence (trainer.py:78-94): returns the
 * 1-based stop epoch in *stop_epoch (or -1). */
int n2f_stop_replay(const double* scores_host, int n, int patience, int* stop_epoch);

/* window mean of n planes (in epoch order, ring[slot]) + f64 denormalise
 * (trainer.py:104-109, imaging.py:208-211).  ring: n_slots*plane f32;
 * first_slot = slot of the oldest plane. */
int n2f_window_mean(const float* ring, int n_slots, int first_slot, int n, int64_t plane,
                    double vmin, double vmax, double* out, void* stream);

/* ---- context-level step/epoch entry points (parity suite) ------------------
 * prepare: HOST image (and clean) -> min/max + normalise + pairs (+ seeded
 * init when init_from_seed).
 * Arena = all 18 parameter tensors in order w0,b0,...,w8,b8; weights in the
 * engine layout [cout][ky][kx][cin].  which: 0 params, 1 Adam m, 2 Adam v,
 * 3 summed gradients of the last step.  set_params resets Adam + stop state. */
int n2f_ctx_prepare(n2f_ctx* ctx, const void* image, int dtype, const void* clean,
                    int init_from_seed);
int n2f_ctx_param_count(n2f_ctx* ctx, int64_t* n);
/* seed of the next fit's He-uniform init (TrainConfig.seed, trainer.py:178) */
int n2f_ctx_set_seed(n2f_ctx* ctx, uint64_t seed);
int n2f_ctx_get_arena(n2f_ctx* ctx, int which, float* host);
int n2f_ctx_set_params(n2f_ctx* ctx, const float* host);
int n2f_ctx_set_arena(n2f_ctx* ctx, int which, const float* host, int adam_step);
int n2f_ctx_step(n2f_ctx* ctx, int pair, float* logits_host);
int n2f_ctx_epoch(n2f_ctx* ctx, int* stopped);
/* Profile one epoch: per (class, layer) device ms / algorithmic FLOPs / launches
 * in arrays of N2F_PROF_CLASSES * 9 (classes: 0 first-layer fwd, 1 conv fwd,
 * 2 head+loss, 3 wgrad, 4 dgrad, 5 first-layer wgrad, 6 Adam, 7 validation
 * first layer, 8 validation conv, 9 validation head, 10 stop rule). */
#define N2F_PROF_CLASSES 11
int n2f_ctx_profile_epoch(n2f_ctx* ctx, double* ms, double* flop, int* launches);
int n2f_ctx_validate(n2f_ctx* ctx, float* out_host, double* score);
int n2f_ctx_get_pairs(n2f_ctx* ctx, float* pair_in, float* pair_tgt, float* norm, int ph[4],
                      int pw[4]);

/* ---- FP16x3 range guard ----------------------------------------------------
 * Every tensor-core operand is an fp16 pair of x * 2^e (activations and
 * weights e = 8, gradients e = ceil(log2 P) + 8).  Each epoch the kernels
 * that write such pairs record max |x * 2^e| per (tensor class, layer) slot:
 * slot = class * 9 + layer, classes 0 training activations (output of
 * layer), 1 validation activations, 2 gradients (at the output of layer),
 * 3 weights.  A slot >= 2^15 (or a non-finite validation score) stops the
 * fit: n2f_fit_denoise_* and n2f_ctx_epoch return N2F_ERR_RANGE naming the
 * slot.  range_history copies the per-epoch maxima of the last fit (or of the
 * epochs run since n2f_ctx_prepare / set_params): [n_epochs][N2F_RANGE_SLOTS]
 * floats (0 = no pair written in that slot), at most max_rows rows. */
#define N2F_RANGE_SLOTS 36
int n2f_ctx_range_history(n2f_ctx* ctx, float* host, int max_rows, int* n_rows);

/* Out-of-bounds write check: every context allocation is bracketed by 256
 * guard bytes of a fixed pattern; *n_bad = guards that no longer hold it. */
int n2f_ctx_check_guards(n2f_ctx* ctx, int* n_bad);

/* ---- image-quality metrics (benchmark mode; imaging.psnr / imaging.ssim,
 * imaging.py:249-311), f64 device buffers of one single-channel plane ------ */
/* sum of (a - b)^2 over n samples (host result) */
int n2f_sq_err_sum(const double* a, const double* b, int64_t n, double* out, void* stream);
/* 10 log10(range^2 / mse), +inf when mse == 0 (imaging.psnr) */
int n2f_psnr(const double* a, const double* b, int64_t n, double data_range, double* out,
             void* stream);
/* mean SSIM, 11x11 Gaussian window (sigma 1.5), fully valid positions only
 * (imaging.ssim); N2F_ERR_ARG below 11x11 or for data_range <= 0 */
int n2f_ssim(const double* a, const double* b, int height, int width, double data_range, double k1,
             double k2, double* out, void* stream);
/* CUDA devices visible to this process (worker -> GPU mapping) */
int n2f_device_count(int* n);

#ifdef __cplusplus
}
#endif
#endif /* N2F_H */
