// Device loss math shared by the standalone head kernels (train.cu) and the
// heads fused into the last convolution's epilogue (conv_tc.cu).
#pragma once
#include <cuda_runtime.h>

namespace n2f {

// Two-branch logistic (tensor.py:153-161), IEEE division.
__device__ __forceinline__ float sigmoid_ref(float z) {
  if (z >= 0.f) return __fdiv_rn(1.f, __fadd_rn(1.f, expf(-z)));
  const float e = expf(z);
  return __fdiv_rn(e, __fadd_rn(1.f, e));
}

// dloss/dz and the per-element loss for the two training losses
// (tensor.py:164-193, trainer.py:112-117).
__device__ __forceinline__ float loss_grad(float z, float t, int loss, float inv_n_num,
                                           float two_over_n, float* elem) {
  const float s = sigmoid_ref(z);
  if (loss == 0) {
    *elem = __fadd_rn(__fsub_rn(fmaxf(z, 0.f), __fmul_rn(z, t)), log1pf(expf(-fabsf(z))));
    return __fdiv_rn(__fsub_rn(s, t), inv_n_num);  // (sigmoid(z) - t) / N
  }
  const float d = __fsub_rn(s, t);
  *elem = __fmul_rn(d, d);
  const float gs = __fmul_rn(two_over_n, d);              // (2/N) * diff
  return __fmul_rn(__fmul_rn(gs, s), __fsub_rn(1.f, s));  // grad_s * s * (1 - s)
}

// Validation output clip (model.py:136-140): [nextafter(0,1), nextafter(1,0)].
__device__ __forceinline__ float clip_unit(float s) {
  return fminf(fmaxf(s, __int_as_float(1)), __int_as_float(0x3f7fffff));
}

}  // namespace n2f
