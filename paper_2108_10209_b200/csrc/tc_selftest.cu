// tcgen05 self-test (n2f_tc_selftest): D[128 x N] = A[128 x 32] . B[N x 32]^T
// with operands staged by threads in the canonical UMMA layouts, four
// kind::tf32 MMAs (K = 8 each), read back with tcgen05.ld.  It pins the
// descriptor encodings (K-major SWIZZLE_128B, MN-major SWIZZLE_128B_BASE32B)
// and shows how the tensor core converts fp32 inputs (it truncates to tf32).
#include "n2f_internal.cuh"
#include "tc_common.cuh"

namespace n2f {
namespace {

using namespace tc;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// operand modes: 0 = K-major SW128, 1 = MN-major SW128, 2 = MN-major SW128_BASE32B
__device__ __forceinline__ uint32_t operand_offset(int mode, int row, int k) {
  if (mode == 0) return sw128_offset(row, 4 * k);
  if (mode == 1) return (row / 32) * 4096 + sw128_offset(k, 4 * (row % 32));
  return (row / 32) * 4096 + sw128b32_offset(k, 4 * (row % 32));
}
__device__ __forceinline__ uint64_t operand_desc(int mode, uint32_t base, int s) {
  if (mode == 0) return sw128_desc(base + s * 32, 16, 1024);
  if (mode == 1) return sw128_desc(base + s * 1024, 4096, 1024);
  return sw128_desc(base + s * 1024, 4096, 512, kLayoutSw128Base32);
}

template <int AM, int BM>
__global__ void __launch_bounds__(128) k_tc_selftest(const float* __restrict__ A,
                                                     const float* __restrict__ B,
                                                     float* __restrict__ D, int N) {
  constexpr bool A_MN = AM != 0, B_MN = BM != 0;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* base = align1024(smem_raw);
  uint8_t* sA = base;
  uint8_t* sB = base + 16384;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 32; i += 128)
    *reinterpret_cast<float*>(sA + operand_offset(AM, i / 32, i % 32)) = A[i];
  for (int i = tid; i < N * 32; i += 128)
    *reinterpret_cast<float*>(sB + operand_offset(BM, i / 32, i % 32)) = B[i];
  fence_proxy_async();
  if (warp == 0) tmem_alloc<256>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tslot;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, N, A_MN, B_MN);
    for (int s = 0; s < 4; ++s)
      mma_tf32(taddr, operand_desc(AM, smem_u32(sA), s), operand_desc(BM, smem_u32(sB), s), idesc,
               s > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(taddr + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(taddr);
}

// kind::f16 variant: A[128 x 64] fp16, B[N x 64] fp16, four K=16 MMAs.
// mode 0: K-major SWIZZLE_128B (row = 64 halves = 128 B, K step = 32 B);
// mode 1: MN-major SWIZZLE_128B (blocks of 64 MN elements x 64 K rows).
// mode 2: MN-major SWIZZLE_64B (blocks of 32 MN elements = 64-byte rows).
__device__ __forceinline__ uint32_t sw64_offset(uint32_t row, uint32_t b) {
  return row * 64u + ((((b >> 4) ^ ((row >> 1) & 3u)) << 4) | (b & 15u));
}
__device__ __forceinline__ uint32_t f16_offset(int mode, int row, int k) {
  if (mode == 0) return sw128_offset(row, 2 * k);
  if (mode == 1) return (row / 64) * 8192 + sw128_offset(k, 2 * (row % 64));
  return (row / 32) * 4096 + sw64_offset(k, 2 * (row % 32));
}
__device__ __forceinline__ uint64_t f16_desc(int mode, uint32_t base, int s) {
  if (mode == 0) return sw128_desc(base + s * 32, 16, 1024);
  if (mode == 1) return sw128_desc(base + s * 2048, 8192, 1024);
  return sw128_desc(base + s * 1024, 4096, 512, 4);
}

template <int AM, int BM>
__global__ void __launch_bounds__(128) k_tc_selftest_f16(const uint16_t* __restrict__ A,
                                                         const uint16_t* __restrict__ B,
                                                         float* __restrict__ D, int N) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* base = align1024(smem_raw);
  uint8_t* sA = base;
  uint8_t* sB = base + 16384;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 64; i += 128)
    *reinterpret_cast<uint16_t*>(sA + f16_offset(AM, i / 64, i % 64)) = A[i];
  for (int i = tid; i < N * 64; i += 128)
    *reinterpret_cast<uint16_t*>(sB + f16_offset(BM, i / 64, i % 64)) = B[i];
  fence_proxy_async();
  if (warp == 0) tmem_alloc<256>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tslot;
  if (tid == 0) {
    const uint32_t idesc = idesc_f16(128, N, AM != 0, BM != 0);
    for (int s = 0; s < 4; ++s)
      mma_f16(taddr, f16_desc(AM, smem_u32(sA), s), f16_desc(BM, smem_u32(sB), s), idesc, s > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(taddr + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(taddr);
}


// 2-SM variant (cluster of 2 CTAs, tcgen05.mma.cta_group::2, M = 256):
// CTA r stages A rows [128 r, 128 r + 128) and B rows [N/2 r, N/2 r + N/2)
// (K-major SW128, K = 64 fp16); CTA 0 issues four K = 16 MMAs; each CTA
// reads its 128 accumulator lanes = D rows [128 r, 128 r + 128).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    k_tc_selftest_2sm(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B,
                      float* __restrict__ D, int N) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* base = align1024(smem_raw);
  uint8_t* sA = base;
  uint8_t* sB = base + 16384;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const int nh = N / 2;
  for (int i = tid; i < 128 * 64; i += 128)
    *reinterpret_cast<uint16_t*>(sA + sw128_offset(i / 64, 2 * (i % 64))) = A[128 * rank * 64 + i];
  for (int i = tid; i < nh * 64; i += 128)
    *reinterpret_cast<uint16_t*>(sB + sw128_offset(i / 64, 2 * (i % 64))) = B[nh * rank * 64 + i];
  fence_proxy_async();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t taddr = tslot;
  if (rank == 0 && warp == 0) {
    if (elect_one_sync()) {
      const uint32_t idesc = idesc_f16(256, N, false, false);
      for (int s = 0; s < 4; ++s) {
        const uint64_t a = sw128_desc(smem_u32(sA) + s * 32, 16, 1024);
        const uint64_t b = sw128_desc(smem_u32(sB) + s * 32, 16, 1024);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(taddr),
            "l"(a), "l"(b), "r"(idesc), "r"(s)
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
          "[%0], %1;" ::"r"(smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(taddr + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j)
      D[(int64_t)(128 * rank + warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(taddr) : "memory");
}

}  // namespace
}  // namespace n2f

using namespace n2f;

extern "C" int n2f_tc_selftest_f16(const uint16_t* A, const uint16_t* B, float* D, int N, int a_mn,
                                   int b_mn, void* stream) {
  if (N < 64 || N > 256 || N % 64) return fail(N2F_ERR_ARG, "selftest_f16 N=%d", N);
  const int smem = 1024 + 16384 + N * 128;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto launch = [&](auto kern) -> int {
    N2F_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, 128, smem, st>>>(A, B, D, N);
    N2F_LAUNCH_CHECK();
    return N2F_OK;
  };
  if (a_mn < 0 || a_mn > 2 || b_mn < 0 || b_mn > 2) return fail(N2F_ERR_ARG, "selftest_f16 modes");
  int s;
  switch (a_mn * 3 + b_mn) {
    case 0: s = launch(k_tc_selftest_f16<0, 0>); break;
    case 1: s = launch(k_tc_selftest_f16<0, 1>); break;
    case 2: s = launch(k_tc_selftest_f16<0, 2>); break;
    case 3: s = launch(k_tc_selftest_f16<1, 0>); break;
    case 4: s = launch(k_tc_selftest_f16<1, 1>); break;
    case 5: s = launch(k_tc_selftest_f16<1, 2>); break;
    case 6: s = launch(k_tc_selftest_f16<2, 0>); break;
    case 7: s = launch(k_tc_selftest_f16<2, 1>); break;
    default: s = launch(k_tc_selftest_f16<2, 2>); break;
  }
  if (s != N2F_OK) return s;
  N2F_CUDA(cudaStreamSynchronize(st));
  return N2F_OK;
}

extern "C" int n2f_tc_selftest(const float* A, const float* B, float* D, int N, int a_mn, int b_mn,
                               void* stream) {
  if (N < 32 || N > 256 || N % 32) return fail(N2F_ERR_ARG, "selftest N=%d", N);
  if (a_mn < 0 || a_mn > 2 || b_mn < 0 || b_mn > 2) return fail(N2F_ERR_ARG, "selftest modes");
  const int smem = 1024 + 16384 + N * 128;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto launch = [&](auto kern) -> int {
    N2F_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, 128, smem, st>>>(A, B, D, N);
    N2F_LAUNCH_CHECK();
    return N2F_OK;
  };
  int s = N2F_OK;
  switch (a_mn * 3 + b_mn) {
    case 0: s = launch(k_tc_selftest<0, 0>); break;
    case 1: s = launch(k_tc_selftest<0, 1>); break;
    case 2: s = launch(k_tc_selftest<0, 2>); break;
    case 3: s = launch(k_tc_selftest<1, 0>); break;
    case 4: s = launch(k_tc_selftest<1, 1>); break;
    case 5: s = launch(k_tc_selftest<1, 2>); break;
    case 6: s = launch(k_tc_selftest<2, 0>); break;
    case 7: s = launch(k_tc_selftest<2, 1>); break;
    default: s = launch(k_tc_selftest<2, 2>); break;
  }
  if (s != N2F_OK) return s;
  N2F_CUDA(cudaStreamSynchronize(st));
  return N2F_OK;
}

extern "C" int n2f_tc_selftest_2sm(const uint16_t* A, const uint16_t* B, float* D, int N,
                                   void* stream) {
  if (N < 32 || N > 256 || N % 32) return fail(N2F_ERR_ARG, "selftest_2sm N=%d", N);
  const int smem = 1024 + 16384 + (N / 2) * 128;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  N2F_CUDA(cudaFuncSetAttribute(k_tc_selftest_2sm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_tc_selftest_2sm<<<2, 128, smem, st>>>(A, B, D, N);
  N2F_LAUNCH_CHECK();
  N2F_CUDA(cudaStreamSynchronize(st));
  return N2F_OK;
}
