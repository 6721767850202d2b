// Microbenchmark: tcgen05.mma pipeline with per-group commits.
//  mode 0: one thread issues groups of 12 MMAs (M128 N256 K16 f16), one
//          commit per group to a dummy barrier (nobody waits).
//  mode 1: mode 0 + a producer thread refilling an S-slot ring: the MMA
//          thread waits full[s] per stage (2 stages/group), commits empty[s];
//          the producer waits empty[s] and arrives full[s] (no data moved).
//  mode 2: mode 1 + 8 "accumulate" warps: per group wait tfull[b], arrive
//          tempty[b] (2 TMEM buffers), MMA thread waits tempty before reuse.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint32_t elect() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, 0xffffffff;\n\t@px mov.s32 %0, 1;\n\t}" : "+r"(pred));
  return pred;
}
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t acc) {
  constexpr uint32_t id = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: "r"(t), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

constexpr int S = 4, G = 2, STAGE = 48 * 1024;

template <int MODE, int RANDOM>
__global__ void __launch_bounds__(320, 1) k(int ngroups, long long* out) {
  extern __shared__ uint8_t sm[];
  __shared__ uint64_t full[S], empty[S], tfull[2], tempty[2], dummy;
  __shared__ uint32_t tslot;
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < S * STAGE / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + 12345u;  // random fp16 pairs in [-2, 2] (no inf/nan)
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<uint32_t*>(base)[i] = RANDOM ? (h & 0xBFFFBFFFu) : 0x3c003c00u;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { init(&full[s], 1); init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { init(&tfull[b], 1); init(&tempty[b], 8); }
    init(&dummy, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tslot;
  long long t0 = clock64();
  const int nst = ngroups * G;
  if (warp == 0) {
    if (MODE >= 1)
      for (int it = 0; it < nst; ++it) {
        const int s = it % S, r = it / S;
        if (r > 0) wait(&empty[s], (r - 1) & 1);
        if (elect()) arrive(&full[s]);
        __syncwarp();
      }
  } else if (warp == 1) {
    const uint64_t d0 = desc(su32(base), 512, 4);
    int it = 0;
    for (int g = 0; g < ngroups; ++g) {
      const int b = g & 1;
      if (MODE >= 2 && g >= 2) wait(&tempty[b], ((g >> 1) - 1) & 1);
      if (MODE >= 1) for (int j = 0; j < G; ++j) wait(&full[(it + j) % S], ((it + j) / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (elect()) {
        const uint32_t d = t + b * 256;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const uint64_t a = d0 + (uint64_t)(((it + j) % S) * (STAGE >> 4));
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            mma(d, a + 2 * kk, a + 2048 + 2 * kk, (j | kk) != 0);  // A-hi x B-lo
            mma(d, a + 512 + 2 * kk, a + 1024 + 2 * kk, 1);                // A-lo x B-hi
          }
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const uint64_t a = d0 + (uint64_t)(((it + j) % S) * (STAGE >> 4));
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) mma(d, a + 2 * kk, a + 1024 + 2 * kk, 1);
        }
        if (MODE >= 1) for (int j = 0; j < G; ++j) commit(&empty[(it + j) % S]);
        commit(MODE >= 2 ? &tfull[b] : &dummy);
      }
      __syncwarp();
      it += G;
    }
    if (MODE < 2) {  // wait for the tensor pipe to drain
      if (elect()) commit(&dummy);
      __syncwarp();
    }
  } else if (MODE >= 2) {
    for (int g = 0; g < ngroups; ++g) {
      const int b = g & 1;
      wait(&tfull[b], (g >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if ((threadIdx.x & 31) == 0) arrive(&tempty[b]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 64) out[blockIdx.x] = clock64() - t0;
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t) : "memory");
}

template <int MODE, int RANDOM = 0>
void run(int blocks) {
  long long* d; cudaMalloc(&d, blocks * 8);
  cudaFuncSetAttribute(k<MODE, RANDOM>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * STAGE + 1024);
  const int ng = blocks > 1 ? 20000 : 1000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE, RANDOM><<<blocks, 320, S * STAGE + 1024>>>(ng, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("random %d mode %d blocks %3d: %7.1f cycles/group (MMA bound 1536), %.3f ms, eff clock %.0f MHz, %.0f TF/s f16 %s\n",
         RANDOM, MODE, blocks, mx / ng, ms, mx / (ms * 1e3), blocks * ng * 12.0 * 128 * 256 * 16 * 2 / (ms * 1e9),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int b : {1, 148}) { run<0>(b); run<2>(b); run<0, 1>(b); run<2, 1>(b); }
  return 0;
}
