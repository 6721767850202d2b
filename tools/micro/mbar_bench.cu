// Microbenchmark: producer/consumer handoff through an S-slot ring of
// shared-memory mbarriers (one thread each side), in clock cycles per slot.
// mode 0: try_wait loop (no hint); 1: try_wait with suspend-time hint;
// 2: test_wait spin; 3: consumer arrives via tcgen05.commit (no MMAs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
template <int MODE>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    if (MODE == 1)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(par), "r"(0x989680) : "memory");
    else if (MODE == 2)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  }
}

template <int MODE, int S>
__global__ void k(int n, long long* out) {
  __shared__ uint64_t full[S], empty[S];
  __shared__ uint32_t tslot;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { init(&full[s], 1); init(&empty[s], 1); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (MODE == 3 && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < n; ++i) {
      int s = i % S, r = i / S;
      if (r > 0) wait<MODE == 3 ? 0 : MODE>(&empty[s], (r - 1) & 1);
      arrive(&full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < n; ++i) {
      int s = i % S;
      wait<MODE == 3 ? 0 : MODE>(&full[s], (i / S) & 1);
      if (MODE == 3)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&empty[s])) : "memory");
      else
        arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (MODE == 3 && warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tslot) : "memory");
}

template <int MODE, int S>
void run(int blocks, int threads) {
  long long* d; cudaMalloc(&d, blocks * 8);
  const int n = 20000;
  k<MODE, S><<<blocks, threads>>>(n, d);
  long long h[200]; cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("mode %d S=%d blocks=%d threads=%d: %.1f cycles/slot (%s)\n", MODE, S, blocks, threads, (double)h[0] / n, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 4>(1, 64); run<1, 4>(1, 64); run<2, 4>(1, 64); run<3, 4>(1, 64);
  run<0, 4>(148, 320); run<1, 4>(148, 320); run<2, 4>(148, 320); run<3, 4>(148, 320);
  run<0, 1>(1, 64); run<3, 1>(1, 64);
  return 0;
}
