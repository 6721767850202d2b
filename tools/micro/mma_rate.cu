// Microbenchmark: issue rate of back-to-back tcgen05.mma (M=128) with
// K-major operands in different swizzle layouts; cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int kind_f16, int M, int N) {
  // c_format f32 (bit 4), a/b format: f16 = 0, tf32 = 2 (bits 7-9, 10-12); K-major both
  return (1u << 4) | ((kind_f16 ? 0u : 2u) << 7) | ((kind_f16 ? 0u : 2u) << 10) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int KIND_F16, int N, int LAYOUT>
__global__ void k(int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)) : "memory"); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t t = tslot;
  // row bytes: LAYOUT 2 (SW128) -> 128 B rows, SBO 1024; LAYOUT 4 (SW64) -> 64 B rows, SBO 512
  const uint32_t sbo = LAYOUT == 2 ? 1024 : 512;
  const uint64_t a = desc(su32(base), 16, sbo, LAYOUT), b = desc(su32(base) + 16384, 16, sbo, LAYOUT);
  constexpr uint32_t id = idesc(KIND_F16, 128, N);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      const uint64_t o = (i & 1) * 2;
      if (KIND_F16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: "r"(t), "l"(a + o), "l"(b + o), "r"(id), "r"(i) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" :: "r"(t), "l"(a + o), "l"(b + o), "r"(id), "r"(i) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t) : "memory");
}

template <int KIND_F16, int N, int LAYOUT>
void run(const char* name, int blocks) {
  long long* d; cudaMalloc(&d, blocks * 8);
  auto kern = k<KIND_F16, N, LAYOUT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int n = 4000;
  kern<<<blocks, 128, 64 * 1024>>>(n, d);
  long long h[148]; cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  const double macs = 128.0 * N * (KIND_F16 ? 16 : 8);
  printf("%-22s blocks=%3d: %7.1f cycles/MMA  -> %6.0f MAC/clk/SM (%s)\n", name, blocks, mx / n, macs / (mx / n),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int b : {1, 148}) {
    run<1, 256, 2>("f16 N256 SW128", b);
    run<1, 256, 4>("f16 N256 SW64", b);
    run<1, 128, 2>("f16 N128 SW128", b);
    run<1, 128, 4>("f16 N128 SW64", b);
    run<0, 256, 2>("tf32 N256 SW128", b);
    run<0, 128, 2>("tf32 N128 SW128", b);
  }
  return 0;
}
