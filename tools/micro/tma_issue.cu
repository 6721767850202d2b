// Microbenchmark: issue cost of cp.async.bulk.tensor loads (cycles per
// instruction seen by the issuing thread) for different box sizes / ranks.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int RANK>
__global__ void k(const __grid_constant__ CUtensorMap map, int n, int bytes, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&map) : "memory");
    uint32_t phase = 0;
    long long tot = 0;
    for (int rep = 0; rep < 20; ++rep) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar)), "r"(n * bytes) : "memory");
      long long t0 = clock64();
      for (int i = 0; i < n; ++i) {
        uint8_t* dst = base + (i % 8) * bytes;
        if (RANK == 3)
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                       :: "r"(su32(dst)), "l"((uint64_t)&map), "r"(su32(&bar)), "r"(0), "r"(i % 32), "r"(i % 16) : "memory");
        else
          asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                       :: "r"(su32(dst)), "l"((uint64_t)&map), "r"(su32(&bar)), "r"(0), "r"(i % 32), "r"(0), "r"(i % 16) : "memory");
      }
      long long t1 = clock64();
      if (rep >= 4) tot += t1 - t0;
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)), "r"(phase) : "memory");
      phase ^= 1;
    }
    out[blockIdx.x] = tot / 16;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int C = 256, W = 256, H = 64;
  void* buf; cudaMalloc(&buf, (size_t)C * W * H * 2);
  cudaMemset(buf, 0, (size_t)C * W * H * 2);
  long long* d; cudaMalloc(&d, 148 * 8);
  for (int bw : {8, 32}) for (int brows : {1, 4}) for (int rank : {3, 4}) for (int blocks : {1, 148}) {
    CUtensorMap m;
    int nblk = rank == 4 ? 4 : 1;
    if (rank == 3) {
      cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H};
      cuuint64_t str[2] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2};
      cuuint32_t box[3] = {32, (cuuint32_t)bw, (cuuint32_t)brows}, es[3] = {1, 1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[4] = {32, (cuuint64_t)W, (cuuint64_t)(C / 32), (cuuint64_t)H};
      cuuint64_t str[3] = {(cuuint64_t)C * 2, 64, (cuuint64_t)W * C * 2};
      cuuint32_t box[4] = {32, (cuuint32_t)bw, (cuuint32_t)nblk, (cuuint32_t)brows}, es[4] = {1, 1, 1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const int bytes = 64 * bw * brows * nblk;
    const int n = 64;
    auto kern = rank == 3 ? k<3> : k<4>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * bytes + 1024);
    kern<<<blocks, 32, 8 * bytes + 1024>>>(m, n, bytes, d);
    long long h[148]; cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("rank %d box %2dpx x %d rows x %d blk (%6d B) blocks %3d: %6.1f cycles/issue %s\n", rank, bw, brows, nblk, bytes,
           blocks, mx / n, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
