// Microbenchmark: fixed cost per kernel node of a CUDA graph for kernels shaped
// like the engine's tcgen05 convolutions (320 threads, CTA pairs, ~200 KB
// dynamic smem, TMEM alloc/dealloc, cluster syncs, PDL trigger/wait), doing no
// work.  Prints us per node with and without programmatic dependent launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o graph_gap graph_gap.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int TMEM>
__global__ void __launch_bounds__(320, 1) k_skel(int* sink) {
  extern __shared__ uint8_t smem[];
  __shared__ uint32_t slot;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5;
  if (TMEM && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] += 1;
  smem[threadIdx.x] = 0;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (TMEM && warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

__global__ void k_simt(int* sink, int n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[1] += n;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 16);
  cudaMemset(sink, 0, 16);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_skel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_skel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int N = 100;
  for (int variant = 0; variant < 6; ++variant) {
    const bool pdl = variant & 1;
    const int kind = variant >> 1;  // 0 tc skeleton with TMEM, 1 without TMEM, 2 small SIMT kernel
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < N; ++i) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = pdl;
      cfg.stream = st;
      cfg.attrs = attr;
      if (kind < 2) {
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(320);
        cfg.dynamicSmemBytes = smem;
        cfg.numAttrs = 2;
        cudaLaunchKernelEx(&cfg, kind == 0 ? k_skel<1> : k_skel<0>, sink);
      } else {
        cfg.gridDim = dim3(1024);
        cfg.blockDim = dim3(256);
        cfg.numAttrs = 1;
        cfg.attrs = attr + 1;
        cudaLaunchKernelEx(&cfg, k_simt, sink, i);
      }
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ex;
    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
      printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ex, st);
    cudaEventRecord(a, st);
    const int R = 20;
    for (int r = 0; r < R; ++r) cudaGraphLaunch(ex, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const char* names[3] = {"tc skeleton (TMEM, cluster 2, 200 KB smem)", "tc skeleton without TMEM",
                            "SIMT 1024x256"};
    printf("%-45s pdl=%d: %.2f us per node (%s)\n", names[kind], (int)pdl, 1000.0 * ms / (R * N),
           cudaGetErrorString(cudaGetLastError()));
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
  }
  return 0;
}
