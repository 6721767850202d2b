// tcgen05 (5th-gen tensor core) kernels for the 3x3 convolutions, 3xTF32
// split precision: x = hi + lo (hi = tf32 top bits, lo = exact residual);
// A.B ~= Ah.Bh + Ah.Bl + Al.Bh.  The tensor core truncates fp32 operands to
// tf32 by itself, so the raw fp32 tensor IS the "hi" operand and only the lo
// residual is stored beside it.
//
// Accumulation: the tensor core's fp32 accumulation truncates (measured bias
// -4.9e-6 relative at K = 2304 when one TMEM accumulator takes the whole
// K loop, tests/test_gpu_kernels.py::test_conv_accuracy_vs_f64), and that
// systematic shrink compounds through the 7-layer dgrad chain.  So the K loop
// is cut into groups of kGroup chunks; each group accumulates into a fresh
// TMEM buffer (ping-pong, 2 x BN columns) and the epilogue warps add the
// group results into fp32 registers with round-to-nearest while the tensor
// core runs the next group.
#include <cudaTypedefs.h>

#include "n2f_internal.cuh"
#include "tc_common.cuh"

namespace n2f {
namespace {

using namespace tc;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ---------------------------------------------------------------------------
// 3x3 conv forward / dgrad as a TMA-fed tcgen05 implicit GEMM.
//   M = 128 pixels (a 32 x 4 spatial tile), N = all output channels (BN),
//   K = 9 taps x C in chunks of 32 channels (128 B rows, SWIZZLE_128B).
// Per K chunk, TMA loads the shifted input tile for the tap (out-of-bounds
// coordinates zero-fill = the reference's zero padding, tensor.py:231-238)
// and its lo residual, plus the weight slice and its lo residual.
// Warp roles (320 threads): w0.lane0 TMA producer; w1.lane0 MMA issuer (w1
// owns TMEM); w2..w9 accumulate/epilogue: warp w reads TMEM lane quarter
// (w % 4) and column half (w - 2) / 4.  Epilogue: fused bias+ReLU (forward)
// or ReLU-mask of the layer input (dgrad), optional per-tile column sums
// (the bias gradient of that tensor), output + lo residual stores.
// ---------------------------------------------------------------------------
constexpr int kTW = 32, kTH = 4;
constexpr int kThreadsTc = 320;
// Each pipeline stage carries K = kKC (channels for fwd/dgrad, pixels for
// wgrad) and kGroup stages form one TMEM accumulation group; within a group
// the small cross-term MMAs are issued first, then the hi*hi MMAs, so only 4
// truncating accumulates per group act on a large accumulator value.
// Measured on the box: 32-channel stages (128-byte rows, SWIZZLE_128B),
// kGroup = 1 beat 16-channel stages with 4-6 stages in flight and kGroup = 2
// (L8 fwd 229 vs 217 TF/s, L8 wgrad 214 vs 119 TF/s).
constexpr int kKC = 32;
#ifndef N2F_KGROUP
#define N2F_KGROUP 1
#endif
constexpr int kGroup = N2F_KGROUP;
constexpr int kRowBytes = kKC * 4;

template <int BN>
struct FwdCfg {
  static constexpr int kStageA = 128 * kRowBytes;
  static constexpr int kStageB = BN * kRowBytes;
  static constexpr int kStageBytes = 2 * kStageA + 2 * kStageB;
  // wide layers: as many stages as fit one CTA per SM; narrow layers (short K
  // loops, per-tile overhead dominates): 2 stages so two CTAs share an SM and
  // one's prologue/epilogue overlaps the other's MMAs
  static constexpr int kStages =
      BN >= 128 ? ((200 * 1024) / kStageBytes > 4 ? 4 : (200 * 1024) / kStageBytes) : 2;
  static constexpr int kSmem = kStages * kStageBytes + 1024;
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;  // two group buffers
  static constexpr int kHalf = BN / 2;                         // columns per epilogue warp
};

// K-major operand, rows of kRowBytes: SWIZZLE_128B (32 ch) or SWIZZLE_64B (16 ch)
__device__ __forceinline__ uint64_t kdesc(uint32_t addr) {
  return kKC == 32 ? sw128_desc(addr, 16, 1024, 2) : sw128_desc(addr, 16, 512, 4);
}
// MN-major operand (SW128_BASE32B), blocks of kKC pixel rows x 128 B
__device__ __forceinline__ uint64_t mndesc(uint32_t addr) {
  return sw128_desc(addr, kKC * 128, 512, kLayoutSw128Base32);
}

__device__ __forceinline__ float4 lo4(float4 v) {
  float4 r;
  float h;
  split_tf32(v.x, h, r.x);
  split_tf32(v.y, h, r.y);
  split_tf32(v.z, h, r.z);
  split_tf32(v.w, h, r.w);
  return r;
}

// Persistent: each CTA (one per SM) walks tiles blockIdx.x, +gridDim.x, ...
// The producer streams stages across tile boundaries, the MMA issuer keeps the
// two TMEM group buffers busy across tiles, and the accumulate warps' epilogue
// of tile t overlaps the first groups of tile t+1; barrier init, TMEM alloc
// and descriptor prefetch happen once per CTA.
template <int BN>
__global__ void __launch_bounds__(kThreadsTc, 1)
    k_conv3x3_tc(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mxl,
                 const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mwl,
                 const float* __restrict__ bias, const float* __restrict__ mask,
                 float* __restrict__ y, float* __restrict__ ylo, float* __restrict__ colsum,
                 int H, int W, int C, int epi) {
  using Cfg = FwdCfg<BN>;
  constexpr int S = Cfg::kStages;
  constexpr int HALF = Cfg::kHalf;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[S], empty[S], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  __shared__ float csum[4][BN];
  uint8_t* base = align1024(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tiles_x = (W + kTW - 1) / kTW;
  const int ntiles = tiles_x * ((H + kTH - 1) / kTH);
  const int cpt = C / kKC, KB = 9 * cpt;  // C % 32 == 0, so KB is even
  const int NG = KB / kGroup;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // one arrive per accumulate warp
    }
    fence_barrier_init();
    tma_prefetch(&mx);
    tma_prefetch(&mxl);
    tma_prefetch(&mw);
    tma_prefetch(&mwl);
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (stage index `it` runs across tiles)
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int x0 = (tile % tiles_x) * kTW, y0 = (tile / tiles_x) * kTH;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % S, round = it / S;
          if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
          const int tap = kb / cpt, c0 = (kb - tap * cpt) * kKC;
          const int ky = tap / 3, kx = tap - 3 * ky;
          uint8_t* st = base + s * Cfg::kStageBytes;
          mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
          tma_load_3d(st, &mx, &full[s], c0, x0 + kx - 1, y0 + ky - 1);
          tma_load_3d(st + Cfg::kStageA, &mxl, &full[s], c0, x0 + kx - 1, y0 + ky - 1);
          tma_load_2d(st + 2 * Cfg::kStageA, &mw, &full[s], tap * C + c0, 0);
          tma_load_2d(st + 2 * Cfg::kStageA + Cfg::kStageB, &mwl, &full[s], tap * C + c0, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: one group = kGroup stages (K = 32) into a fresh buffer
      constexpr uint32_t idesc = idesc_tf32(128, BN, false, false);
      int it = 0, gg = 0;  // stage and group counters across tiles
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int g = 0; g < NG; ++g, ++gg) {
          const int b = gg & 1;
          if (gg >= 2) mbar_wait(&tempty[b], ((gg >> 1) - 1) & 1);
          const uint32_t d = taddr + b * BN;
          // per stage: the small cross terms first (accumulator still tiny), then hi*hi
          for (int j = 0; j < kGroup; ++j, ++it) {
            const int s = it % S;
            mbar_wait(&full[s], (it / S) & 1);
            tc_fence_after();
            const uint32_t ah = smem_u32(base + s * Cfg::kStageBytes), al = ah + Cfg::kStageA,
                           bh = ah + 2 * Cfg::kStageA, bl = bh + Cfg::kStageB;
#pragma unroll
            for (int k = 0; k < kKC / 8; ++k) {
              mma_tf32(d, kdesc(ah + 32 * k), kdesc(bl + 32 * k), idesc, (j | k) != 0);
              mma_tf32(d, kdesc(al + 32 * k), kdesc(bh + 32 * k), idesc, 1);
            }
#pragma unroll
            for (int k = 0; k < kKC / 8; ++k)
              mma_tf32(d, kdesc(ah + 32 * k), kdesc(bh + 32 * k), idesc, 1);
            mma_commit(&empty[s]);
          }
          mma_commit(&tfull[b]);
        }
      }
    }
  } else {
    // ---- group accumulation in registers (round-to-nearest fp32 adds)
    const int q = warp & 3;          // TMEM lane quarter
    const int half = (warp - 2) >> 2;  // column half
    const uint32_t lane_base = taddr + ((uint32_t)(q * 32) << 16) + half * HALF;
    int gg = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int x0 = (tile % tiles_x) * kTW, y0 = (tile / tiles_x) * kTH;
    float acc[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) acc[j] = 0.f;
    for (int g = 0; g < NG; ++g, ++gg) {
      const int b = gg & 1;
      mbar_wait(&tfull[b], (gg >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < HALF; c += (HALF < 32 ? HALF : 32)) {
        uint32_t r[32];
        if (HALF < 32)
          tmem_ld16(lane_base + b * BN + c, r);
        else
          tmem_ld32(lane_base + b * BN + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < (HALF < 32 ? HALF : 32); ++j) acc[c + j] += __uint_as_float(r[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }

    // ---- epilogue
    const int m = q * 32 + lane;
    const int py = y0 + m / kTW, px = x0 + m % kTW;
    const bool valid = py < H && px < W;
    const int64_t p = (int64_t)py * W + px;
    const int n0 = half * HALF;
#pragma unroll
    for (int j = 0; j < HALF; j += 4) {
      float4 v = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
      if (epi == kEpiBiasRelu || epi == kEpiBias) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + n0 + j));
        v.x += bb.x; v.y += bb.y; v.z += bb.z; v.w += bb.w;
        if (epi == kEpiBiasRelu) {
          v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
        }
      } else if (epi == kEpiMask) {
        float4 mk = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) mk = __ldg(reinterpret_cast<const float4*>(mask + p * BN + n0 + j));
        v.x = mk.x > 0.f ? v.x : 0.f;
        v.y = mk.y > 0.f ? v.y : 0.f;
        v.z = mk.z > 0.f ? v.z : 0.f;
        v.w = mk.w > 0.f ? v.w : 0.f;
      }
      if (!valid) v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (colsum) {  // deterministic per-tile column sums (bias gradient of this tensor)
        float s0 = v.x, s1 = v.y, s2 = v.z, s3 = v.w;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s0 += __shfl_xor_sync(0xffffffffu, s0, o);
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          s3 += __shfl_xor_sync(0xffffffffu, s3, o);
        }
        if (lane == 0) {
          csum[q][n0 + j] = s0;
          csum[q][n0 + j + 1] = s1;
          csum[q][n0 + j + 2] = s2;
          csum[q][n0 + j + 3] = s3;
        }
      }
      if (valid) {
        *reinterpret_cast<float4*>(y + p * BN + n0 + j) = v;
        if (ylo) *reinterpret_cast<float4*>(ylo + p * BN + n0 + j) = lo4(v);
      }
    }
    if (colsum) {  // the 8 accumulate warps only (named barrier 1)
      asm volatile("bar.sync 1, 256;" ::: "memory");
      for (int n = tid - 64; n < BN; n += 256)
        colsum[(int64_t)tile * BN + n] = (csum[0][n] + csum[1][n]) + (csum[2][n] + csum[3][n]);
      asm volatile("bar.sync 1, 256;" ::: "memory");  // csum reusable for the next tile
    }
    }  // tile loop
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(taddr);
}

// ---------------------------------------------------------------------------
// 3x3 conv wgrad as a tcgen05 GEMM with both operands MN-major:
//   D[m = (tap, c)][n = o] = sum_p X[p + d(tap)][c] * G[p][o]
//   M = 128 (tap, c) rows (4 blocks of 32 channels, each within one tap),
//   N = Cout, K = pixels in chunks of 32 (one image-row segment).
// TMA boxes (32 ch x 32 px) land as [pixel][32 ch] rows with the 32-byte
// swizzle atom (SWIZZLE_128B_ATOM_32B), the MN-major tf32 operand layout
// (UMMA SWIZZLE_128B_BASE32B).  The pixel range is split across CTAs
// (deterministic split-K); each CTA writes its partial dW[o][tap][c] and Adam
// reduces the partials in fixed order.  Accumulation is grouped exactly like
// the forward kernel (fresh TMEM buffer per group, fp32 register sums).
// ---------------------------------------------------------------------------
constexpr int kSegW = kKC;  // pixels per stage (one image-row segment)

template <int BN>
__global__ void __launch_bounds__(kThreadsTc, 1)
    k_wgrad3x3_tc(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mxl,
                  const __grid_constant__ CUtensorMap mg, const __grid_constant__ CUtensorMap mgl,
                  float* __restrict__ part, int H, int W, int C, int nsplit) {
  using Cfg = FwdCfg<BN>;  // same stage bytes: A = 4 x 16 px x 128 B, B = BN/32 x 16 px x 128 B
  constexpr int kBlk = kSegW * 128;  // bytes of one 32-channel MN block
  constexpr int S = Cfg::kStages;
  constexpr int HALF = Cfg::kHalf;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[S], empty[S], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  uint8_t* base = align1024(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K9 = 9 * C;
  const int m0 = blockIdx.x * 128;
  const int split = blockIdx.y;
  const int segs_x = (W + kSegW - 1) / kSegW;
  const int nseg = segs_x * H;
  const int s0 = (int)((int64_t)nseg * split / nsplit), s1 = (int)((int64_t)nseg * (split + 1) / nsplit);
  const int KB = s1 - s0;
  const int NG = (KB + kGroup - 1) / kGroup;
  int nblk_a = (K9 - m0 + 31) / 32;
  if (nblk_a > 4) nblk_a = 4;
  const uint32_t stage_bytes = (uint32_t)nblk_a * kBlk * 2u + (uint32_t)Cfg::kStageB * 2u;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_barrier_init();
    tma_prefetch(&mx);
    tma_prefetch(&mxl);
    tma_prefetch(&mg);
    tma_prefetch(&mgl);
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tslot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % S, round = kb / S;
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
        const int seg = s0 + kb;
        const int y0 = seg / segs_x, x0 = (seg - y0 * segs_x) * kSegW;
        uint8_t* st = base + s * Cfg::kStageBytes;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        for (int j = 0; j < nblk_a; ++j) {
          const int mm = m0 + 32 * j, tap = mm / C, c = mm - tap * C;
          const int ky = tap / 3, kx = tap - 3 * ky;
          tma_load_3d(st + j * kBlk, &mx, &full[s], c, x0 + kx - 1, y0 + ky - 1);
          tma_load_3d(st + Cfg::kStageA + j * kBlk, &mxl, &full[s], c, x0 + kx - 1, y0 + ky - 1);
        }
        for (int jn = 0; jn < BN / 32; ++jn) {
          tma_load_3d(st + 2 * Cfg::kStageA + jn * kBlk, &mg, &full[s], 32 * jn, x0, y0);
          tma_load_3d(st + 2 * Cfg::kStageA + Cfg::kStageB + jn * kBlk, &mgl, &full[s], 32 * jn, x0,
                      y0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(128, BN, true, true);
      for (int g = 0; g < NG; ++g) {
        const int b = g & 1;
        if (g >= 2) mbar_wait(&tempty[b], ((g >> 1) - 1) & 1);
        const int ng = (g + 1) * kGroup <= KB ? kGroup : KB - g * kGroup;
        const uint32_t d = taddr + b * BN;
        for (int j = 0; j < ng; ++j) {  // per stage: cross terms first, then hi*hi
          const int kb = g * kGroup + j, s = kb % S;
          mbar_wait(&full[s], (kb / S) & 1);
          tc_fence_after();
          const uint32_t ah = smem_u32(base + s * Cfg::kStageBytes), al = ah + Cfg::kStageA,
                         bh = ah + 2 * Cfg::kStageA, bl = bh + Cfg::kStageB;
#pragma unroll
          for (int k = 0; k < kSegW / 8; ++k) {
            mma_tf32(d, mndesc(ah + 1024 * k), mndesc(bl + 1024 * k), idesc, (j | k) != 0);
            mma_tf32(d, mndesc(al + 1024 * k), mndesc(bh + 1024 * k), idesc, 1);
          }
#pragma unroll
          for (int k = 0; k < kSegW / 8; ++k)
            mma_tf32(d, mndesc(ah + 1024 * k), mndesc(bh + 1024 * k), idesc, 1);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[b]);
      }
    }
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_base = taddr + ((uint32_t)(q * 32) << 16) + half * HALF;
    float acc[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) acc[j] = 0.f;
    for (int g = 0; g < NG; ++g) {
      const int b = g & 1;
      mbar_wait(&tfull[b], (g >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < HALF; c += (HALF < 32 ? HALF : 32)) {
        uint32_t r[32];
        if (HALF < 32)
          tmem_ld16(lane_base + b * BN + c, r);
        else
          tmem_ld32(lane_base + b * BN + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < (HALF < 32 ? HALF : 32); ++j) acc[c + j] += __uint_as_float(r[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    const int m = m0 + q * 32 + lane;
    if (m < K9) {
      float* dst = part + (int64_t)split * BN * K9 + m;
#pragma unroll
      for (int j = 0; j < HALF; ++j) dst[(int64_t)(half * HALF + j) * K9] = acc[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(taddr);
}

__global__ void k_split_lo(const float* __restrict__ x, float* __restrict__ lo, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float h;
    split_tf32(x[i], h, lo[i]);
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int encoder() {
  if (g_encode) return N2F_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  N2F_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess)
    return fail(N2F_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return N2F_OK;
}

// NHWC activation [H][W][C] fp32 viewed as 3-D (C, W, H).
int map_act(CUtensorMap* m, const float* p, int C, int W, int H, int bc, int bw, int bh,
            CUtensorMapSwizzle sw) {
  N2F_TRY(encoder());
  const cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H};
  const cuuint64_t strides[2] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4};
  const cuuint32_t box[3] = {(cuuint32_t)bc, (cuuint32_t)bw, (cuuint32_t)bh};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(N2F_ERR_CUDA, "cuTensorMapEncodeTiled(act) failed: %d", (int)r);
  return N2F_OK;
}

// Row-major matrix [rows][cols] fp32 viewed as 2-D (cols, rows).
int map_mat(CUtensorMap* m, const float* p, int cols, int rows, int bc, int br,
            CUtensorMapSwizzle sw) {
  N2F_TRY(encoder());
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  const cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(N2F_ERR_CUDA, "cuTensorMapEncodeTiled(mat) failed: %d", (int)r);
  return N2F_OK;
}

template <int BN>
int set_attr_bn() {
  N2F_CUDA(cudaFuncSetAttribute(k_conv3x3_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                FwdCfg<BN>::kSmem));
  return N2F_OK;
}

template <int BN>
int launch_conv_tc_bn(const ConvTcPlan& pl, const float* bias, const float* mask, float* y,
                      float* ylo, float* colsum, int epi, cudaStream_t st) {
  k_conv3x3_tc<BN><<<pl.grid, kThreadsTc, FwdCfg<BN>::kSmem, st>>>(
      pl.mx, pl.mxl, pl.mw, pl.mwl, bias, mask, y, ylo, colsum, pl.H, pl.W, pl.C, epi);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
      n = 148;
  }
  return n;
}

template <int BN>
int set_attr_wg() {
  N2F_CUDA(cudaFuncSetAttribute(k_wgrad3x3_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                FwdCfg<BN>::kSmem));
  return N2F_OK;
}

template <int BN>
int launch_wgrad_tc_bn(const WgradTcPlan& pl, float* part, cudaStream_t st) {
  dim3 grid(pl.mblocks, pl.nsplit);
  k_wgrad3x3_tc<BN><<<grid, kThreadsTc, FwdCfg<BN>::kSmem, st>>>(pl.mx, pl.mxl, pl.mg, pl.mgl, part,
                                                                pl.H, pl.W, pl.C, pl.nsplit);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

int set_attrs_once() {
  static bool done = false;
  if (done) return N2F_OK;
  N2F_TRY(set_attr_bn<32>());
  N2F_TRY(set_attr_bn<64>());
  N2F_TRY(set_attr_bn<128>());
  N2F_TRY(set_attr_bn<256>());
  N2F_TRY(set_attr_wg<32>());
  N2F_TRY(set_attr_wg<64>());
  N2F_TRY(set_attr_wg<128>());
  N2F_TRY(set_attr_wg<256>());
  done = true;
  return N2F_OK;
}

}  // namespace

bool tc_supported(int cin, int cout) {
  return cin % 32 == 0 && (cout == 32 || cout == 64 || cout == 128 || cout == 256);
}

int conv_tc_plan(ConvTcPlan* pl, const float* x, const float* xlo, const float* w, const float* wlo,
                 int H, int W, int C, int N) {
  if (!tc_supported(C, N)) return fail(N2F_ERR_ARG, "conv_tc_plan: C=%d N=%d", C, N);
  N2F_TRY(set_attrs_once());  // outside any stream capture
  pl->H = H;
  pl->W = W;
  pl->C = C;
  pl->N = N;
  // persistent grid: one CTA per SM (two for the narrow layers, whose smem
  // and register footprints allow it), each walking tiles with a fixed stride
  const int tiles = conv_tc_tiles(H, W);
  const int per_sm = N <= 64 ? 2 : 1;
  pl->grid = tiles < per_sm * sm_count() ? tiles : per_sm * sm_count();
  pl->cs = 1;
  const CUtensorMapSwizzle sw = kKC == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  N2F_TRY(map_act(&pl->mx, x, C, W, H, kKC, kTW, kTH, sw));
  N2F_TRY(map_act(&pl->mxl, xlo, C, W, H, kKC, kTW, kTH, sw));
  N2F_TRY(map_mat(&pl->mw, w, 9 * C, N, kKC, N, sw));
  N2F_TRY(map_mat(&pl->mwl, wlo, 9 * C, N, kKC, N, sw));
  return N2F_OK;
}

int conv_tc_tiles(int H, int W) { return ((W + kTW - 1) / kTW) * ((H + kTH - 1) / kTH); }

int conv_tc_launch(const ConvTcPlan& pl, const float* bias, const float* mask, float* y, float* ylo,
                   float* colsum, int epi, cudaStream_t st) {
  switch (pl.N) {
    case 32: return launch_conv_tc_bn<32>(pl, bias, mask, y, ylo, colsum, epi, st);
    case 64: return launch_conv_tc_bn<64>(pl, bias, mask, y, ylo, colsum, epi, st);
    case 128: return launch_conv_tc_bn<128>(pl, bias, mask, y, ylo, colsum, epi, st);
    case 256: return launch_conv_tc_bn<256>(pl, bias, mask, y, ylo, colsum, epi, st);
  }
  return fail(N2F_ERR_ARG, "conv_tc_launch: N=%d", pl.N);
}

int wgrad_tc_nsplit(int cin, int H, int W) {
  const int mblocks = (9 * cin + 127) / 128;
  const int nseg = ((W + kSegW - 1) / kSegW) * H;
  int n = 148 / mblocks;
  if (n < 1) n = 1;
  if (n > nseg) n = nseg;
  return n;
}

int wgrad_tc_plan(WgradTcPlan* pl, const float* x, const float* xlo, const float* g, const float* glo,
                  int H, int W, int C, int N, int nsplit) {
  if (!tc_supported(C, N)) return fail(N2F_ERR_ARG, "wgrad_tc_plan: C=%d N=%d", C, N);
  N2F_TRY(set_attrs_once());
  pl->H = H;
  pl->W = W;
  pl->C = C;
  pl->N = N;
  pl->mblocks = (9 * C + 127) / 128;
  pl->nsplit = nsplit;
  const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  N2F_TRY(map_act(&pl->mx, x, C, W, H, 32, kSegW, 1, sw));
  N2F_TRY(map_act(&pl->mxl, xlo, C, W, H, 32, kSegW, 1, sw));
  N2F_TRY(map_act(&pl->mg, g, N, W, H, 32, kSegW, 1, sw));
  N2F_TRY(map_act(&pl->mgl, glo, N, W, H, 32, kSegW, 1, sw));
  return N2F_OK;
}

int wgrad_tc_launch(const WgradTcPlan& pl, float* part, cudaStream_t st) {
  switch (pl.N) {
    case 32: return launch_wgrad_tc_bn<32>(pl, part, st);
    case 64: return launch_wgrad_tc_bn<64>(pl, part, st);
    case 128: return launch_wgrad_tc_bn<128>(pl, part, st);
    case 256: return launch_wgrad_tc_bn<256>(pl, part, st);
  }
  return fail(N2F_ERR_ARG, "wgrad_tc_launch: N=%d", pl.N);
}

int split_lo(const float* x, float* lo, int64_t n, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_split_lo<<<(unsigned)blocks, 256, 0, st>>>(x, lo, n);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

}  // namespace n2f
