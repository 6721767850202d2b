// tcgen05 (5th-gen tensor core) kernels for the 3x3 convolutions in split
// precision ("FP16x3").  Every operand x is held as an fp16 pair of the scaled
// value, hi = fp16(x * 2^e), lo = fp16(x * 2^e - hi), with a per-tensor
// power-of-two scale e (activations/weights 2^8, gradients 2^(ceil(log2 P) +
// 8)) keeping both parts in fp16's normal range (~22 significant bits), and a
// product as A.B ~= Ah.Bh + Ah.Bl + Al.Bh (3 kind::f16 MMAs).  The epilogue
// removes 2^-(eA + eB) exactly.  Every epilogue that writes an operand pair
// also folds max |x * 2^e| into the range-guard slot of its (tensor class,
// layer) (tc::range_note), which the stop kernel checks once per epoch.
//
// Accumulation: the tensor core's fp32 accumulation truncates (measured bias
// -4.9e-6 relative at K = 2304 when one TMEM accumulator takes the whole K
// loop, tests/test_gpu_kernels.py::test_conv_accuracy_vs_f64), and that
// systematic shrink compounds through the 7-layer dgrad chain.  The K loop is
// cut into groups; each group accumulates into a fresh TMEM buffer, the
// small cross-term MMAs of a group are issued before its hi*hi MMAs, and the
// accumulate warps add the group results into fp32 registers with
// round-to-nearest while the tensor core runs the next group.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "loss_dev.cuh"
#include "n2f_internal.cuh"
#include "tc_common.cuh"
#include "train.cuh"

// Build with -DN2F_TC_TRACE=1 for per-warp cycle accounting (profiling builds only).
// Tuning constants (A/B builds override them with -D via N2F_EXTRA_FLAGS;
// the product build uses these defaults).
// dy kernels with N <= kDy2SmMaxN run two CTAs per SM
#ifndef N2F_DY_2SM_MAXN
#define N2F_DY_2SM_MAXN 32
#endif
constexpr int kDy2SmMaxN = N2F_DY_2SM_MAXN;
// accumulation groups per tile of the dy kernels with N < 256
#ifndef N2F_DY_GROUPS_NARROW
#define N2F_DY_GROUPS_NARROW 4
#endif
// wgrad CTAs per SM for N <= 64 (split-K factor)
#ifndef N2F_WG_PER_SM_NARROW
#define N2F_WG_PER_SM_NARROW 2
#endif
// stages (32 pixels each) per accumulation group of the wgrad CTA pairs
constexpr int kWgGroupPair = 4;
#ifndef N2F_TC_TRACE
#define N2F_TC_TRACE 0
#endif

namespace n2f {
namespace {

using namespace tc;

// Align the dynamic smem base to 1 KB (SWIZZLE_128B atoms) by pointer
// arithmetic on the __shared__ array itself, so that the compiler keeps the
// shared address space (st.shared / ld.shared, not generic ST.E / LD.E).
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// Operand traits (fp16 parts).  A pipeline stage row carries 32 elements
// (64 B); one MMA consumes 32 bytes of K (16 fp16), so a K-major operand
// advances 32 B per MMA and an MN-major one 1 KB (16 rows of 64 B).
struct Prec {
  static constexpr int kES = 2;                  // bytes per element
  static constexpr int kRow = 32 * kES;          // bytes per 32-element row
  static constexpr uint32_t kLayMN = 4;          // SWIZZLE_64B (MN-major)
  // MN-major blocks of 32 channels x 32 pixel rows: LBO = block stride
  template <int CS = 1>
  __device__ static void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (CS == 2)
      mma_f16_2sm(d, a, b, idesc, acc);
    else
      mma_f16(d, a, b, idesc, acc);
  }
  static constexpr uint32_t idesc(int M, int N, bool amn, bool bmn) {
    return idesc_f16(M, N, amn, bmn);
  }
};

// Packed fp32 add (FADD2, round-to-nearest like FADD): a += (r0, r1).
__device__ __forceinline__ void add2(float& a0, float& a1, uint32_t r0, uint32_t r1) {
  asm("{\n\t.reg .b64 x, y;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 y, {%2, %3};\n\t"
      "add.rn.f32x2 x, x, y;\n\tmov.b64 {%0, %1}, x;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "r"(r0), "r"(r1));
}

// Add one TMEM group buffer (this warp's 32 lanes x HALF columns at taddr)
// into the fp32 register accumulators, two tcgen05.ld in flight per wait.
template <int HALF>
__device__ __forceinline__ void drain_add(uint32_t taddr, float (&acc)[HALF]) {
  constexpr int CH = HALF % 32 == 0 ? 32 : 16;  // columns per load (HALF = 16, 32, 48, 64, 96, 128)
  constexpr int NB = HALF / CH;
  constexpr int PB = NB >= 2 ? 2 : 1;        // loads per wait
#pragma unroll
  for (int c = 0; c < NB; c += PB) {
    uint32_t r[PB][32];
#pragma unroll
    for (int p = 0; p < PB; ++p) {
      if (c + p < NB) {
        if (CH == 16)
          tmem_ld16(taddr + (c + p) * CH, r[p]);
        else
          tmem_ld32(taddr + (c + p) * CH, r[p]);
      }
    }
    tmem_ld_wait();
#pragma unroll
    for (int p = 0; p < PB; ++p)
      if (c + p < NB)
#pragma unroll
        for (int j = 0; j < CH; j += 2)
          add2(acc[(c + p) * CH + j], acc[(c + p) * CH + j + 1], r[p][j], r[p][j + 1]);
  }
}

// Load this warp's 32 lanes x HALF accumulator columns at taddr (a tile that
// accumulated its whole K loop in TMEM), two tcgen05.ld in flight per wait.
template <int HALF>
__device__ __forceinline__ void tmem_load_all(uint32_t taddr, float (&acc)[HALF]) {
  constexpr int CH = HALF % 32 == 0 ? 32 : 16;
  constexpr int NB = HALF / CH;
  constexpr int PB = NB >= 2 ? 2 : 1;
#pragma unroll
  for (int c = 0; c < NB; c += PB) {
    uint32_t r[PB][32];
#pragma unroll
    for (int p = 0; p < PB; ++p) {
      if (c + p < NB) {
        if (CH == 16)
          tmem_ld16(taddr + (c + p) * CH, r[p]);
        else
          tmem_ld32(taddr + (c + p) * CH, r[p]);
      }
    }
    tmem_ld_wait();
#pragma unroll
    for (int p = 0; p < PB; ++p)
      if (c + p < NB)
#pragma unroll
        for (int j = 0; j < CH; ++j) acc[(c + p) * CH + j] = __uint_as_float(r[p][j]);
  }
}

// Warp roles of every tcgen05 kernel here (320 threads): warp 0 TMA
// producer, warp 1 MMA issuer (owns TMEM; whole warps walk the schedule and
// wait on mbarriers, elect.sync picks the issuing lane), warps 2..9
// accumulate + epilogue (warp w reads TMEM lane quarter w % 4 and column half
// (w - 2) / 4).
constexpr int kThreadsTc = 320;

// Raw output pointers of a conv plan.  y: fp32 values (may be null);
// yhi/ylo: fp16 pair of y * oscale.
struct ConvOut {
  float* y;
  void* yhi;
  void* ylo;
  float oscale;
};

// Programmatic dependent launch: let the next kernel of the stream launch (its
// prologue overlaps this kernel's tail), and wait for the previous one's
// results only after this kernel's own prologue.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Row-swizzled 16-byte chunk position inside a TMA staging tile whose rows are
// RB bytes (the SWIZZLE_32B / SWIZZLE_64B patterns; none for 16-byte rows).
template <int RB>
__device__ __forceinline__ int swz_chunk(int row, int k) {
  if (RB == 128) return k ^ (row & 7);
  if (RB == 64) return k ^ ((row >> 1) & 3);
  if (RB == 32) return k ^ ((row >> 2) & 1);
  return k;
}

// Epilogue output selection (bit mask of ConvTcPlan output maps).
enum { kOutY = 1, kOutHi = 2, kOutLo = 4 };

// Four fp16 values of a stored activation (the ReLU mask of a dgrad).
__device__ __forceinline__ float4 load_mask4(const void* mask, int64_t idx) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __half*>(mask) + idx));
  return make_float4(__half2float(__ushort_as_half((unsigned short)(u.x & 0xFFFFu))),
                     __half2float(__ushort_as_half((unsigned short)(u.x >> 16))),
                     __half2float(__ushort_as_half((unsigned short)(u.y & 0xFFFFu))),
                     __half2float(__ushort_as_half((unsigned short)(u.y >> 16))));
}

// ---------------------------------------------------------------------------
// FP16x3 3x3 conv forward / dgrad with halo reuse ("dy stages"), CTA pairs.
//   Each CTA owns a 16 (x) x 8 (y) pixel tile whose 128 GEMM rows are ordered
//   y-fastest (m = 8 * x + y); the pair covers 32 x 8 pixels (M = 256,
//   tcgen05.mma.cta_group::2, each CTA staging half of the weight rows).
//   A K stage is (32-channel chunk, dy): ONE activation box of 18 x-columns x
//   8 rows (tile + x halo, shifted by dy) serves the three dx taps, because a
//   dx shift of the tile is exactly 8 GEMM rows = one swizzle atom (descriptor
//   offset); one 4-D weight box holds the three taps' weight rows.  Relative
//   to one box per tap this cuts the activation bytes per MAC by 2.7x and the
//   TMA instruction count by 3x.  A stage is one TMEM accumulation group
//   (K = 96: 18 MMAs, 6 of them hi*hi).  Epilogue: TMA tensor stores.
// ---------------------------------------------------------------------------
template <int BN>
struct DyCfg {
  // K chunk of a stage: 32 channels (SWIZZLE_64B rows; 16-channel chunks with
  // five stages for N = 256 measured no faster).  A stage spans K = 96.
  static constexpr int kKC = 32;
  static constexpr int kRow = kKC * 2;                // bytes per GEMM row (fp16)
  static constexpr int kKSteps = kKC / 16;            // MMA K steps per tap and stage
  static constexpr uint32_t kLayout = 4;              // UMMA SWIZZLE_64B
  static constexpr int kDxUnits = (8 * kRow) >> 4;    // a dx shift: 8 rows, descriptor units
  static constexpr int kRowsA = 18 * 8;               // halo columns x rows
  static constexpr int kStageA = kRowsA * kRow;       // one fp16 part (hi or lo)
  static constexpr int kTapB = (BN / 2) * kRow;       // this CTA's weight rows of one tap
  static constexpr int kStageB = 3 * kTapB;           // the three dx taps
  static constexpr int kStageBytes = 2 * kStageA + 2 * kStageB;
  static constexpr int kCols = BN;                    // TMEM columns of one accumulator
  static constexpr int kTileW = 16;                   // output columns per CTA
  // narrow layers (N <= kDy2SmMaxN) run two CTAs per SM: their short
  // launches are bound by per-tile latency (TMA round trips, epilogue), which
  // a second co-resident CTA pair hides; they take half the smem budget
  static constexpr int kPerSm = BN <= kDy2SmMaxN ? 2 : 1;
  // staging slices: 32 channels (one fence + TMA issue per 32) where smem
  // allows, 16 at two CTAs per SM
  static constexpr int kEpiCols = kPerSm == 2 ? (BN / 2 < 16 ? BN / 2 : 16)
                                              : (BN / 2 < 32 ? BN / 2 : 32);
  static constexpr int kEpiBuf = 32 * kEpiCols * 4;  // one staging buffer (fp32 y, or the fp16 pair)
  static constexpr int kEpiWarpBytes = kEpiBuf;
  static constexpr int kEpiBytes = 8 * kEpiWarpBytes;
  static constexpr int kMaxStages = ((kPerSm == 2 ? 108 : 218) * 1024 - kEpiBytes - 1024) / kStageBytes;
  static constexpr int kStages = kMaxStages > 8 ? 8 : kMaxStages;
  static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + 1024;
  static constexpr int kTmemBudget = kPerSm == 2 ? 256 : 512;
  static constexpr int kBufs = kTmemBudget / kCols > 4 ? 4 : kTmemBudget / kCols;  // TMEM group buffers
  // accumulation groups per tile: each group (a run of consecutive K stages)
  // accumulates in a fresh TMEM buffer and is added into fp32 registers with
  // round-to-nearest, bounding the tensor core's truncating accumulation to
  // K / kGroupsPerTile.  The MMAs run kBufs groups ahead of the accumulate
  // warps, so (kBufs / kGroupsPerTile) of a tile's MMA time hides that tile's
  // predecessor's epilogue: 2/3 of a tile for N = 256, a whole tile below.
  static constexpr int kGroupsPerTile = BN >= 256 ? 3 : N2F_DY_GROUPS_NARROW;
  static constexpr int kTmemCols = kBufs * kCols <= 32 ? 32 : kBufs * kCols <= 64 ? 64
                                   : kBufs * kCols <= 128 ? 128 : kBufs * kCols <= 256 ? 256 : 512;
  static constexpr int kHalf = BN / 2;
};

// HEAD: 0 plain conv; 1 / 2 (BN = 256 only) = the L9 training / validation
// head fused into the epilogue (see HeadTrainArgs / HeadValArgs).
// amax: range-guard slot of the operand pair this launch writes (or null).
template <int BN, int HEAD>
__global__ void __launch_bounds__(kThreadsTc, DyCfg<BN>::kPerSm)  // 168 registers at 1 CTA/SM
    k_conv3x3_dy(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mxl,
                 const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mwl,
                 const __grid_constant__ CUtensorMap my, const __grid_constant__ CUtensorMap myh,
                 const __grid_constant__ CUtensorMap myl, int omask, float oscale, ConvOut out,
                 const float* __restrict__ bias, const void* __restrict__ mask, int mask_bits,
                 uint32_t* __restrict__ mbits_out, float* __restrict__ colsum, unsigned* __restrict__ amax,
                 float unscale, int H, int W, int C, int epi, HeadTrainArgs ht, HeadValArgs hv) {
  using Cfg = DyCfg<BN>;
  using P = Prec;
  constexpr int S = Cfg::kStages;
  constexpr int HALF = Cfg::kHalf;
  constexpr int NB = Cfg::kBufs;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[S], empty[S], tfull[NB], tempty[NB];
  __shared__ uint32_t tslot;
  __shared__ __align__(16) float csum[4][BN];
  __shared__ __align__(16) float sbias[BN];  // the bias, staged once (L1 is mostly smem here)
  __shared__ float zp[HEAD ? 2 : 1][HEAD ? 128 : 1];  // fused head: per-half partial dots
  __shared__ float sw9[HEAD ? BN : 1];                 // fused head: the 1x1 weights
  __shared__ double hred_d[4];
  __shared__ float hred_f[4];
  uint8_t* base = align1024(smem_raw);
  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  const int tiles_x = (W + 2 * Cfg::kTileW - 1) / (2 * Cfg::kTileW);
  const int nunits = tiles_x * ((H + 7) / 8);
  const int KB = 3 * (C / Cfg::kKC);  // stages per tile
  const int NG = KB < Cfg::kGroupsPerTile ? KB : Cfg::kGroupsPerTile;  // accumulation groups per tile

  if (tid == 0) {
    if (HEAD == 1 && blockIdx.x == 0 && ht.step_counter) *ht.step_counter += 1;  // Adam t
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16);  // every accumulate warp of the pair
    }
    fence_barrier_init();
    tma_prefetch(&mx);
    tma_prefetch(&mxl);
    tma_prefetch(&mw);
    tma_prefetch(&mwl);
    if (omask & kOutY) tma_prefetch(&my);
    if (omask & kOutHi) tma_prefetch(&myh);
    if (omask & kOutLo) tma_prefetch(&myl);
  }
  if (warp == 1) tmem_alloc_2sm<Cfg::kTmemCols>(&tslot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t taddr = tslot;
  pdl_wait();  // everything above overlaps the previous kernel's tail (PDL)

  if (warp == 0) {
    // ---- TMA producer: per stage one activation box (hi, lo) and one
    // three-tap weight box (hi, lo); bytes complete on the leader's barrier
    const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
    const int n0 = (int)rank * (BN / 2);
    int it = 0;
    for (int ut = cid; ut < nunits; ut += ncl) {
      const int x0 = (ut % tiles_x) * 2 * Cfg::kTileW + Cfg::kTileW * (int)rank, y0 = (ut / tiles_x) * 8;
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int s = it % S, round = it / S;
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
        const int c0 = (kb / 3) * Cfg::kKC, dy = kb % 3;
        uint8_t* st = base + s * Cfg::kStageBytes;
        if (elect_one_sync()) {
          const uint32_t fb = full0 + 8u * s;
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStageBytes);
          tma_load_3d_2sm(st, &mx, fb, c0, y0 + dy - 1, x0 - 1);
          tma_load_3d_2sm(st + Cfg::kStageA, &mxl, fb, c0, y0 + dy - 1, x0 - 1);
          tma_load_4d_2sm(st + 2 * Cfg::kStageA, &mw, fb, c0, n0, 0, dy);
          tma_load_4d_2sm(st + 2 * Cfg::kStageA + Cfg::kStageB, &mwl, fb, c0, n0, 0, dy);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (the leader issues for the pair): one stage = one group
    if (rank == 0) {
      constexpr uint32_t idesc = P::idesc(256, Cfg::kCols, false, false);
      constexpr uint32_t kAl = Cfg::kStageA >> 4, kBh = (2 * Cfg::kStageA) >> 4,
                         kBl = (2 * Cfg::kStageA + Cfg::kStageB) >> 4, kTap = Cfg::kTapB >> 4;
      const uint64_t desc0 = sw128_desc(smem_u32(base), 16, 8 * Cfg::kRow, Cfg::kLayout);
      int gg = 0, it = 0;
#if N2F_TC_TRACE
      long long we_ = 0, wf_ = 0, t0_ = clock64();
#endif
      for (int ut = cid; ut < nunits; ut += ncl) {
        for (int g = 0; g < NG; ++g, ++gg) {
          const int b = gg % NB;
#if N2F_TC_TRACE
          const long long c0 = clock64();
#endif
          if (gg >= NB) mbar_wait(&tempty[b], ((gg / NB) - 1) & 1);
#if N2F_TC_TRACE
          we_ += clock64() - c0;
#endif
          const uint32_t d = taddr + b * Cfg::kCols;
          const int s0 = g * KB / NG, s1 = (g + 1) * KB / NG;
          // stage by stage (the MMAs stream behind the TMA): the stage's cross
          // terms, then its hi*hi; a dx shift is 8 rows (one swizzle atom), a
          // K step 32 B = 2 descriptor units; the group's first MMA starts
          // its TMEM buffer from zero
          for (int kb = s0; kb < s1; ++kb, ++it) {
            const int st = it % S;
#if N2F_TC_TRACE
            const long long c1 = clock64();
#endif
            mbar_wait(&full[st], (it / S) & 1);
#if N2F_TC_TRACE
            wf_ += clock64() - c1;
#endif
            tc_fence_after();
            if (elect_one_sync()) {
              const uint64_t a0 = desc0 + (uint64_t)(st * (Cfg::kStageBytes >> 4));
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
                for (int k = 0; k < Cfg::kKSteps; ++k) {
                  const uint64_t a = a0 + Cfg::kDxUnits * dx + 2 * k;
                  const uint64_t bh = a0 + kBh + kTap * dx + 2 * k;
                  mma_f16_2sm(d, a, bh + (kBl - kBh), idesc, ((kb - s0) | dx | k) != 0);
                  mma_f16_2sm(d, a + kAl, bh, idesc, 1);
                }
              }
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
                for (int k = 0; k < Cfg::kKSteps; ++k)
                  mma_f16_2sm(d, a0 + Cfg::kDxUnits * dx + 2 * k, a0 + kBh + kTap * dx + 2 * k,
                              idesc, 1);
              }
              mma_commit_2sm(&empty[st]);
            }
            __syncwarp();
          }
          if (elect_one_sync()) mma_commit_2sm(&tfull[b]);
          __syncwarp();
        }
      }
#if N2F_TC_TRACE
      if (lane == 0 && blockIdx.x == 0)
        printf("[dy mma] C %d BN %d units/cta %d groups %d total %lld wait_tempty %lld wait_full %lld\n",
               C, BN, (nunits + ncl - 1) / ncl, gg, clock64() - t0_, we_, wf_);
#endif
    }
  } else {
    // ---- group accumulation in registers (round-to-nearest fp32 adds)
    const int q = warp & 3;            // TMEM lane quarter
    const int half = (warp - 2) >> 2;  // column half
    constexpr int ACOLS = HALF;
    const uint32_t lane_base = taddr + ((uint32_t)(q * 32) << 16) + half * ACOLS;
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
#if N2F_TC_TRACE
    long long tw = 0, td = 0, te = 0, twr = 0, tcomp = 0, tstg = 0, tiss = 0, t_0 = clock64();
#endif
    if (epi == kEpiBiasRelu || epi == kEpiBias) {
      for (int n = tid - 64; n < BN; n += 256) {
        sbias[n] = bias[n];
        if (HEAD) sw9[n] = (HEAD == 1 ? ht.w9 : hv.w9)[n];
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    // fused training head: the L8 gradient pair this thread writes is
    // w9[n] * dz * 2^e (ReLU-masked), so max |w9| of its column half bounds the
    // range-guard value per pixel (one product per pixel instead of per element)
    float w9max = 0.f;
    if constexpr (HEAD == 1) {
      const int nh = ((warp - 2) >> 2) * HALF;
      for (int j = 0; j < HALF; ++j) w9max = fmaxf(w9max, fabsf(sw9[nh + j]));
    }
    // this lane's pixel: GEMM row m = 32 q + lane = 8 * xl + yl
    const int xl = 4 * q + (lane >> 3), yl = lane & 7;
    constexpr int EC = Cfg::kEpiCols, CH = EC / 4;
    constexpr int RBY = EC * 4, RBH = EC * 2;  // staging row bytes: fp32 / fp16
    const int srow = lane;  // staging row: box {EC ch, 8 y, 4 x} staged [x][y][ch]
    uint8_t* stg0 = base + S * Cfg::kStageBytes + (warp - 2) * Cfg::kEpiWarpBytes;
    int gg = 0;
    unsigned rmax = 0;  // max |x * 2^e| of the pair values this thread wrote (range guard)
    for (int ut = cid; ut < nunits; ut += ncl) {
      const int x0 = (ut % tiles_x) * 2 * Cfg::kTileW + Cfg::kTileW * (int)rank, y0 = (ut / tiles_x) * 8;
      const int tile = ut * 2 + (int)rank;  // colsum row
      // this tile's pixel and (dgrad) its bit-packed ReLU mask words, requested
      // before the accumulation wait so the load latency hides behind the MMAs
      const int px = x0 + xl, py = y0 + yl;
      const bool valid = py < H && px < W;
      const int n0 = half * HALF;
      constexpr int WPP = BN / 32, MW = HALF / 32 > 0 ? HALF / 32 : 1;
      const int64_t pix = (int64_t)py * W + px;
      uint32_t mw[MW];
      if (epi == kEpiMask && mask_bits) {
#pragma unroll
        for (int k = 0; k < MW; ++k)
          mw[k] = valid ? __ldg(reinterpret_cast<const uint32_t*>(mask) + pix * WPP + n0 / 32 + k) : 0u;
      }
      float acc[ACOLS];
#pragma unroll
      for (int j = 0; j < ACOLS; ++j) acc[j] = 0.f;
      for (int g = 0; g < NG; ++g, ++gg) {
        const int b = gg % NB;
#if N2F_TC_TRACE
        const long long c0 = clock64();
#endif
        mbar_wait(&tfull[b], (gg / NB) & 1);
#if N2F_TC_TRACE
        const long long c1 = clock64();
        tw += c1 - c0;
#endif
        tc_fence_after();
        if (g == 0)
          tmem_load_all<ACOLS>(lane_base + b * Cfg::kCols, acc);
        else
          drain_add<ACOLS>(lane_base + b * Cfg::kCols, acc);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + 8u * b);
#if N2F_TC_TRACE
        td += clock64() - c1;
#endif
      }
#if N2F_TC_TRACE
      const long long ce = clock64();
#endif


      // ---- epilogue (see k_conv3x3_tc): scale removal, bias+ReLU or the ReLU
      // mask, column sums, bit masks, staging in the TMA swizzle layout and
      // TMA tensor stores of {EC channels, 4 x, 8 y} boxes
      uint32_t ob = 0;
      if constexpr (HEAD != 0) {
        // ---- fused L9 head.  The L8 activation (fp32, the regular epilogue's
        // rounding: scale, bias add, ReLU) replaces acc in place; the two
        // column halves exchange their partial dots with w9 through smem.
        const float* w9 = sw9;
        float pd = 0.f;
#pragma unroll
        for (int j = 0; j < HALF; ++j) {
          const float a = fmaxf(__fadd_rn(__fmul_rn(acc[j], unscale), sbias[n0 + j]), 0.f);
          acc[j] = a;
          pd = fmaf(a, w9[n0 + j], pd);
        }
        const int m = 32 * q + lane;
        zp[half][m] = pd;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const float z = __fadd_rn(__fadd_rn(zp[0][m], zp[1][m]), __ldg(HEAD == 1 ? ht.b9 : hv.b9));
        if constexpr (HEAD == 2) {
          double se = 0.0;
          if (half == 0 && valid) {
            const float o = clip_unit(sigmoid_ref(z));
            hv.ring[(int64_t)(hv.st->epoch % hv.window) * ((int64_t)H * W) + pix] = o;
            const double d = (double)o - (double)__ldg(hv.norm + pix);
            se = d * d;
          }
          if (half == 0) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
            if (lane == 0) hred_d[q] = se;
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (tid == 64) hv.part_se[tile] = (hred_d[0] + hred_d[1]) + (hred_d[2] + hred_d[3]);
        } else {
          float elem = 0.f, dz = 0.f;
          if (valid) dz = loss_grad(z, __ldg(ht.tgt + pix), ht.loss, ht.nf, ht.two_over_n, &elem);
          if (valid) rmax = max(rmax, range_bits(fabsf(dz) * w9max * oscale));
          if (half == 0 && valid) ht.zout[pix] = z;
#pragma unroll
          for (int c0 = 0; c0 < HALF; c0 += EC) {
            const int n = n0 + c0;
            float g[EC], wa[EC], gk[EC];
#pragma unroll
            for (int i = 0; i < EC; ++i) {
              const float a = acc[c0 + i];
              g[i] = (valid && a > 0.f) ? __fmul_rn(w9[n + i], dz) : 0.f;  // head backward
              gk[i] = g[i];
              wa[i] = valid ? __fmul_rn(dz, a) : 0.f;  // dW9 terms
            }
            // transpose-reduce both column sums (bias grad of L8, dW9 partial)
            int ch = 0;
#pragma unroll
            for (int o = 16, cnt = EC; o >= 1; o >>= 1) {
              if (cnt > 1) {
                const int hcnt = cnt / 2;
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < EC / 2; ++i) {
                  if (i < hcnt) {
                    const float s1 = up ? g[i] : g[i + hcnt], k1 = up ? g[i + hcnt] : g[i];
                    const float s2 = up ? wa[i] : wa[i + hcnt], k2 = up ? wa[i + hcnt] : wa[i];
                    g[i] = k1 + __shfl_xor_sync(0xffffffffu, s1, o);
                    wa[i] = k2 + __shfl_xor_sync(0xffffffffu, s2, o);
                  }
                }
                ch += up ? hcnt : 0;
                cnt = hcnt;
              } else {
                g[0] += __shfl_xor_sync(0xffffffffu, g[0], o);
                wa[0] += __shfl_xor_sync(0xffffffffu, wa[0], o);
              }
            }
            if ((lane & (32 / EC - 1)) == 0) {
              if (colsum) csum[q][n + ch] = g[0];
              ht.part_w9[((int64_t)tile * 4 + q) * BN + n + ch] = wa[0];
            }
            // stage this lane's g pair (gk: the values before the reduction)
            uint32_t hw[EC / 2], lw[EC / 2];
#pragma unroll
            for (int i = 0; i < EC; i += 2) {
              split_f16x2(__fmul_rn(gk[i], oscale), __fmul_rn(gk[i + 1], oscale), hw[i / 2], lw[i / 2]);
            }
            uint8_t* stg = stg0;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int k = 0; k < EC / 8; ++k) {
              const int off = srow * RBH + 16 * swz_chunk<RBH>(srow, k);
              *reinterpret_cast<uint4*>(stg + off) =
                  make_uint4(hw[4 * k], hw[4 * k + 1], hw[4 * k + 2], hw[4 * k + 3]);
              *reinterpret_cast<uint4*>(stg + 32 * RBH + off) =
                  make_uint4(lw[4 * k], lw[4 * k + 1], lw[4 * k + 2], lw[4 * k + 3]);
            }
            fence_proxy_async();
            __syncwarp();
            if (elect_one_sync()) {
              const int bx = x0 + 4 * q;
              tma_store_3d(&myh, stg, n, y0, bx);
              tma_store_3d(&myl, stg + 32 * RBH, n, y0, bx);
              bulk_commit_group();
            }
          }
          // per-tile db9 / loss partials over the tile's valid pixels (half 0)
          if (half == 0) {
            float sdz = dz;
            double sl = (double)elem;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              sdz += __shfl_xor_sync(0xffffffffu, sdz, o);
              sl += __shfl_xor_sync(0xffffffffu, sl, o);
            }
            if (lane == 0) {
              hred_f[q] = sdz;
              hred_d[q] = sl;
            }
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (tid == 64) {
            ht.part_b9[tile] = (hred_f[0] + hred_f[1]) + (hred_f[2] + hred_f[3]);
            ht.part_loss[tile] = (hred_d[0] + hred_d[1]) + (hred_d[2] + hred_d[3]);
          }
        }
      } else {
#pragma unroll
      for (int c0 = 0; c0 < HALF; c0 += EC) {
#if N2F_TC_TRACE
        const long long cs0 = clock64();
#endif
        const int n = n0 + c0;
        float v[EC];
#pragma unroll
        for (int i = 0; i < EC; ++i) v[i] = acc[c0 + i] * unscale;
        if (epi == kEpiBiasRelu || epi == kEpiBias) {
#pragma unroll
          for (int k = 0; k < CH; ++k) {
            const float4 bb = *reinterpret_cast<const float4*>(sbias + n + 4 * k);
            v[4 * k] += bb.x; v[4 * k + 1] += bb.y; v[4 * k + 2] += bb.z; v[4 * k + 3] += bb.w;
          }
          if (epi == kEpiBiasRelu) {
#pragma unroll
            for (int i = 0; i < EC; ++i) v[i] = fmaxf(v[i], 0.f);
          }
        } else if (epi == kEpiMask && mask_bits) {
          const uint32_t bits = mw[(c0 / 32) % MW] >> (n % 32);
#pragma unroll
          for (int i = 0; i < EC; ++i) v[i] = ((bits >> i) & 1u) ? v[i] : 0.f;
        } else if (epi == kEpiMask) {
          const int64_t idx = pix * BN + n;
#pragma unroll
          for (int k = 0; k < CH; ++k) {
            float4 mk = make_float4(0.f, 0.f, 0.f, 0.f);
            if (valid) mk = load_mask4(mask, idx + 4 * k);
            v[4 * k] = mk.x > 0.f ? v[4 * k] : 0.f;
            v[4 * k + 1] = mk.y > 0.f ? v[4 * k + 1] : 0.f;
            v[4 * k + 2] = mk.z > 0.f ? v[4 * k + 2] : 0.f;
            v[4 * k + 3] = mk.w > 0.f ? v[4 * k + 3] : 0.f;
          }
        }
        if (mbits_out) {  // this layer's ReLU mask for the next layer's dgrad
          uint32_t sbits = 0;
#pragma unroll
          for (int i = 0; i < EC; ++i) sbits |= (v[i] > 0.f ? 1u : 0u) << i;
          if constexpr (HALF < 32) {  // N = 32: each column half owns a 16-bit half word
            if (valid) reinterpret_cast<uint16_t*>(mbits_out)[pix * (BN / 16) + n / 16] = (uint16_t)sbits;
          } else {
            ob |= sbits << (n % 32);
            if ((n + EC) % 32 == 0) {
              if (valid) mbits_out[pix * WPP + n / 32] = ob;
              ob = 0;
            }
          }
        }
        if (colsum) {  // transpose-reduce column sums over the warp's 32 pixels
          float r[EC];
#pragma unroll
          for (int i = 0; i < EC; ++i) r[i] = valid ? v[i] : 0.f;
          int ch = 0;
#pragma unroll
          for (int o = 16, cnt = EC; o >= 1; o >>= 1) {
            if (cnt > 1) {
              const int hcnt = cnt / 2;
              const bool up = (lane & o) != 0;
#pragma unroll
              for (int i = 0; i < EC / 2; ++i) {
                if (i < hcnt) {
                  const float send = up ? r[i] : r[i + hcnt];
                  const float keep = up ? r[i + hcnt] : r[i];
                  r[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
              }
              ch += up ? hcnt : 0;
              cnt = hcnt;
            } else {
              r[0] += __shfl_xor_sync(0xffffffffu, r[0], o);
            }
          }
          if ((lane & (32 / EC - 1)) == 0) csum[q][n + ch] = r[0];
        }
        // the staging buffer's previous TMA stores must be done reading it
        uint8_t* stg = stg0;
#if N2F_TC_TRACE
        const long long cw = clock64();
        tcomp += cw - cs0;
#endif
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
#if N2F_TC_TRACE
        twr += clock64() - cw;
#endif
        if (omask & kOutY) {
#pragma unroll
          for (int k = 0; k < CH; ++k)
            *reinterpret_cast<float4*>(stg + srow * RBY + 16 * swz_chunk<RBY>(srow, k)) =
                make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        }
        if (omask & (kOutHi | kOutLo)) {
          uint32_t hw[EC / 2], lw[EC / 2];
#pragma unroll
          for (int i = 0; i < EC; i += 2) {
            const float a0 = v[i] * oscale, a1 = v[i + 1] * oscale;
            if (valid) rmax = max(rmax, max(range_bits(a0), range_bits(a1)));
            split_f16x2(a0, a1, hw[i / 2], lw[i / 2]);
          }
#pragma unroll
          for (int k = 0; k < EC / 8; ++k) {
            const int off = srow * RBH + 16 * swz_chunk<RBH>(srow, k);
            *reinterpret_cast<uint4*>(stg + off) =
                make_uint4(hw[4 * k], hw[4 * k + 1], hw[4 * k + 2], hw[4 * k + 3]);
            *reinterpret_cast<uint4*>(stg + 32 * RBH + off) =
                make_uint4(lw[4 * k], lw[4 * k + 1], lw[4 * k + 2], lw[4 * k + 3]);
          }
        }
        fence_proxy_async();
        __syncwarp();
#if N2F_TC_TRACE
        const long long cf = clock64();
        tstg += cf - cw;
#endif
        if (elect_one_sync()) {
          const int bx = x0 + 4 * q;
          if (omask & kOutY) tma_store_3d(&my, stg, n, y0, bx);
          if (omask & kOutHi) tma_store_3d(&myh, stg, n, y0, bx);
          if (omask & kOutLo) tma_store_3d(&myl, stg + 32 * RBH, n, y0, bx);
          bulk_commit_group();
        }
#if N2F_TC_TRACE
        __syncwarp();
        tiss += clock64() - cf;
#endif
      }
      }  // HEAD
      if (colsum) {  // the 8 accumulate warps only (named barrier 1)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        for (int n = tid - 64; n < BN; n += 256)
          colsum[(int64_t)tile * BN + n] = (csum[0][n] + csum[1][n]) + (csum[2][n] + csum[3][n]);
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
#if N2F_TC_TRACE
      te += clock64() - ce;
#endif
    }
#if N2F_TC_TRACE
    if (lane == 0 && blockIdx.x == 0 && (warp == 2 || warp == 9))
      printf("[dy acc w%d] C %d BN %d total %lld wait_tfull %lld drain %lld epilogue %lld (compute %lld "
             "wait_read %lld stage+fence %lld issue %lld)\n",
             warp, C, BN, clock64() - t_0, tw, td, te, tcomp, twr, tstg - twr, tiss);
#endif
    if (amax) range_note(amax, rmax);
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc_2sm<Cfg::kTmemCols>(taddr);
}

// ---------------------------------------------------------------------------
// 3x3 conv wgrad as a tcgen05 GEMM with both operands MN-major:
//   D[m = (tap, c)][n = o] = sum_p X[p + d(tap)][c] * G[p][o]
//   M = 128 (tap, c) rows (4 blocks of 32 channels, each within one tap),
//   N = Cout, K = pixels in stages of 32 (one image-row segment).
// TMA boxes (32 ch x 32 px) land as [pixel][32 ch] rows: the MN-major
// operand layout (TF32: 128-byte rows with the 32-byte swizzle atom,
// SWIZZLE_128B_BASE32B; FP16: 64-byte rows, SWIZZLE_64B).  The pixel range is
// split across CTAs (deterministic split-K); each CTA writes its partial
// dW[o][tap][c] (scale removed) and the partials are reduced in fixed order
// before Adam.  Accumulation is grouped exactly like the forward kernel.
// ---------------------------------------------------------------------------
constexpr int kSegW = 32;  // default pixels per stage (one image-row segment)

// wgrad stage geometry: SEG pixels (K) per stage; A = 4 MN blocks of 32
// (tap, channel) rows, B = BN / CS / 32 blocks of gradient channels.  Narrow
// layers take 64-pixel stages (twice the MMA work per TMA instruction) with
// one stage per accumulation group (K = 64, as the 2 x 32 grouping).
template <int BN, int CS, int SEG>
struct WgCfg {
  using P = Prec;
  static constexpr int kBlk = SEG * P::kRow;  // bytes of one 32-channel MN block
  static constexpr int kStageA = 4 * kBlk;
  static constexpr int kStageB = (BN / CS / 32) * kBlk;
  static constexpr int kStageBytes = 2 * kStageA + 2 * kStageB;
  static constexpr bool kTwoPerSm = CS == 1 && BN <= 64 && SEG == 32;
  // stages per TMEM accumulation group.  A group's drain reads BN fp32
  // columns x 128 lanes from TMEM (~64 B/clk): the pair kernels (N >= 128)
  // take 4 stages (128 pixels) so the MMAs of a group outlast its drain
  static constexpr int kGroup = SEG == 64 ? 1 : (CS == 2 ? kWgGroupPair : 2);
  static constexpr int kMaxStages = (200 * 1024) / kStageBytes;
  static constexpr int kStages = kTwoPerSm ? 4 : (kMaxStages > 8 ? 8 : kMaxStages);
  static constexpr int kSmem = kStages * kStageBytes + 1024;
  static constexpr int kTmemBudget = kTwoPerSm ? 256 : 512;
  static constexpr int kBufs = kTmemBudget / BN > 4 ? 4 : kTmemBudget / BN;
  static constexpr int kTmemCols = kBufs * BN;
  static constexpr int kHalf = BN / 2;
  static constexpr int kKSteps = SEG / 16;  // MMA K steps per stage
};

// CTA pairs (CS = 2, used when C % 128 == 0 and N >= 128): a cluster owns
// two consecutive M blocks (cta_group::2 MMA, M = 256); each CTA stages its
// own activation blocks and half of the gradient channels.
template <int BN, int CS, int SEG>
__global__ void __launch_bounds__(kThreadsTc, 1)
    k_wgrad3x3_tc(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mxl,
                  const __grid_constant__ CUtensorMap mg, const __grid_constant__ CUtensorMap mgl,
                  float* __restrict__ part, float unscale, int H, int W, int C, int nsplit, int xblk) {
  using Cfg = WgCfg<BN, CS, SEG>;
  using P = Prec;
  constexpr int kBlk = Cfg::kBlk;
  constexpr int S = Cfg::kStages;
  constexpr int HALF = Cfg::kHalf;
  constexpr int G = Cfg::kGroup;
  constexpr int NB = Cfg::kBufs;  // TMEM group buffers (4 for N <= 128: the short
                                  // narrow-layer groups need a deep hand-off queue)
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[S], empty[S], tfull[NB], tempty[NB];
  __shared__ uint32_t tslot;
  uint8_t* base = align1024(smem_raw);
  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = CS > 1 ? cluster_ctarank() : 0;
  const int K9 = 9 * C;
  const int m0 = blockIdx.x * 128;  // this CTA's M block ((tap, c) rows)
  // the second CTA of the last pair may have no M block of its own: it loads
  // block 0 (valid data for the pair MMA) and stores nothing
  const bool ghost = m0 >= K9;
  const int ml = ghost ? 0 : m0;
  const int split = blockIdx.y;
  const int segs_x = (W + SEG - 1) / SEG;
  const int nseg = segs_x * H;
  const int s0 = (int)((int64_t)nseg * split / nsplit), s1 = (int)((int64_t)nseg * (split + 1) / nsplit);
  const int KB = s1 - s0;
  const int NG = (KB + G - 1) / G;
  int nblk_a = (K9 - ml + 31) / 32;
  if (nblk_a > 4) nblk_a = 4;
  const uint32_t stage_bytes = (uint32_t)nblk_a * kBlk * 2u + (uint32_t)Cfg::kStageB * 2u;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8 * CS);
    }
    fence_barrier_init();
    tma_prefetch(&mx);
    tma_prefetch(&mxl);
    tma_prefetch(&mg);
    tma_prefetch(&mgl);
  }
  constexpr int kWCols = Cfg::kTmemCols;
  if (warp == 1) {
    if (CS == 2)
      tmem_alloc_2sm<kWCols>(&tslot);
    else
      tmem_alloc<kWCols>(&tslot);
  }
  tc_fence_before();
  if (CS == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tslot;
  pdl_wait();  // everything above overlaps the previous kernel's tail (PDL)

  if (warp == 0) {
    // ---- TMA producer (whole warp walks the schedule, one elected lane issues)
    const uint32_t full0 = CS == 2 ? mapa_shared(smem_u32(&full[0]), 0) : smem_u32(&full[0]);
    const int gblk0 = (int)rank * (BN / 32 / CS);  // this CTA's first gradient block
#if N2F_TC_TRACE
    long long pw = 0, pi = 0, p0 = clock64();
#endif
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % S, round = kb / S;
#if N2F_TC_TRACE
      const long long c0 = clock64();
#endif
      if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
#if N2F_TC_TRACE
      const long long c1 = clock64();
      pw += c1 - c0;
#endif
      const int seg = s0 + kb;
      const int y0 = seg / segs_x, x0 = (seg - y0 * segs_x) * SEG;
      uint8_t* st = base + s * Cfg::kStageBytes;
      if (elect_one_sync()) {
        if (CS == 1) {
          mbar_arrive_expect_tx(&full[s], stage_bytes);
          if (xblk) {  // the 4 blocks share one tap: one 4-D box
            const int tap = ml / C, c = ml - tap * C;
            const int ky = tap / 3, kx = tap - 3 * ky;
            tma_load_4d(st, &mx, &full[s], 0, x0 + kx - 1, c / 32, y0 + ky - 1);
            tma_load_4d(st + Cfg::kStageA, &mxl, &full[s], 0, x0 + kx - 1, c / 32, y0 + ky - 1);
          } else {  // one 4-D box per tap (C / 32 blocks of it)
            const int bpt = C / 32;
            for (int j = 0; j < nblk_a; j += bpt) {
              const int mm = ml + 32 * j, tap = mm / C, c = mm - tap * C;
              const int ky = tap / 3, kx = tap - 3 * ky;
              tma_load_4d(st + j * kBlk, &mx, &full[s], 0, x0 + kx - 1, c / 32, y0 + ky - 1);
              tma_load_4d(st + Cfg::kStageA + j * kBlk, &mxl, &full[s], 0, x0 + kx - 1, c / 32,
                          y0 + ky - 1);
            }
          }
          tma_load_4d(st + 2 * Cfg::kStageA, &mg, &full[s], 0, x0, 0, y0);
          tma_load_4d(st + 2 * Cfg::kStageA + Cfg::kStageB, &mgl, &full[s], 0, x0, 0, y0);
        } else {  // pair: xblk always holds, bytes complete on the leader's barrier
          const uint32_t fb = full0 + 8u * s;
          if (rank == 0) mbar_arrive_expect_tx(&full[s], CS * stage_bytes);
          const int tap = ml / C, c = ml - tap * C;
          const int ky = tap / 3, kx = tap - 3 * ky;
          tma_load_4d_2sm(st, &mx, fb, 0, x0 + kx - 1, c / 32, y0 + ky - 1);
          tma_load_4d_2sm(st + Cfg::kStageA, &mxl, fb, 0, x0 + kx - 1, c / 32, y0 + ky - 1);
          tma_load_4d_2sm(st + 2 * Cfg::kStageA, &mg, fb, 0, x0, gblk0, y0);
          tma_load_4d_2sm(st + 2 * Cfg::kStageA + Cfg::kStageB, &mgl, fb, 0, x0, gblk0, y0);
        }
      }
      __syncwarp();
#if N2F_TC_TRACE
      pi += clock64() - c1;
#endif
    }
#if N2F_TC_TRACE
    if (lane == 0 && (blockIdx.x == 0 && blockIdx.y == 0))
      printf("[wg prod] C %d BN %d CS %d stages %d total %lld wait_empty %lld issue %lld\n", C, BN, CS,
             KB, clock64() - p0, pw, pi);
#endif
  } else if (warp == 1) {
    // ---- MMA issuer (the pair's leader issues for both; whole warp waits,
    // one elected lane issues)
    if (rank == 0) {
      constexpr uint32_t idesc = P::idesc(128 * CS, BN, true, true);
      constexpr uint32_t kAl = Cfg::kStageA >> 4, kBh = (2 * Cfg::kStageA) >> 4,
                         kBl = (2 * Cfg::kStageA + Cfg::kStageB) >> 4;
      // MN-major: LBO = the stride of the 32-element MN blocks (SEG pixel rows)
      const uint64_t desc0 = sw128_desc(smem_u32(base), kBlk, 512, P::kLayMN);
      int it = 0;
#if N2F_TC_TRACE
      long long we_ = 0, wf_ = 0, is_ = 0, t0_ = clock64();
#endif
      for (int g = 0; g < NG; ++g) {
        const int b = g % NB;
#if N2F_TC_TRACE
        const long long c0 = clock64();
#endif
        if (g >= NB) mbar_wait(&tempty[b], ((g / NB) - 1) & 1);
#if N2F_TC_TRACE
        const long long c1 = clock64();
        we_ += c1 - c0;
#endif
        const int ng = (g + 1) * G <= KB ? G : KB - g * G;
        const uint32_t d = taddr + b * BN;
#if N2F_TC_TRACE
        const long long c2 = clock64();
#endif
        // stage by stage (the group's MMAs stream behind the TMA): cross terms
        // of the stage, then its hi*hi; one K step = 1 KB = 64 descriptor units
        for (int j = 0; j < ng; ++j) {
          const int st = (it + j) % S;
#if N2F_TC_TRACE
          const long long w0 = clock64();
#endif
          mbar_wait(&full[st], ((it + j) / S) & 1);
#if N2F_TC_TRACE
          wf_ += clock64() - w0;
#endif
          tc_fence_after();
          if (elect_one_sync()) {
            const uint64_t ah = desc0 + (uint64_t)(st * (Cfg::kStageBytes >> 4));
#pragma unroll
            for (int k = 0; k < Cfg::kKSteps; ++k) {
              const uint64_t a = ah + 64 * k;
              P::template mma<CS>(d, a, a + kBl, idesc, (j | k) != 0);
              P::template mma<CS>(d, a + kAl, a + kBh, idesc, 1);
            }
#pragma unroll
            for (int k = 0; k < Cfg::kKSteps; ++k) {
              const uint64_t a = ah + 64 * k;
              P::template mma<CS>(d, a, a + kBh, idesc, 1);
            }
            if (CS == 2)
              mma_commit_2sm(&empty[st]);
            else
              mma_commit(&empty[st]);
          }
          __syncwarp();
        }
        if (elect_one_sync()) {
          if (CS == 2)
            mma_commit_2sm(&tfull[b]);
          else
            mma_commit(&tfull[b]);
        }
        __syncwarp();
#if N2F_TC_TRACE
        is_ += clock64() - c2;
#endif
        it += ng;
      }
#if N2F_TC_TRACE
      if (lane == 0 && (blockIdx.x == 0 && blockIdx.y == 0))
        printf("[wg mma] C %d BN %d CS %d groups %d total %lld wait_tempty %lld wait_full %lld issue %lld\n",
               C, BN, CS, NG, clock64() - t0_, we_, wf_, is_);
#endif
    }
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_base = taddr + ((uint32_t)(q * 32) << 16) + half * HALF;
    const uint32_t tempty0 = CS == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
    float acc[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) acc[j] = 0.f;
    for (int g = 0; g < NG; ++g) {
      const int b = g % NB;
      mbar_wait(&tfull[b], (g / NB) & 1);
      tc_fence_after();
      drain_add<HALF>(lane_base + b * BN, acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CS == 2)
          mbar_arrive_cluster(tempty0 + 8u * b);
        else
          mbar_arrive(&tempty[b]);
      }
    }
    const int m = m0 + q * 32 + lane;
    if (!ghost && m < K9) {
      float* dst = part + (int64_t)split * BN * K9 + m;
#pragma unroll
      for (int j = 0; j < HALF; ++j) dst[(int64_t)(half * HALF + j) * K9] = acc[j] * unscale;
    }
  }
  tc_fence_before();
  if (CS == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    if (CS == 2)
      tmem_dealloc_2sm<kWCols>(taddr);
    else
      tmem_dealloc<kWCols>(taddr);
  }
}

__global__ void k_split_f16(const float* __restrict__ x, __half* __restrict__ hi,
                            __half* __restrict__ lo, float scale, int64_t n, unsigned* __restrict__ amax) {
  unsigned mx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float a = x[i] * scale;
    mx = max(mx, range_bits(a));
    const __half h = __float2half_rn(a);
    hi[i] = h;
    lo[i] = __float2half_rn(__fsub_rn(a, __half2float(h)));
  }
  if (amax) range_note(amax, mx);
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

// NHWC activation viewed as 4-D (32 channels, W, C / 32 blocks, H): a box
// {32, bw, nblk, 1} lands as [block][pixel][32 channels], i.e. nblk MN-major
// operand blocks of bw pixel rows in one TMA.
int map_act_blk(CUtensorMap* m, const void* p, int C, int W, int H, int bw, int nblk) {
  N2F_TRY(encoder());
  const cuuint64_t es = 2;
  const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_64B;
  const cuuint64_t dims[4] = {32, (cuuint64_t)W, (cuuint64_t)(C / 32), (cuuint64_t)H};
  const cuuint64_t strides[3] = {(cuuint64_t)C * es, 32 * es, (cuuint64_t)W * C * es};
  const cuuint32_t box[4] = {32, (cuuint32_t)bw, (cuuint32_t)nblk, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(p), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(N2F_ERR_CUDA, "cuTensorMapEncodeTiled(act4) failed: %d", (int)r);
  return N2F_OK;
}

// NHWC activation viewed as 3-D (C, H, W): a box {32, bh, bw} lands as
// [x][y][32 channels], i.e. GEMM rows ordered y-fastest (the dy-stage conv).
int map_act_yx(CUtensorMap* m, const void* p, int C, int W, int H, int bc, int bh, int bw) {
  N2F_TRY(encoder());
  const cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)W};
  const cuuint64_t strides[2] = {(cuuint64_t)W * C * 2, (cuuint64_t)C * 2};
  const cuuint32_t box[3] = {(cuuint32_t)bc, (cuuint32_t)bh, (cuuint32_t)bw};
  const CUtensorMapSwizzle sw = bc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(p), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(N2F_ERR_CUDA, "cuTensorMapEncodeTiled(act yx) failed: %d", (int)r);
  return N2F_OK;
}

// Output tensor [H][W][C] viewed as 3-D (C, H, W) for the dy kernel's TMA
// stores: a box {bc, 8 y, 4 x} is staged as [x][y][channels], i.e. row = lane.
int map_out_yx(CUtensorMap* m, void* p, bool f16, int C, int W, int H, int bc,
               CUtensorMapSwizzle sw) {
  N2F_TRY(encoder());
  const cuuint64_t es = f16 ? 2 : 4;
  const cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)W};
  const cuuint64_t strides[2] = {(cuuint64_t)W * C * es, (cuuint64_t)C * es};
  const cuuint32_t box[3] = {(cuuint32_t)bc, 8, 4};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(N2F_ERR_CUDA, "cuTensorMapEncodeTiled(out yx) failed: %d", (int)r);
  return N2F_OK;
}

// K-major weights [N][9 taps][C] (fp16) viewed as 4-D (C, N, dx, dy): a box
// {32, rows, 3, 1} holds the three dx taps of one dy as [dx][row][32 ch].
int map_w_taps(CUtensorMap* m, const void* p, int C, int N, int bc, int rows) {
  N2F_TRY(encoder());
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)N, 3, 3};
  const cuuint64_t strides[3] = {(cuuint64_t)9 * C * 2, (cuuint64_t)C * 2, (cuuint64_t)3 * C * 2};
  const cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)rows, 3, 1};
  const CUtensorMapSwizzle sw = bc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(p), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(N2F_ERR_CUDA, "cuTensorMapEncodeTiled(w taps) failed: %d", (int)r);
  return N2F_OK;
}

int set_attrs_once() {
  static bool done = false;
  if (done) return N2F_OK;
#define N2F_SMEM(kern, bytes) \
  N2F_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))
  N2F_SMEM((k_conv3x3_dy<32, 0>), DyCfg<32>::kSmem);
  N2F_SMEM((k_conv3x3_dy<64, 0>), DyCfg<64>::kSmem);
  N2F_SMEM((k_conv3x3_dy<128, 0>), DyCfg<128>::kSmem);
  N2F_SMEM((k_conv3x3_dy<256, 0>), DyCfg<256>::kSmem);
  N2F_SMEM((k_conv3x3_dy<256, 1>), DyCfg<256>::kSmem);
  N2F_SMEM((k_conv3x3_dy<256, 2>), DyCfg<256>::kSmem);
  N2F_SMEM((k_wgrad3x3_tc<32, 1, 64>), (WgCfg<32, 1, 64>::kSmem));
  N2F_SMEM((k_wgrad3x3_tc<32, 1, 128>), (WgCfg<32, 1, 128>::kSmem));
  N2F_SMEM((k_wgrad3x3_tc<64, 1, 64>), (WgCfg<64, 1, 64>::kSmem));
  N2F_SMEM((k_wgrad3x3_tc<64, 1, 128>), (WgCfg<64, 1, 128>::kSmem));
  N2F_SMEM((k_wgrad3x3_tc<128, 1, 64>), (WgCfg<128, 1, 64>::kSmem));
  N2F_SMEM((k_wgrad3x3_tc<128, 2, 32>), (WgCfg<128, 2, 32>::kSmem));
  N2F_SMEM((k_wgrad3x3_tc<256, 1, 64>), (WgCfg<256, 1, 64>::kSmem));
  N2F_SMEM((k_wgrad3x3_tc<256, 2, 32>), (WgCfg<256, 2, 32>::kSmem));
#undef N2F_SMEM
  done = true;
  return N2F_OK;
}

// Launch attributes of every tcgen05 kernel: a cluster of cs CTAs, and
// programmatic dependent launch (the prologue -- barrier init, TMEM alloc,
// descriptor prefetch -- overlaps the previous kernel's tail; measured 0.7 %
// faster per epoch).
struct LaunchCfg {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  LaunchCfg(dim3 grid, int smem, int cs, cudaStream_t st) {
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreadsTc);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
  }
};

template <int BN, int HEAD>
int launch_conv_dy(const ConvTcPlan& pl, const float* bias, const void* mask, float* colsum, int epi,
                   const HeadTrainArgs& ht, const HeadValArgs& hv, cudaStream_t st) {
  LaunchCfg lc(dim3(pl.grid), DyCfg<BN>::kSmem, 2, st);
  N2F_CUDA(cudaLaunchKernelEx(&lc.cfg, k_conv3x3_dy<BN, HEAD>, pl.mx, pl.mxl, pl.mw, pl.mwl, pl.my,
                              pl.myh, pl.myl, pl.omask, pl.oscale,
                              ConvOut{pl.y, pl.yhi, pl.ylo, pl.oscale}, bias, mask, pl.mask_bits,
                              pl.mbits_out, colsum, pl.amax, pl.unscale, pl.H, pl.W, pl.C, epi, ht, hv));
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

template <int BN, int CS, int SEG>
int launch_wgrad_tc_bn(const WgradTcPlan& pl, float* part, cudaStream_t st) {
  LaunchCfg lc(dim3(pl.gridx, pl.nsplit), WgCfg<BN, CS, SEG>::kSmem, CS, st);
  N2F_CUDA(cudaLaunchKernelEx(&lc.cfg, k_wgrad3x3_tc<BN, CS, SEG>, pl.mx, pl.mxl, pl.mg, pl.mgl,
                              part, pl.unscale, pl.H, pl.W, pl.C, pl.nsplit, pl.xblk));
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

// CTA pairs for the wide wgrads (one 4-D activation box per stage and an even
// split of the gradient channels)
int wgrad_cs(int cin, int cout) { return (cin % 128 == 0 && cout >= 128) ? 2 : 1; }

// DyCfg<N>::kEpiCols on the host (the TMA-store box must match the staging slice)
int dy_epi_cols(int N) {
  switch (N) {
    case 32: return DyCfg<32>::kEpiCols;
    case 64: return DyCfg<64>::kEpiCols;
    case 128: return DyCfg<128>::kEpiCols;
    default: return DyCfg<256>::kEpiCols;
  }
}

}  // namespace

bool tc_supported(int cin, int cout) {
  return cin % 32 == 0 && (cout == 32 || cout == 64 || cout == 128 || cout == 256);
}

// A conv plan: the dy-stage CTA-pair kernel over 32 x 8 pixel pair tiles,
// persistent grid (one CTA pair per SM, two for N <= kDy2SmMaxN).
int conv_tc_plan(ConvTcPlan* pl, const TcOperand& x, const TcOperand& w, int H, int W, int C, int N) {
  if (!tc_supported(C, N)) return fail(N2F_ERR_ARG, "conv_tc_plan: C=%d N=%d", C, N);
  N2F_TRY(set_attrs_once());  // outside any stream capture
  pl->H = H;
  pl->W = W;
  pl->C = C;
  pl->N = N;
  pl->unscale = ldexpf(1.f, -(x.exp + w.exp));
  pl->amax = nullptr;
  const int units = ((W + 31) / 32) * ((H + 7) / 8);
  const int max_units = (N <= kDy2SmMaxN ? 2 : 1) * sm_count() / 2;  // DyCfg<N>::kPerSm
  pl->grid = 2 * (units < max_units ? units : max_units);
  pl->tiles = 2 * units;
  N2F_TRY(map_act_yx(&pl->mx, x.hi, C, W, H, 32, 8, 18));
  N2F_TRY(map_act_yx(&pl->mxl, x.lo, C, W, H, 32, 8, 18));
  N2F_TRY(map_w_taps(&pl->mw, w.hi, C, N, 32, N / 2));
  N2F_TRY(map_w_taps(&pl->mwl, w.lo, C, N, 32, N / 2));
  return N2F_OK;
}

int conv_tc_tiles(int H, int W) { return 2 * ((W + 31) / 32) * ((H + 7) / 8); }

// Output tensor maps of a conv plan: NHWC [H][W][N] viewed as (N, H, W), box
// {EC channels, 8 y, 4 x} = one accumulate warp's staging slice.
int conv_tc_plan_out(ConvTcPlan* pl, float* y, void* yhi, void* ylo, float oscale) {
  const int ec = dy_epi_cols(pl->N);
  auto sw_for = [](int row_bytes) {
    return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
           : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
           : (row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE);
  };
  pl->omask = 0;
  pl->oscale = oscale;
  pl->mbits_out = nullptr;
  pl->mask_bits = 0;
  pl->y = y;
  pl->yhi = yhi;
  pl->ylo = ylo;
  // staged [x][y][channels] (row = lane: conflict-free swizzle)
  auto omap = [&](CUtensorMap* m, void* p, bool half) -> int {
    return map_out_yx(m, p, half, pl->N, pl->W, pl->H, ec, sw_for(ec * (half ? 2 : 4)));
  };
  if (y) {
    N2F_TRY(omap(&pl->my, y, false));
    pl->omask |= kOutY;
  }
  if (yhi) {
    N2F_TRY(omap(&pl->myh, yhi, true));
    pl->omask |= kOutHi;
  }
  if (ylo) {
    N2F_TRY(omap(&pl->myl, ylo, true));
    pl->omask |= kOutLo;
  }
  return N2F_OK;
}

int conv_tc_plan_maskbits(ConvTcPlan* pl, uint32_t* mbits_out, int mask_bits_in) {
  if ((mbits_out || mask_bits_in) && pl->N < 32)
    return fail(N2F_ERR_ARG, "bit-packed ReLU masks need N >= 32, N=%d", pl->N);
  pl->mbits_out = mbits_out;
  pl->mask_bits = mask_bits_in;
  return N2F_OK;
}

int conv_tc_plan_range(ConvTcPlan* pl, unsigned* amax) {
  pl->amax = amax;
  return N2F_OK;
}

int conv_tc_launch_head_train(const ConvTcPlan& pl, const float* bias, float* colsum,
                              const HeadTrainArgs& ht, cudaStream_t st) {
  if (pl.N != 256 || !(pl.omask & kOutHi) || !(pl.omask & kOutLo))
    return fail(N2F_ERR_ARG, "fused training head needs the plan of L8 with a pair output");
  return launch_conv_dy<256, 1>(pl, bias, nullptr, colsum, kEpiBiasRelu, ht, HeadValArgs{}, st);
}

int conv_tc_launch_head_val(const ConvTcPlan& pl, const float* bias, const HeadValArgs& hv,
                            cudaStream_t st) {
  if (pl.N != 256) return fail(N2F_ERR_ARG, "fused validation head needs the plan of L8");
  return launch_conv_dy<256, 2>(pl, bias, nullptr, nullptr, kEpiBiasRelu, HeadTrainArgs{}, hv, st);
}

int conv_tc_launch(const ConvTcPlan& pl, const float* bias, const void* mask, float* colsum, int epi,
                   cudaStream_t st) {
  const HeadTrainArgs ht{};
  const HeadValArgs hv{};
  switch (pl.N) {
    case 32: return launch_conv_dy<32, 0>(pl, bias, mask, colsum, epi, ht, hv, st);
    case 64: return launch_conv_dy<64, 0>(pl, bias, mask, colsum, epi, ht, hv, st);
    case 128: return launch_conv_dy<128, 0>(pl, bias, mask, colsum, epi, ht, hv, st);
    case 256: return launch_conv_dy<256, 0>(pl, bias, mask, colsum, epi, ht, hv, st);
  }
  return fail(N2F_ERR_ARG, "conv_tc_launch: N=%d", pl.N);
}

int wgrad_tc_nsplit(int cin, int cout, int H, int W) {
  const int cs = wgrad_cs(cin, cout);
  const int mblocks = (9 * cin + 127) / 128;
  const int gridx = cs * ((mblocks + cs - 1) / cs);
  const int nseg = ((W + kSegW - 1) / kSegW) * H;
  // narrow layers (N <= 64) fit two CTAs per SM: twice the splits keeps two
  // TMA pipelines in flight per SM (their short MMA stages are latency-bound)
  const int per_sm = cout <= 64 ? N2F_WG_PER_SM_NARROW : 1;
  int n = per_sm * sm_count() / gridx;
  if (n < 1) n = 1;
  if (n > nseg) n = nseg;
  return n;
}

int wgrad_tc_plan(WgradTcPlan* pl, const TcOperand& x, const TcOperand& g, int H, int W, int C,
                  int N, int nsplit) {
  if (!tc_supported(C, N)) return fail(N2F_ERR_ARG, "wgrad_tc_plan: C=%d N=%d", C, N);
  N2F_TRY(set_attrs_once());
  pl->H = H;
  pl->W = W;
  pl->C = C;
  pl->N = N;
  pl->mblocks = (9 * C + 127) / 128;
  pl->cs = wgrad_cs(C, N);
  pl->gridx = pl->cs * ((pl->mblocks + pl->cs - 1) / pl->cs);
  pl->nsplit = nsplit;
  pl->unscale = ldexpf(1.f, -(x.exp + g.exp));
  // one TMA per operand part and stage: the 4 activation blocks of an M block
  // share a tap when C % 128 == 0 (else one box per block), the gradient's
  // N / 32 blocks always come as one box
  pl->xblk = C % 128 == 0;
  // pixels per K stage: CTA pairs 32; single CTAs 64, or 128 for C = 32 with
  // N <= 64 (their 4 per-tap activation boxes per part make them TMA-issue
  // bound: 128-pixel stages halve the TMA instructions per pixel)
  pl->seg = pl->cs == 2 ? kSegW : (C == 32 && N <= 64) ? 128 : 64;
  const int bpt = pl->xblk ? 4 : C / 32;  // activation blocks per box (one tap)
  N2F_TRY(map_act_blk(&pl->mx, x.hi, C, W, H, pl->seg, bpt));
  N2F_TRY(map_act_blk(&pl->mxl, x.lo, C, W, H, pl->seg, bpt));
  N2F_TRY(map_act_blk(&pl->mg, g.hi, N, W, H, pl->seg, N / 32 / pl->cs));
  N2F_TRY(map_act_blk(&pl->mgl, g.lo, N, W, H, pl->seg, N / 32 / pl->cs));
  return N2F_OK;
}

int wgrad_tc_launch(const WgradTcPlan& pl, float* part, cudaStream_t st) {
  if (pl.cs == 2) {
    switch (pl.N) {
      case 128: return launch_wgrad_tc_bn<128, 2, 32>(pl, part, st);
      case 256: return launch_wgrad_tc_bn<256, 2, 32>(pl, part, st);
    }
  } else if (pl.seg == 128) {
    switch (pl.N) {
      case 32: return launch_wgrad_tc_bn<32, 1, 128>(pl, part, st);
      case 64: return launch_wgrad_tc_bn<64, 1, 128>(pl, part, st);
    }
  } else {
    switch (pl.N) {
      case 32: return launch_wgrad_tc_bn<32, 1, 64>(pl, part, st);
      case 64: return launch_wgrad_tc_bn<64, 1, 64>(pl, part, st);
      case 128: return launch_wgrad_tc_bn<128, 1, 64>(pl, part, st);
      case 256: return launch_wgrad_tc_bn<256, 1, 64>(pl, part, st);
    }
  }
  return fail(N2F_ERR_ARG, "wgrad_tc_launch: N=%d cs=%d seg=%d", pl.N, pl.cs, pl.seg);
}

// fp16 operand pair of an fp32 tensor (init / set_params refresh of the
// weights; parity entry points); folds max |x * 2^exp2| into amax (or null).
int split_f16(const float* x, void* hi, void* lo, int exp2, int64_t n, cudaStream_t st,
              unsigned* amax) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_split_f16<<<(unsigned)blocks, 256, 0, st>>>(x, reinterpret_cast<__half*>(hi),
                                                reinterpret_cast<__half*>(lo), ldexpf(1.f, exp2), n,
                                                amax);
  N2F_LAUNCH_CHECK();
  return N2F_OK;
}

}  // namespace n2f
