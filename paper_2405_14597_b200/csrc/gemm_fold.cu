// K3 prefill variant — integer scale FOLDED into the weight expansion.
//
// Reference: gemm_integer_scale (gemm.cpp:205-262), paper Eq. 2:
//   acc = sum_g k_g * P_g,  P_g = sum_{k in g} x_k * w_k  (int32, exact).
// Because k_g is an integer, sum_g k_g * P_g = sum_k x_k * (k_g(k) * w_k): when
// every k_g <= 16, k_g * w lies in [-128, 112] and fits the int8 tensor-core
// operand, so the transform warps expand int4 -> (k_g * w) int8 and the tensor
// core accumulates the whole K reduction — the scaled int32 accumulator — in
// TMEM, with no per-group epilogue at all (SURVEY H1 "k <= 16 fold band";
// llama_like weights at alpha = 1024 have k_g in [1, 15]). The result is
// bit-identical to the per-group kernel: every partial sum is bounded by the
// static overflow bound (analysis.cpp:24-59), which callers gate on.
//
// Tile: 128 output channels (UMMA M) x 192 tokens (UMMA N), persistent CTAs.
// TMEM: A ring 4 x 32 columns (expanded weights) + 2 x 192-column int32
// accumulators, so the epilogue of tile t overlaps the MMAs of tile t+1.
//
//   warp 0      producer : per 128-K block one bulk copy of the 8 KiB packed
//                          weight block + 512 B of k_g, and a TMA (SWIZZLE_128B)
//                          of the 192 x 128 int8 activation tile.
//   warp 1      MMA      : 4 x tcgen05.mma.kind::i8 (K = 32) per block into D[t & 1].
//   warp 2      TMEM allocator.
//   warps 4-11  transform: two warpgroups alternate blocks; thread r owns channel r:
//                          nibble -> fp16 lane (exponent-bias trick) -> one HFMA2
//                          computes 1536 + k*c exactly -> low byte = k*c.
//   warps 12-15 epilogue : tcgen05.ld of D, out = float((double(acc) / 2^e) * s_a).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "fold.cuh"
#include "layout.cuh"

namespace isb {
namespace {

constexpr int kFMT = 192;                     // tokens per tile (UMMA N)
constexpr int kFXBytes = kFMT * 128;          // 24 KiB activation tile per block
constexpr int kFStage = kBlockBytes + kFXBytes;  // 32 KiB (W first, X 1024-aligned)
constexpr int kFNA = 4;                       // TMEM A ring
constexpr int kFXformWG = 2;
constexpr int kFThreads = 128 + 128 * kFXformWG + 128;
constexpr int kFStages = 6;
constexpr int kFSmem = 1024 + kFStages * (kFStage + kTileN * 4) + 2 * kFMT * 8 + 512;
static_assert(kFSmem <= 227 * 1024, "smem");
constexpr uint32_t kFDCol = kFNA * 32;        // D buffers start after the A ring

struct FoldParams {
  const uint8_t* packed;  // [n_tiles][kblocks][8 KiB]
  const int32_t* kscale;  // [n_tiles][G][128]
  const double* sa;       // [M]
  void* out;              // [M][N]
  int M, N, G, gb, kblocks, m_tiles, tiles, out_dtype;
  double inv_amp;
  int dbg;  // measurement knobs (isb_debug_set_flags): 1 skip the fold ALU, 2 skip A stores
};

__device__ __forceinline__ void store_out_f(void* out, int dtype, int64_t idx, float f) {
  if (dtype == ISB_F32)
    static_cast<float*>(out)[idx] = f;
  else if (dtype == ISB_BF16)
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
  else
    static_cast<__half*>(out)[idx] = __float2half_rn(f);
}

__global__ void __launch_bounds__(kFThreads, 1)
    gemm_w4a8_fold(const __grid_constant__ CUtensorMap x_map, const FoldParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_sc = smem + kFStages * kFStage;                        // [stage][128] k_g
  double* sa_s = reinterpret_cast<double*>(smem_sc + kFStages * kTileN * 4);  // [2][MT]
  uint64_t* full = reinterpret_cast<uint64_t*>(sa_s + 2 * kFMT);
  uint64_t* empty = full + kFStages;
  uint64_t* a_full = empty + kFStages;
  uint64_t* a_empty = a_full + kFNA;
  uint64_t* d_full = a_empty + kFNA;
  uint64_t* d_empty = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int ntiles = static_cast<int>(blockIdx.x) < p.tiles
                         ? (p.tiles - static_cast<int>(blockIdx.x) + gridDim.x - 1) / gridDim.x
                         : 0;
  const int total = ntiles * p.kblocks;  // (tile, block) steps of this CTA

  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&x_map);
    for (int i = 0; i < kFStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1 + 4);
    }
    for (int i = 0; i < kFNA; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) pdl_launch_dependents();

  auto tile_of = [&](int it, int& nt, int& mt) {
    const int t = blockIdx.x + it * gridDim.x;
    nt = t / p.m_tiles;
    mt = t % p.m_tiles;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      auto load_static = [&](int j, int stage) {
        int nt, mt;
        tile_of(j / p.kblocks, nt, mt);
        const int kb = j % p.kblocks;
        mbar_arrive_expect_tx(&full[stage], kFStage + kTileN * 4);
        bulk_load(smem + stage * kFStage,
                  p.packed + (static_cast<int64_t>(nt) * p.kblocks + kb) * kBlockBytes,
                  kBlockBytes, &full[stage]);
        bulk_load(smem_sc + stage * kTileN * 4,
                  p.kscale + (static_cast<int64_t>(nt) * p.G + kb / p.gb) * kTileN, kTileN * 4,
                  &full[stage]);
      };
      const int pre = min(total, kFStages);
      for (int j = 0; j < pre; ++j) load_static(j, j);
      pdl_wait();
      for (int j = 0; j < total; ++j) {
        const int stage = j % kFStages;
        if (j >= pre) {
          mbar_wait(&empty[stage], ((j / kFStages) & 1) ^ 1);
          load_static(j, stage);
        }
        int nt, mt;
        tile_of(j / p.kblocks, nt, mt);
        tma_load_2d(smem + stage * kFStage + kBlockBytes, &x_map, &full[stage],
                    (j % p.kblocks) * kBlockK, mt * kFMT);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = make_idesc_i8(128, kFMT);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t s_base = smem_u32(smem);
    int j = 0;
    for (int it = 0; it < ntiles; ++it) {
      const int ds = it & 1;
      mbar_wait(&d_empty[ds], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tbase + kFDCol + ds * kFMT;
      for (int kb = 0; kb < p.kblocks; ++kb, ++j) {
        const int stage = j % kFStages, as = j % kFNA;
        mbar_wait(&a_full[as], (j / kFNA) & 1);  // implies full[stage] (transform saw it)
        tc_fence_after();
        const uint64_t bdesc = make_sw128_kmajor_desc(s_base + stage * kFStage + kBlockBytes);
        const uint32_t a_tmem = tbase + as * 32;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          mma_i8_ts_warp(d_tmem, a_tmem + c * 8, bdesc + static_cast<uint64_t>(c * 2), idesc,
                         (kb > 0 || c > 0) ? 1u : 0u);
        mma_commit_warp(&empty[stage]);
        mma_commit_warp(&a_empty[as]);
      }
      mma_commit_warp(&d_full[ds]);
    }
  } else if (warp >= 4 && warp < 4 + 4 * kFXformWG) {
    // ---------------------------------------------------------------- transform
    const int xw = static_cast<int>(warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;  // output channel == TMEM lane
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t w_base = smem_u32(smem) + r * 16;
    const uint32_t sc_base = smem_u32(smem_sc) + r * 4;
    for (int j = xw; j < total; j += kFXformWG) {
      const int stage = j % kFStages, as = j % kFNA;
      mbar_wait(&full[stage], (j / kFStages) & 1);
      uint4 q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c] = ld_shared_v4(w_base + stage * kFStage + c * (kTileN * 16));
      const int32_t k = static_cast<int32_t>(ld_shared_u32(sc_base + stage * kTileN * 4));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the async refill
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      const float kf = static_cast<float>(k);
      const uint32_t k1 = half2_bits(kf);
      const uint32_t k16 = half2_bits(kf * 0.0625f);
      const uint32_t cA = half2_bits(1536.0f - 1032.0f * kf);
      const uint32_t cB = half2_bits(1536.0f - 72.0f * kf);
      uint32_t a[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t w4[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
        for (int w = 0; w < 4; ++w) fold_word(w4[w], k1, k16, cA, cB, a[c * 8 + 2 * w], a[c * 8 + 2 * w + 1]);
      }
      mbar_wait(&a_empty[as], ((j / kFNA) & 1) ^ 1);
      tc_fence_after();
      tmem_st_x32(tmem_base + lane_base + as * 32, a);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[as]);
    }
  } else if (warp >= 4 + 4 * kFXformWG) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t ew = warp - (4 + 4 * kFXformWG);
    const uint32_t t128 = ew * 32 + lane;
    const uint32_t r = t128;                      // TMEM lane == channel in tile
    const uint32_t lane_base = (ew * 32) << 16;
    pdl_wait();  // sa / out may be touched by the preceding grid
    auto sa_prefetch = [&](int it) {
      if (it < ntiles) {
        int nt, mt;
        tile_of(it, nt, mt);
        for (int t = t128; t < kFMT; t += 128) {
          const int64_t m = static_cast<int64_t>(mt) * kFMT + t;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                           smem_u32(sa_s + (it & 1) * kFMT + t)),
                       "l"(p.sa + (m < p.M ? m : 0)), "r"(m < p.M ? 8 : 0)
                       : "memory");
        }
      }
      cp_async_commit();
    };
    sa_prefetch(0);
    for (int it = 0; it < ntiles; ++it) {
      int nt, mt;
      tile_of(it, nt, mt);
      const int ds = it & 1;
      sa_prefetch(it + 1);
      cp_async_wait<1>();
      named_bar_sync(1, 128);  // sa_s[it & 1] complete for all epilogue threads
      const double* sa_t = sa_s + (it & 1) * kFMT;
      mbar_wait(&d_full[ds], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + lane_base + kFDCol + ds * kFMT;
      const int64_t n = static_cast<int64_t>(nt) * kTileN + r;
      const int64_t m0 = static_cast<int64_t>(mt) * kFMT;
#pragma unroll 1
      for (int cc = 0; cc < kFMT; cc += 32) {
        uint32_t v[32];
        tmem_ld_x16_(taddr + cc, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld_x16_(taddr + cc + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        tmem_wait_ld();
        if (cc + 32 >= kFMT) {  // all of D[ds] read: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[ds]);
        }
        if (n < p.N) {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int64_t m = m0 + cc + t;
            if (m < p.M) {
              if (p.out_dtype == ISB_I32) {  // raw acc (row-parallel TP)
                static_cast<int32_t*>(p.out)[m * p.N + n] = static_cast<int32_t>(v[t]);
              } else {
                const double o = __dmul_rn(
                    static_cast<double>(static_cast<int32_t>(v[t])) * p.inv_amp, sa_t[cc + t]);
                store_out_f(p.out, p.out_dtype, m * p.N + n, __double2float_rn(o));
              }
            }
          }
        }
      }
      named_bar_sync(1, 128);  // done with sa_s[it & 1] before it is refilled
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}


// ============================================================================
// SS variant: the transform warps write the folded int8 weights into a shared-
// memory ring in the canonical SWIZZLE_128B K-major layout (row = channel,
// 16-byte chunk c of row r at r*128 + ((c ^ (r & 7)) * 16)) and the MMA reads
// both operands from shared memory (tcgen05.mma kind::i8, SS form), so TMEM only
// holds the two int32 accumulators and the tile can be 256 tokens wide.
template <int MT, int NA = 2, int SX = 4, int SW = 6, int EW = 2>
struct FoldSS {
  static constexpr int kXBytes = MT * 128;
  static constexpr int kNA = NA;             // folded-weight ring (16 KiB each)
  static constexpr int kABytes = 128 * 128;
  static constexpr int kSX = SX;             // activation ring (consumed by the MMA)
  static constexpr int kSW = SW;             // packed-weight ring (consumed by the transform)
  static constexpr int kSmem = 1024 + NA * kABytes + SX * kXBytes + SW * (kBlockBytes + kTileN * 4) +
                               2 * MT * 8 + 1024;
  static constexpr int kEW = EW;             // epilogue warpgroups (each owns MT/EW tokens)
  static constexpr int kThreads = 128 + 128 * kFXformWG + 128 * kEW;
  static_assert(kXBytes % 1024 == 0, "SW128 tiles need 1 KiB alignment");
  // Each ring slot must always be served by the same transform warpgroup (slots are
  // waited on by parity, which only tracks a lead of one phase).
  static_assert(NA % kFXformWG == 0 && SW % kFXformWG == 0, "ring slots per warpgroup");
  static_assert(kSmem <= 227 * 1024, "smem");
  static_assert(2 * MT <= 512, "TMEM");
};

// Two producer threads keep separate rings: the packed weights (+ k_g) run ahead
// of the transform warps, the activation tiles are recycled by the MMA alone, so
// the transform's latency is not part of the activation ring's turnaround.
template <int MT, int NA, int SX, int SW, int EW>
__global__ void __launch_bounds__(FoldSS<MT, NA, SX, SW, EW>::kThreads, 1)
    gemm_w4a8_fold_ss(const __grid_constant__ CUtensorMap x_map, const FoldParams p) {
  using F = FoldSS<MT, NA, SX, SW, EW>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;                                   // [NA][128 x 128] folded int8
  uint8_t* smem_x = smem_a + NA * F::kABytes;               // [SX][MT x 128] activations
  uint8_t* smem_w = smem_x + SX * F::kXBytes;               // [SW][8 KiB] packed weights
  uint8_t* smem_sc = smem_w + SW * kBlockBytes;             // [SW][128] k_g
  double* sa_s = reinterpret_cast<double*>(smem_sc + SW * kTileN * 4);  // [2][MT]
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sa_s + 2 * MT);
  uint64_t* wempty = wfull + SW;
  uint64_t* xfull = wempty + SW;
  uint64_t* xempty = xfull + SX;
  uint64_t* a_full = xempty + SX;
  uint64_t* a_empty = a_full + NA;
  uint64_t* d_full = a_empty + NA;
  uint64_t* d_empty = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int ntiles = static_cast<int>(blockIdx.x) < p.tiles
                         ? (p.tiles - static_cast<int>(blockIdx.x) + gridDim.x - 1) / gridDim.x
                         : 0;
  const int total = ntiles * p.kblocks;

  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&x_map);
    for (int i = 0; i < SW; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], 4);
    }
    for (int i = 0; i < SX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4 * F::kEW);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * MT <= 256 ? 256 : 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) pdl_launch_dependents();

  auto tile_of = [&](int it, int& nt, int& mt) {
    const int t = blockIdx.x + it * gridDim.x;
    nt = t / p.m_tiles;
    mt = t % p.m_tiles;
  };

  if (warp == 0) {
    // ------------------------------------------------ producer: packed weights + k_g
    if (elect_one()) {
      for (int j = 0; j < total; ++j) {
        const int s = j % SW;
        mbar_wait(&wempty[s], ((j / SW) & 1) ^ 1);
        int nt, mt;
        tile_of(j / p.kblocks, nt, mt);
        const int kb = j % p.kblocks;
        mbar_arrive_expect_tx(&wfull[s], kBlockBytes + kTileN * 4);
        bulk_load(smem_w + s * kBlockBytes,
                  p.packed + (static_cast<int64_t>(nt) * p.kblocks + kb) * kBlockBytes,
                  kBlockBytes, &wfull[s]);
        bulk_load(smem_sc + s * kTileN * 4,
                  p.kscale + (static_cast<int64_t>(nt) * p.G + kb / p.gb) * kTileN, kTileN * 4,
                  &wfull[s]);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ------------------------------------------------ producer: activation tiles
    if (elect_one()) {
      pdl_wait();
      for (int j = 0; j < total; ++j) {
        const int s = j % SX;
        mbar_wait(&xempty[s], ((j / SX) & 1) ^ 1);
        int nt, mt;
        tile_of(j / p.kblocks, nt, mt);
        mbar_arrive_expect_tx(&xfull[s], F::kXBytes);
        tma_load_2d(smem_x + s * F::kXBytes, &x_map, &xfull[s], (j % p.kblocks) * kBlockK, mt * MT);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_i8(128, MT);
      int j = 0;
      for (int it = 0; it < ntiles; ++it) {
        const int ds = it & 1;
        mbar_wait(&d_empty[ds], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + ds * MT;
        for (int kb = 0; kb < p.kblocks; ++kb, ++j) {
          const int xs = j % SX, as = j % NA;
          mbar_wait(&a_full[as], (j / NA) & 1);
          mbar_wait(&xfull[xs], (j / SX) & 1);
          tc_fence_after();
          const uint64_t adesc = make_sw128_kmajor_desc(smem_u32(smem_a + as * F::kABytes));
          const uint64_t bdesc = make_sw128_kmajor_desc(smem_u32(smem_x + xs * F::kXBytes));
#pragma unroll
          for (int c = 0; c < 4; ++c)
            mma_i8_ss(d_tmem, adesc + static_cast<uint64_t>(c * 2), bdesc + static_cast<uint64_t>(c * 2),
                      idesc, (kb > 0 || c > 0) ? 1u : 0u);
          mma_commit(&xempty[xs]);
          mma_commit(&a_empty[as]);
        }
        mma_commit(&d_full[ds]);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + 4 * kFXformWG) {
    // ---------------------------------------------------------------- transform
    const int xw = static_cast<int>(warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;  // output channel == A row
    const uint32_t w_base = smem_u32(smem_w) + r * 16;
    const uint32_t sc_base = smem_u32(smem_sc) + r * 4;
    const uint32_t a_row = smem_u32(smem_a) + r * 128;
    for (int j = xw; j < total; j += kFXformWG) {
      const int s = j % SW, as = j % NA;
      mbar_wait(&wfull[s], (j / SW) & 1);
      uint4 q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c] = ld_shared_v4(w_base + s * kBlockBytes + c * (kTileN * 16));
      const int32_t k = static_cast<int32_t>(ld_shared_u32(sc_base + s * kTileN * 4));
      const float kf = static_cast<float>(k);
      const uint32_t k1 = half2_bits(kf);
      const uint32_t k16 = half2_bits(kf * 0.0625f);
      const uint32_t cA = half2_bits(1536.0f - 1032.0f * kf);
      const uint32_t cB = half2_bits(1536.0f - 72.0f * kf);
      uint32_t a[32];
      if (p.dbg & 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t w4[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
          for (int w = 0; w < 4; ++w) { a[c * 8 + 2 * w] = w4[w] ^ k1; a[c * 8 + 2 * w + 1] = w4[w]; }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t w4[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
          for (int w = 0; w < 4; ++w) fold_word(w4[w], k1, k16, cA, cB, a[c * 8 + 2 * w], a[c * 8 + 2 * w + 1]);
        }
      }
      // Release the packed slot only once its values have been consumed: the refill
      // is an async-proxy bulk copy that must not overtake these shared loads.
      // generic-proxy reads of the slot ordered before the async-proxy refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&wempty[s]);
      mbar_wait(&a_empty[as], ((j / NA) & 1) ^ 1);
      const uint32_t dst = a_row + as * F::kABytes;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        if (!(p.dbg & 2))
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + ((ch ^ (r & 7)) * 16)),
                     "r"(a[4 * ch]), "r"(a[4 * ch + 1]), "r"(a[4 * ch + 2]), "r"(a[4 * ch + 3])
                     : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
      named_bar_sync(2 + xw, 128);  // the whole warpgroup's rows are written and fenced
      if (warp % 4 == 0 && lane == 0) mbar_arrive(&a_full[as]);
    }
  } else if (warp >= 4 + 4 * kFXformWG) {
    // ---------------------------------------------------------------- epilogue
    // kEW warpgroups; warpgroup g finalises tokens [g*MT/kEW, (g+1)*MT/kEW) of the
    // tile, warp q of it the TMEM lanes (channels) [32q, 32q+32). Eq. 2 per output:
    // float(double(acc) * (2^-e * s_a)) — 2^-e * s_a is exact, so this is the
    // reference's (acc / 2^e) * s_a with one DMUL.
    constexpr int kEW = F::kEW;
    constexpr int kCols = MT / kEW;
    const uint32_t ew = warp - (4 + 4 * kFXformWG);
    const uint32_t q = ew % 4, g = ew / 4;
    const int te = static_cast<int>(ew * 32 + lane);
    const uint32_t r = q * 32 + lane;
    const uint32_t lane_base = (q * 32) << 16;
    pdl_wait();
    auto sa_prefetch = [&](int it) {
      if (it < ntiles) {
        int nt, mt;
        tile_of(it, nt, mt);
        for (int t = te; t < MT; t += 128 * kEW) {
          const int64_t m = static_cast<int64_t>(mt) * MT + t;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                           smem_u32(sa_s + (it & 1) * MT + t)),
                       "l"(p.sa + (m < p.M ? m : 0)), "r"(m < p.M ? 8 : 0)
                       : "memory");
        }
      }
      cp_async_commit();
    };
    sa_prefetch(0);
    for (int it = 0; it < ntiles; ++it) {
      int nt, mt;
      tile_of(it, nt, mt);
      const int ds = it & 1;
      sa_prefetch(it + 1);
      cp_async_wait<1>();
      // s_a * 2^-e (exact: a power-of-two scaling), once per token
      for (int t = te; t < MT; t += 128 * kEW) sa_s[(it & 1) * MT + t] *= p.inv_amp;
      named_bar_sync(1, 128 * kEW);
      const double* sa_t = sa_s + (it & 1) * MT;
      mbar_wait(&d_full[ds], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + lane_base + ds * MT;
      const int64_t n = static_cast<int64_t>(nt) * kTileN + r;
      const int64_t m0 = static_cast<int64_t>(mt) * MT;
      const bool n_ok = n < p.N && !(p.dbg & 4);
#pragma unroll 1
      for (int cc = g * kCols; cc < (g + 1) * kCols; cc += 32) {
        uint32_t v[32];
        tmem_ld_x16_(taddr + cc, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld_x16_(taddr + cc + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        tmem_wait_ld();
        if (cc + 32 >= (g + 1) * kCols) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[ds]);
        }
        if (!n_ok) continue;
        const int64_t mb = m0 + cc;
        const int tv = p.M - mb < 32 ? static_cast<int>(p.M - mb) : 32;  // valid tokens here
        if (p.dbg & 8) {  // measurement: conversions without the stores
          uint32_t x = 0;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const double o = static_cast<double>(static_cast<int32_t>(v[t])) * sa_t[cc + t];
            x ^= __bfloat16_as_ushort(__float2bfloat16_rn(__double2float_rn(o)));
          }
          if (x == 0x12345u) static_cast<uint32_t*>(p.out)[0] = x;
        } else if (p.out_dtype == ISB_BF16 && tv == 32 && (p.dbg & 16)) {  // A/B: previous form
          __nv_bfloat16* po = static_cast<__nv_bfloat16*>(p.out) + mb * p.N + n;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const double o = static_cast<double>(static_cast<int32_t>(v[t])) * sa_t[cc + t];
            const uint16_t b = __bfloat16_as_ushort(__float2bfloat16_rn(__double2float_rn(o)));
            asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(po + static_cast<int64_t>(t) * p.N), "h"(b)
                         : "memory");
          }
        } else if ((p.out_dtype == ISB_BF16 || p.out_dtype == ISB_F16) && tv == 32) {
          // Eq. 2 (gemm.cpp:252) for 32 tokens: (double)acc via the 2^52 + 2^31 bias (a DADD
          // on the FP64 pipe instead of an I2F.F64 conversion), one DMUL, one F2F.F32.F64;
          // all 32 chains independent (no store in between), then lane pairs exchange one
          // value so each lane stores two adjacent channels of one token as a 32-bit word.
          float f[32];
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const double d = __hiloint2double(0x43300000, static_cast<int>(v[t] ^ 0x80000000u)) -
                             4503601774854144.0;
            f[t] = __double2float_rn(d * sa_t[cc + t]);
          }
          const bool pairs = (p.N % 2 == 0) && static_cast<int64_t>(nt) * kTileN + q * 32 + 32 <= p.N;
          if (pairs) {
            // even lane: token t, channels (n, n+1); odd lane: token t+1, channels (n-1, n)
            const bool odd = lane & 1;
            uint32_t* po = reinterpret_cast<uint32_t*>(static_cast<uint16_t*>(p.out) +
                                                       (mb + (odd ? 1 : 0)) * p.N + (n - (odd ? 1 : 0)));
#pragma unroll
            for (int t = 0; t < 32; t += 2) {
              const float x = __shfl_xor_sync(0xffffffffu, odd ? f[t] : f[t + 1], 1);
              const float lo = odd ? x : f[t], hi = odd ? f[t + 1] : x;
              uint32_t w;
              if (p.out_dtype == ISB_BF16) {
                const __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
                w = *reinterpret_cast<const uint32_t*>(&b);
              } else {
                const __half2 b = __floats2half2_rn(lo, hi);
                w = *reinterpret_cast<const uint32_t*>(&b);
              }
              // streaming store: written once, must not evict the L2-resident activations
              asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(po + static_cast<int64_t>(t) * (p.N / 2)), "r"(w));
            }
          } else {
            uint16_t* po = static_cast<uint16_t*>(p.out) + mb * p.N + n;
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const uint16_t b = p.out_dtype == ISB_BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(f[t]))
                                                         : __half_as_ushort(__float2half_rn(f[t]));
              asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(po + static_cast<int64_t>(t) * p.N), "h"(b));
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            if (t < tv) {
              const int64_t idx = (mb + t) * p.N + n;
              if (p.out_dtype == ISB_I32) {
                static_cast<int32_t*>(p.out)[idx] = static_cast<int32_t>(v[t]);
              } else {
                const double o = static_cast<double>(static_cast<int32_t>(v[t])) * sa_t[cc + t];
                store_out_f(p.out, p.out_dtype, idx, __double2float_rn(o));
              }
            }
          }
        }
      }
      named_bar_sync(1, 128 * kEW);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, 2 * MT <= 256 ? 256 : 512);
}

template <int MT, int NA = 2, int SX = 4, int SW = 6, int EW = 2>
void launch_fold_ss(const int8_t* xq, int64_t m, const isb_weight& w, FoldParams prm, int num_sms,
                    cudaStream_t s) {
  using F = FoldSS<MT, NA, SX, SW, EW>;
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemm_w4a8_fold_ss<MT, NA, SX, SW, EW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    F::kSmem),
               "cudaFuncSetAttribute(fold ss smem)");
  });
  prm.m_tiles = static_cast<int>((m + MT - 1) / MT);
  prm.tiles = static_cast<int>(w.n_tiles) * prm.m_tiles;
  const CUtensorMap map = make_x_map(xq, m, w.k, MT);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(prm.tiles, num_sms));
  cfg.blockDim = dim3(F::kThreads);
  cfg.dynamicSmemBytes = F::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_fold_ss<MT, NA, SX, SW, EW>, map, prm), "gemm_w4a8_fold_ss launch");
  count_launch();
}

// ============================================================================
// 2-SM variant (tcgen05.mma.cta_group::2). A CTA pair computes 256 channels
// (each CTA its own 128: weights expanded into its own TMEM) x 192 tokens; each
// CTA TMA-loads only HALF of the activation tile (96 tokens) into its own smem
// and the pair's MMA reads both halves. Per SM and 128-K block that is 8 KiB of
// weights + 12 KiB of activations for 3.1 M MACs — 151 MAC/B instead of 96,
// aimed at the per-SM L2->SMEM ingest bound of the 1-SM kernel. The leader
// (cluster rank 0) issues the MMAs; commits are multicast to both CTAs; the
// peer's transform and epilogue arrive on the leader's barriers over DSMEM.
constexpr int k2MT = 192;                        // tokens per pair tile (UMMA N)
constexpr int k2XH = (k2MT / 2) * 128;           // 12 KiB activation half per CTA
constexpr int k2Stage = kBlockBytes + k2XH;      // [W 8 KiB][X half 12 KiB]
constexpr int k2Stages = 8;
constexpr int k2NA = 4;
constexpr int k2Threads = 128 + 128 * 2 + 128;
constexpr int k2Smem = 1024 + k2Stages * (k2Stage + kTileN * 4) + 2 * k2MT * 8 + 512;
static_assert(k2Smem <= 227 * 1024, "smem");
static_assert(k2Stage % 1024 == 0, "SW128 activation tiles need 1 KiB alignment");
constexpr uint32_t k2DCol = k2NA * 32;
static_assert(k2DCol + 2 * k2MT <= 512, "TMEM");

struct Fold2Params {
  const uint8_t* packed;
  const int32_t* kscale;
  const double* sa;
  void* out;
  int M, N, G, gb, kblocks, m_tiles, n_tiles, units, out_dtype;
  double inv_amp;
};

__device__ __forceinline__ void arrive_on_leader(uint64_t* bar, uint32_t rank) {
  if (rank == 0)
    mbar_arrive(bar);
  else
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                     mapa_shared(smem_u32(bar), 0))
                 : "memory");
}

__device__ __forceinline__ void mma_i8_ts_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}

__device__ __forceinline__ void commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__global__ void __launch_bounds__(k2Threads, 1)
    gemm_w4a8_fold2(const __grid_constant__ CUtensorMap x_map, const Fold2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_sc = smem + k2Stages * k2Stage;                          // [stage][128] k_g
  double* sa_s = reinterpret_cast<double*>(smem_sc + k2Stages * kTileN * 4);  // [2][MT]
  uint64_t* full = reinterpret_cast<uint64_t*>(sa_s + 2 * k2MT);    // local: W + k_g
  uint64_t* xfull = full + k2Stages;        // leader: both activation halves
  uint64_t* empty = xfull + k2Stages;       // local: transform (W) + MMA commit (X)
  uint64_t* a_full = empty + k2Stages;      // leader: both CTAs' expanded weights
  uint64_t* a_empty = a_full + k2NA;        // local (multicast commit)
  uint64_t* d_full = a_empty + k2NA;        // local (multicast commit)
  uint64_t* d_empty = d_full + 2;           // leader: both CTAs drained D
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cid = static_cast<int>(blockIdx.x) / 2, ncl = static_cast<int>(gridDim.x) / 2;
  const int nunits = cid < p.units ? (p.units - cid + ncl - 1) / ncl : 0;
  const int total = nunits * p.kblocks;

  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&x_map);
    for (int i = 0; i < k2Stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&xfull[i], 1);
      mbar_init(&empty[i], 1 + 4);
    }
    for (int i = 0; i < k2NA; ++i) {
      mbar_init(&a_full[i], 8);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) pdl_launch_dependents();

  auto unit_of = [&](int it, int& np, int& mt) {
    const int u = cid + it * ncl;
    np = u / p.m_tiles;
    mt = u % p.m_tiles;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      const uint32_t xfull_leader = mapa_shared(smem_u32(xfull), 0);
      auto load_static = [&](int j, int stage) {
        int np, mt;
        unit_of(j / p.kblocks, np, mt);
        const int kb = j % p.kblocks;
        const int nt = np * 2 + static_cast<int>(rank);
        if (nt < p.n_tiles) {
          mbar_arrive_expect_tx(&full[stage], kBlockBytes + kTileN * 4);
          bulk_load(smem + stage * k2Stage,
                    p.packed + (static_cast<int64_t>(nt) * p.kblocks + kb) * kBlockBytes,
                    kBlockBytes, &full[stage]);
          bulk_load(smem_sc + stage * kTileN * 4,
                    p.kscale + (static_cast<int64_t>(nt) * p.G + kb / p.gb) * kTileN,
                    kTileN * 4, &full[stage]);
        } else {
          mbar_arrive(&full[stage]);  // no channels here: the transform writes zeros
        }
      };
      auto load_x = [&](int j, int stage) {
        int np, mt;
        unit_of(j / p.kblocks, np, mt);
        if (rank == 0) mbar_arrive_expect_tx(&xfull[stage], 2 * k2XH);  // both halves
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem + stage * k2Stage + kBlockBytes)),
            "l"(reinterpret_cast<uint64_t>(&x_map)),
            "r"(xfull_leader + static_cast<uint32_t>(stage) * 8u),
            "r"((j % p.kblocks) * kBlockK), "r"(mt * k2MT + static_cast<int>(rank) * (k2MT / 2))
            : "memory");
      };
      const int pre = min(total, k2Stages);
      for (int j = 0; j < pre; ++j) load_static(j, j);
      pdl_wait();
      for (int j = 0; j < total; ++j) {
        const int stage = j % k2Stages;
        if (j >= pre) {
          mbar_wait(&empty[stage], ((j / k2Stages) & 1) ^ 1);
          load_static(j, stage);
        }
        load_x(j, stage);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader)
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc_i8(256, k2MT);
      const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t s_base = smem_u32(smem);
      int j = 0;
      for (int it = 0; it < nunits; ++it) {
        const int ds = it & 1;
        mbar_wait(&d_empty[ds], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tbase + k2DCol + ds * k2MT;
        for (int kb = 0; kb < p.kblocks; ++kb, ++j) {
          const int stage = j % k2Stages, as = j % k2NA;
          mbar_wait(&xfull[stage], (j / k2Stages) & 1);
          mbar_wait(&a_full[as], (j / k2NA) & 1);
          tc_fence_after();
          const uint64_t bdesc = make_sw128_kmajor_desc(s_base + stage * k2Stage + kBlockBytes);
          const uint32_t a_tmem = tbase + as * 32;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            mma_i8_ts_2sm(d_tmem, a_tmem + c * 8, bdesc + static_cast<uint64_t>(c * 2), idesc,
                          (kb > 0 || c > 0) ? 1u : 0u);
          commit_2sm_mc(&empty[stage]);
          commit_2sm_mc(&a_empty[as]);
        }
        commit_2sm_mc(&d_full[ds]);
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------------------------------------------------------- transform
    const int xw = static_cast<int>(warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t w_base = smem_u32(smem) + r * 16;
    const uint32_t sc_base = smem_u32(smem_sc) + r * 4;
    for (int j = xw; j < total; j += 2) {
      const int stage = j % k2Stages, as = j % k2NA;
      int np, mt;
      unit_of(j / p.kblocks, np, mt);
      const bool valid = np * 2 + static_cast<int>(rank) < p.n_tiles;
      mbar_wait(&full[stage], (j / k2Stages) & 1);
      uint4 q[4];
      int32_t k = 0;
      if (valid) {
#pragma unroll
        for (int c = 0; c < 4; ++c) q[c] = ld_shared_v4(w_base + stage * k2Stage + c * (kTileN * 16));
        k = static_cast<int32_t>(ld_shared_u32(sc_base + stage * kTileN * 4));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the async refill
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      uint32_t a[32];
      if (valid) {
        const float kf = static_cast<float>(k);
        const uint32_t k1 = half2_bits(kf);
        const uint32_t k16 = half2_bits(kf * 0.0625f);
        const uint32_t cA = half2_bits(1536.0f - 1032.0f * kf);
        const uint32_t cB = half2_bits(1536.0f - 72.0f * kf);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t w4[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
          for (int w = 0; w < 4; ++w)
            fold_word(w4[w], k1, k16, cA, cB, a[c * 8 + 2 * w], a[c * 8 + 2 * w + 1]);
        }
      } else {
#pragma unroll
        for (int z = 0; z < 32; ++z) a[z] = 0u;
      }
      mbar_wait(&a_empty[as], ((j / k2NA) & 1) ^ 1);
      tc_fence_after();
      tmem_st_x32(tmem_base + lane_base + as * 32, a);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_on_leader(&a_full[as], rank);
    }
  } else if (warp >= 12) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t ew = warp - 12;
    const uint32_t t128 = ew * 32 + lane;
    const uint32_t r = t128;
    const uint32_t lane_base = (ew * 32) << 16;
    pdl_wait();
    auto sa_prefetch = [&](int it) {
      if (it < nunits) {
        int np, mt;
        unit_of(it, np, mt);
        for (int t = t128; t < k2MT; t += 128) {
          const int64_t m = static_cast<int64_t>(mt) * k2MT + t;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                           smem_u32(sa_s + (it & 1) * k2MT + t)),
                       "l"(p.sa + (m < p.M ? m : 0)), "r"(m < p.M ? 8 : 0)
                       : "memory");
        }
      }
      cp_async_commit();
    };
    sa_prefetch(0);
    for (int it = 0; it < nunits; ++it) {
      int np, mt;
      unit_of(it, np, mt);
      const int ds = it & 1;
      sa_prefetch(it + 1);
      cp_async_wait<1>();
      named_bar_sync(1, 128);
      const double* sa_t = sa_s + (it & 1) * k2MT;
      mbar_wait(&d_full[ds], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + lane_base + k2DCol + ds * k2MT;
      const int64_t n = static_cast<int64_t>(np * 2 + static_cast<int>(rank)) * kTileN + r;
      const int64_t m0 = static_cast<int64_t>(mt) * k2MT;
#pragma unroll 1
      for (int cc = 0; cc < k2MT; cc += 32) {
        uint32_t v[32];
        tmem_ld_x16_(taddr + cc, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld_x16_(taddr + cc + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        tmem_wait_ld();
        if (cc + 32 >= k2MT) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_on_leader(&d_empty[ds], rank);
        }
        if (n < p.N) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int64_t m = m0 + cc + i;
            if (m < p.M) {
              if (p.out_dtype == ISB_I32) {
                static_cast<int32_t*>(p.out)[m * p.N + n] = static_cast<int32_t>(v[i]);
              } else {
                const double o = __dmul_rn(
                    static_cast<double>(static_cast<int32_t>(v[i])) * p.inv_amp, sa_t[cc + i]);
                store_out_f(p.out, p.out_dtype, m * p.N + n, __double2float_rn(o));
              }
            }
          }
        }
      }
      named_bar_sync(1, 128);
    }
  }

  tc_fence_before();
  cluster_sync_all();  // no peer arrives on our barriers after this point
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512)
                 : "memory");
}

// Opt-in (ISB_FOLD2=1): bit-exact, but measured slower than the 1-SM kernel at the
// LLaMA-2-7B prefill shapes (1040 vs 1422 TOPS at M = 2048).
bool fold2_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ISB_FOLD2");
    return e && e[0] == '1';
  }();
  return on;
}

void launch_fold2(const CUtensorMap& map, const Fold2Params& prm, int num_sms, cudaStream_t s) {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemm_w4a8_fold2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    k2Smem),
               "cudaFuncSetAttribute(fold2 smem)");
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * std::min(prm.units, num_sms / 2));
  cfg.blockDim = dim3(k2Threads);
  cfg.dynamicSmemBytes = k2Smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_fold2, map, prm), "gemm_w4a8_fold2 launch");
  count_launch();
}

}  // namespace

bool fold_eligible(int64_t m, const isb_weight& w, int path) {
  return path == ISB_PATH_INTEGER_SCALE && w.has_int_scales && w.tensor_core_ok() &&
         w.max_int_scale >= 1 && w.max_int_scale <= 16 && m >= kFoldMinM;
}

void launch_gemm_fold(const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                      void* out, int out_dtype, int num_sms, cudaStream_t s) {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemm_w4a8_fold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kFSmem),
               "cudaFuncSetAttribute(fold smem)");
  });
  FoldParams prm{};
  prm.packed = w.packed;
  prm.kscale = w.kscale_tiled;
  prm.sa = sa;
  prm.out = out;
  prm.M = static_cast<int>(m);
  prm.N = static_cast<int>(w.n);
  prm.G = static_cast<int>(w.groups);
  prm.gb = static_cast<int>(w.group / kBlockK);
  prm.kblocks = static_cast<int>(w.kblocks);
  prm.m_tiles = static_cast<int>((m + kFMT - 1) / kFMT);
  prm.tiles = static_cast<int>(w.n_tiles) * prm.m_tiles;
  prm.out_dtype = out_dtype;
  prm.inv_amp = std::ldexp(1.0, -w.exponent);
  prm.dbg = g_dbg;
  if (fold2_enabled()) {
    Fold2Params p2{};
    p2.packed = w.packed;
    p2.kscale = w.kscale_tiled;
    p2.sa = sa;
    p2.out = out;
    p2.M = static_cast<int>(m);
    p2.N = static_cast<int>(w.n);
    p2.G = static_cast<int>(w.groups);
    p2.gb = static_cast<int>(w.group / kBlockK);
    p2.kblocks = static_cast<int>(w.kblocks);
    p2.m_tiles = static_cast<int>((m + k2MT - 1) / k2MT);
    p2.n_tiles = static_cast<int>(w.n_tiles);
    p2.units = static_cast<int>((w.n_tiles + 1) / 2) * p2.m_tiles;
    p2.out_dtype = out_dtype;
    p2.inv_amp = std::ldexp(1.0, -w.exponent);
    launch_fold2(make_x_map(xq, m, w.k, k2MT / 2), p2, num_sms, s);
    return;
  }
  static const int ss_mt = [] {  // default: SS kernel, 256-token tiles; ISB_FOLD_SS=0: TS kernel
    const char* e = std::getenv("ISB_FOLD_SS");
    return e ? std::atoi(e) : 256;
  }();
  if (ss_mt == 256) {  // four epilogue warpgroups (64 tokens each)
    launch_fold_ss<256, 2, 4, 6, 4>(xq, m, w, prm, num_sms, s);
    return;
  }
  if (ss_mt == 2562) {  // two epilogue warpgroups
    launch_fold_ss<256, 2, 4, 6, 2>(xq, m, w, prm, num_sms, s);
    return;
  }

  const CUtensorMap map = make_x_map(xq, m, w.k, kFMT);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(prm.tiles, num_sms));
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = kFSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_fold, map, prm), "gemm_w4a8_fold launch");
  count_launch();
}

}  // namespace isb
