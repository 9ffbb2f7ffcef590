// K3 (integer scale) and K4 (float scale) — fused W4A8 group GEMM on tcgen05.
//
// Reference: gemm_integer_scale (gemm.cpp:205-262) and gemm_float_scale
// (gemm.cpp:156-203); paper Eq. 2 / Eq. 1 (PAPER.md:149 / :80).
//
// Shape of the computation ("swap-AB"): output channels are the UMMA M dimension
// (128 per tile), tokens are UMMA N (MT = 8..128), so decode-sized M still
// issues full-width MMAs. Per CTA (one per SM, stream-K over (tile, group)):
//
//   warp 0      producer : cp.async.bulk of the 8 KiB packed-int4 block of the
//                          128x128 (n, k) tile + TMA (SWIZZLE_128B) of the MT x 128
//                          int8 activation tile, one mbarrier per stage
//   warps 4-7   transform: smem int4 -> int8 (x16) expansion, tcgen05.st into the
//                          TMEM A-operand ring (thread r owns output channel r)
//   warp 1      MMA      : 4 x tcgen05.mma.kind::i8 (K=32) per 128-K block; one
//                          TMEM accumulator slot per quantization group
//   warps 8+    epilogue : tcgen05.ld of each group's int32 partial 16*P_g,
//                          integer path  acc += (D >> 4) * k_g      (int32, IMAD)
//                          float path    acc += float(D) * (s_g/16) (I2F + FFMA)
//                          then one conversion per output (Eq. 2) and the store.
// Groups of one tile may be split across CTAs (stream-K); partial int32 (or
// fp32) sums go to a caller-owned workspace and the last CTA to arrive on the
// tile's counter reduces them in fixed order and writes the output.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

constexpr int kPrefetch = 8;  // epilogue scale prefetch depth (groups)

template <int MT>
struct Cfg {
  static constexpr int kEpiWG = MT >= 128 ? 2 : 1;           // epilogue warpgroups
  static constexpr int kCols = MT / kEpiWG;                   // D columns per epilogue WG
  static constexpr int kXformWG = MT >= 128 ? 1 : 2;          // int4->int8 transform warpgroups
  static constexpr int kThreads = 128 + 128 * kXformWG + 128 * kEpiWG;
  // TMEM: kNA A-operand stages (32 cols each) + kND accumulator slots (MT cols each).
  // The A ring is a transform->MMA->transform loop whose round trip is several
  // mbarrier hops, so it must be deep enough to cover that latency.
  static constexpr int kNA = MT >= 128 ? 4 : 8;
  static constexpr int kND = MT >= 128 ? 3 : (MT >= 64 ? 4 : 8);
  static constexpr int kTmemUsed = kNA * 32 + kND * MT;
  static constexpr int kTmemCols = kTmemUsed <= 32 ? 32 : kTmemUsed <= 64 ? 64
                                   : kTmemUsed <= 128 ? 128 : kTmemUsed <= 256 ? 256 : 512;
  static_assert(kTmemUsed <= 512, "TMEM overflow");
  static constexpr int kXBytes = MT * 128;
  static constexpr int kXSlot = kXBytes < 1024 ? 1024 : kXBytes;
  // Enough smem stages to cover the producer->HBM->transform->MMA->producer loop.
  static constexpr int kStages = (196 * 1024) / (kBlockBytes + kXSlot) > 24
                                     ? 24 : (196 * 1024) / (kBlockBytes + kXSlot);
  static constexpr int kRingBytes = kEpiWG * kPrefetch * kTileN * 4;
  static constexpr int kSmemBytes = 1024 + kStages * (kBlockBytes + kXSlot) + kRingBytes + 1024;
  static_assert(kSmemBytes <= 227 * 1024, "smem budget");
};

struct Params {
  const uint8_t* packed;
  const int32_t* kscale;  // [n_tiles][G][128]
  const float* fscale;    // [n_tiles][G][128], s/16
  const double* sa;       // [M]
  void* out;              // [M][N]
  int32_t* counters;      // [tiles]
  int32_t* partials;      // [tiles][maxc][MT][128]
  int M, N, G, gb, kblocks, m_tiles, tiles, maxc, out_dtype;
  int64_t units;
  double inv_amp;  // 2^-e (exact)
  int64_t* trace;  // optional per-role clock64 timeline of CTA `trace_cta` (debug)
  int trace_cta;
  int dbg;         // debug knobs: 1 skip A st, 2 skip D ld, 4 skip MMA issue
};

// Debug timeline: trace[role * 512 + i] = globaltimer at event i of that role (16 roles).
#define ISB_TRACE_CTA(role)                                                    \
  do {                                                                         \
    if (p.trace != nullptr) p.trace[(role) * 512 + blockIdx.x] = globaltimer_(); \
  } while (0)
#define ISB_TRACE(role, i)                                                              \
  do {                                                                                  \
    if (p.trace != nullptr && static_cast<int>(blockIdx.x) == p.trace_cta && (i) < 512) \
      p.trace[(role) * 512 + (i)] = globaltimer_();                                         \
  } while (0)

__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int P) {
  int c = static_cast<int>((u * P) / U);
  while (c > 0 && (static_cast<int64_t>(c) * U) / P > u) --c;
  while (c + 1 < P && (static_cast<int64_t>(c + 1) * U) / P <= u) ++c;
  return c;
}

__device__ __forceinline__ void store_out(void* out, int dtype, int64_t idx, float f) {
  if (dtype == ISB_F32)
    static_cast<float*>(out)[idx] = f;
  else if (dtype == ISB_BF16)
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
  else
    static_cast<__half*>(out)[idx] = __float2half_rn(f);
}

template <int MT, int PATH>
__global__ void __launch_bounds__(Cfg<MT>::kThreads, 1)
    gemm_w4a8_tc(const __grid_constant__ CUtensorMap x_map, const Params p) {
  using C = Cfg<MT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr int kXSlot = C::kXSlot;
  constexpr int kStages = C::kStages;
  uint8_t* smem_w = smem;                                  // kStages x 8 KiB
  uint8_t* smem_x = smem + kStages * kBlockBytes;          // kStages x kXSlot (1 KiB aligned)
  int32_t* scale_ring = reinterpret_cast<int32_t*>(smem_x + kStages * kXSlot);  // [wg][PF][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_x + kStages * kXSlot + C::kRingBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* a_full = empty + kStages;
  uint64_t* a_empty = a_full + C::kNA;
  uint64_t* d_full = a_empty + C::kNA;
  uint64_t* d_empty = d_full + C::kND;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + C::kND);
  int32_t* last_flag = reinterpret_cast<int32_t*>(tmem_slot + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&x_map);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1 + 4);
    }
    for (int i = 0; i < C::kNA; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < C::kND; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4 * C::kEpiWG);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) ISB_TRACE(7, 0);
  if (threadIdx.x == 0) pdl_launch_dependents();
  if (threadIdx.x == 0 && p.trace != nullptr) p.trace[14 * 512 + blockIdx.x] = globaltimer_();

  const int P = gridDim.x;
  const int64_t U = p.units;
  const int64_t u0 = (static_cast<int64_t>(blockIdx.x) * U) / P;
  const int64_t u1 = (static_cast<int64_t>(blockIdx.x + 1) * U) / P;
  const int G = p.G, gb = p.gb;

  // Every role walks the same kblock sequence j = 0, 1, ... over this CTA's units;
  // ring slots and mbarrier parities are pure functions of j.
  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      ISB_TRACE(5, 0);
      // Weight blocks do not depend on the preceding kernel: stream the first
      // kStages of them before griddepcontrol.wait so their HBM latency hides
      // behind the previous grid's tail (PDL). Activations (X) are loaded after.
      int j = 0;
      bool waited = false;
      for (int64_t u = u0; u < u1;) {
        const int tile = static_cast<int>(u / G);
        const int g0 = static_cast<int>(u % G);
        const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
        const int nt = tile / p.m_tiles;
        for (int kb = g0 * gb; kb < g1 * gb && j < kStages; ++kb, ++j) {
          mbar_arrive_expect_tx(&full[j], kBlockBytes + C::kXBytes);
          bulk_load_evict_first(smem_w + j * kBlockBytes,
                                p.packed + (static_cast<int64_t>(nt) * p.kblocks + kb) * kBlockBytes,
                                kBlockBytes, &full[j]);
        }
        if (j >= kStages) break;
        u += g1 - g0;
      }
      const int prefetched = j;
      pdl_wait();
      waited = true;
      (void)waited;
      j = 0;
      for (int64_t u = u0; u < u1;) {
        const int tile = static_cast<int>(u / G);
        const int g0 = static_cast<int>(u % G);
        const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
        const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
        for (int kb = g0 * gb; kb < g1 * gb; ++kb, ++j) {
          const int stage = j % kStages;
          if (j >= prefetched) {
            mbar_wait(&empty[stage], ((j / kStages) & 1) ^ 1);
            ISB_TRACE(13, j);
            mbar_arrive_expect_tx(&full[stage], kBlockBytes + C::kXBytes);
            bulk_load_evict_first(smem_w + stage * kBlockBytes,
                                  p.packed + (static_cast<int64_t>(nt) * p.kblocks + kb) * kBlockBytes,
                                  kBlockBytes, &full[stage]);
          }
          tma_load_2d(smem_x + stage * kXSlot, &x_map, &full[stage], kb * kBlockK, mt * MT);
          ISB_TRACE(0, j);
        }
        u += g1 - g0;
      }
      ISB_TRACE_CTA(18);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp)
    constexpr uint32_t idesc = make_idesc_i8(128, MT);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t x_base = smem_u32(smem_x);
    int j = 0, gi = 0;
    for (int64_t u = u0; u < u1;) {
      const int g0 = static_cast<int>(u % G);
      const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
      for (int g = g0; g < g1; ++g, ++gi) {
        const int ds = gi % C::kND;
        mbar_wait(&d_empty[ds], ((gi / C::kND) & 1) ^ 1);
        if (lane == 0) ISB_TRACE(8, j);
        const uint32_t d_tmem = tbase + C::kNA * 32 + ds * MT;
        for (int b = 0; b < gb; ++b, ++j) {
          const int stage = j % kStages, as = j % C::kNA;
          // a_full implies full: the transform warps observed full[stage] (weights
          // and activations of this stage) before arriving.
          mbar_wait(&a_full[as], (j / C::kNA) & 1);
          if (lane == 0) ISB_TRACE(10, j);
          tc_fence_after();
          const uint64_t bdesc = make_sw128_kmajor_desc(x_base + stage * kXSlot);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (!(p.dbg & 4))
              mma_i8_ts_warp(d_tmem, tbase + as * 32 + c * 8, bdesc + static_cast<uint64_t>(c * 2),
                             idesc, (b > 0 || c > 0) ? 1u : 0u);
          mma_commit_warp(&empty[stage]);
          mma_commit_warp(&a_empty[as]);
          if (b == gb - 1) mma_commit_warp(&d_full[ds]);
          if (lane == 0) ISB_TRACE(2, j);
        }
      }
      u += g1 - g0;
    }
    if (lane == 0) ISB_TRACE_CTA(19);
  } else if (warp >= 4 && warp < 4 + 4 * C::kXformWG) {
    // ---------------------------------------------------------------- transform
    // kXformWG warpgroups take alternate kblocks; thread r owns output channel r.
    const uint32_t xw = (warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;  // == TMEM lane
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t w_base = smem_u32(smem_w) + r * 16;
    int j = 0;
    for (int64_t u = u0; u < u1;) {
      const int g0 = static_cast<int>(u % G);
      const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
      for (int kb = g0 * gb; kb < g1 * gb; ++kb, ++j) {
        if (j % C::kXformWG != static_cast<int>(xw)) continue;
        const int stage = j % kStages, as = j % C::kNA;
        mbar_wait(&full[stage], (j / kStages) & 1);
        if (warp == 4 && lane == 0) ISB_TRACE(1, j);
        uint4 q[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) q[c] = ld_shared_v4(w_base + stage * kBlockBytes + c * (kTileN * 16));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (warp == 4 && lane == 0) ISB_TRACE(11, j);
        uint32_t a[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t w4[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            a[c * 8 + 2 * w] = (w4[w] << 4) & 0xF0F0F0F0u;
            a[c * 8 + 2 * w + 1] = w4[w] & 0xF0F0F0F0u;
          }
        }
        mbar_wait(&a_empty[as], ((j / C::kNA) & 1) ^ 1);
        if (warp == 4 && lane == 0) ISB_TRACE(12, j);
        tc_fence_after();
        if (!(p.dbg & 1)) tmem_st_x32(tmem_base + lane_base + as * 32, a);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[as]);
        if (warp == 4 && lane == 0) ISB_TRACE(3, j);
      }
      u += g1 - g0;
    }
  } else if (warp >= 4 + 4 * C::kXformWG) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t ew = warp - (4 + 4 * C::kXformWG);  // 0 .. 4*kEpiWG-1
    const uint32_t wg = ew / 4;               // which column half
    const uint32_t r = (ew % 4) * 32 + lane;  // TMEM lane == output channel in tile
    const uint32_t lane_base = ((ew % 4) * 32) << 16;
    const int c0 = wg * C::kCols;
    constexpr int kCols = C::kCols;
    int ds = 0;
    uint32_t dphase = 0;
    // Per-thread async prefetch of this row's group scale kPrefetch groups ahead
    // (the scales stream from HBM; a dependent load per group would serialise
    // the epilogue on DRAM latency).
    const int32_t* scale_src = PATH == ISB_PATH_INTEGER_SCALE
                                   ? p.kscale : reinterpret_cast<const int32_t*>(p.fscale);
    const uint32_t ring = smem_u32(scale_ring) + (wg * kPrefetch * kTileN + r) * 4;
    auto prefetch = [&](int64_t uu) {
      if (uu < u1) {
        const int t = static_cast<int>(uu / G), gg = static_cast<int>(uu % G);
        const int64_t sidx = (static_cast<int64_t>(t / p.m_tiles) * G + gg) * kTileN + r;
        cp_async_4(ring + static_cast<uint32_t>((uu - u0) % kPrefetch) * (kTileN * 4),
                   scale_src + sidx);
      }
      cp_async_commit();
    };
#pragma unroll
    for (int j = 0; j < kPrefetch; ++j) prefetch(u0 + j);
    pdl_wait();  // sa, the workspace and the output may be touched by the previous grid
    for (int64_t u = u0; u < u1;) {
      const int tile = static_cast<int>(u / G);
      const int g0 = static_cast<int>(u % G);
      const int g1 = static_cast<int>(G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u));
      const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
      int32_t iacc[kCols];
      float facc[kCols];
#pragma unroll
      for (int t = 0; t < kCols; ++t) { iacc[t] = 0; facc[t] = 0.0f; }
      for (int g = g0; g < g1; ++g) {
        const int64_t uu = u + (g - g0);
        cp_async_wait<kPrefetch - 1>();
        const uint32_t sraw =
            ld_shared_u32(ring + static_cast<uint32_t>((uu - u0) % kPrefetch) * (kTileN * 4));
        const int32_t kg = static_cast<int32_t>(sraw);
        const float sg = __uint_as_float(sraw);
        prefetch(uu + kPrefetch);
        mbar_wait(&d_full[ds], dphase);
        if (ew == 0 && lane == 0) ISB_TRACE(4, static_cast<int>(uu - u0));
        tc_fence_after();
        const uint32_t taddr = tmem_base + lane_base + C::kNA * 32 + ds * MT + c0;
        constexpr int kChunk = kCols < 16 ? kCols : 16;
#pragma unroll
        for (int cc = 0; cc < kCols; cc += kChunk) {
          uint32_t v[kChunk];
#pragma unroll
          for (int c = 0; c < kChunk; c += 8) {
            if (!(p.dbg & 2)) {
              tmem_ld_x8(taddr + cc + c, *reinterpret_cast<uint32_t(*)[8]>(&v[c]));
            } else {
#pragma unroll
              for (int z = 0; z < 8; ++z) v[c + z] = z;
            }
          }
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < kChunk; ++t) {
            const int32_t d = static_cast<int32_t>(v[t]);  // 16 * P_g, exact
            if (PATH == ISB_PATH_INTEGER_SCALE)
              iacc[cc + t] += (d >> 4) * kg;                      // Eq. 2: int32 scaled accumulation
            else
              facc[cc + t] = fmaf(static_cast<float>(d), sg, facc[cc + t]);  // Eq. 1, fp32
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[ds]);
        if (++ds == C::kND) { ds = 0; dphase ^= 1; }
      }
      // ------------------------------------------------ tile completion
      if (ew == 0 && lane == 0) ISB_TRACE_CTA(16);
      const bool whole = (g0 == 0 && g1 == G);
      bool finalize = whole;
      if (!whole) {
        const int first = cta_of(static_cast<int64_t>(tile) * G, U, P);
        const int last = cta_of(static_cast<int64_t>(tile) * G + G - 1, U, P);
        const int j = blockIdx.x - first;
        int32_t* tile_ws = p.partials + static_cast<int64_t>(tile) * p.maxc * MT * kTileN;
        if (PATH == ISB_PATH_INTEGER_SCALE) {
          // Integer partials commute: reduce in L2 with red.add (order-free, exact).
#pragma unroll
          for (int t = 0; t < kCols; ++t) atomicAdd(tile_ws + (c0 + t) * kTileN + r, iacc[t]);
        } else {
          int32_t* slice = tile_ws + static_cast<int64_t>(j) * MT * kTileN;
#pragma unroll
          for (int t = 0; t < kCols; ++t) slice[(c0 + t) * kTileN + r] = __float_as_int(facc[t]);
        }
        if (ew == 0 && lane == 0) ISB_TRACE_CTA(20);
        __threadfence();
        if (ew == 0 && lane == 0) ISB_TRACE_CTA(21);
        named_bar_sync(1, 128 * C::kEpiWG);
        if (ew == 0 && lane == 0) {
          const int old = atomicAdd(p.counters + tile, 1);
          const int is_last = old == (last - first);
          if (is_last) p.counters[tile] = 0;  // self-cleaning for the next launch
          *last_flag = is_last;
        }
        named_bar_sync(1, 128 * C::kEpiWG);
        finalize = *last_flag != 0;
        named_bar_sync(1, 128 * C::kEpiWG);
        if (ew == 0 && lane == 0) ISB_TRACE_CTA(22);
        if (finalize) {
          __threadfence();
          if (PATH == ISB_PATH_INTEGER_SCALE) {
#pragma unroll
            for (int t = 0; t < kCols; ++t) {
              int32_t* a = tile_ws + (c0 + t) * kTileN + r;
              iacc[t] = __ldcg(a);
              __stcg(a, 0);  // leave the accumulator zeroed for the next launch
            }
          } else {
            // Fixed-order (deterministic) fp32 reduction over the contributors,
            // all slices of a column chunk loaded before use.
            const int nc = last - first + 1;
            constexpr int kMaxC = 8;
#pragma unroll
            for (int t0 = 0; t0 < kCols; t0 += 8) {
              float part[kMaxC][8];
#pragma unroll
              for (int jj = 0; jj < kMaxC; ++jj)
#pragma unroll
                for (int t = 0; t < 8; ++t)
                  part[jj][t] = (jj < nc && t0 + t < kCols)
                                    ? __int_as_float(__ldcg(tile_ws + static_cast<int64_t>(jj) * MT * kTileN +
                                                            (c0 + t0 + t) * kTileN + r))
                                    : 0.0f;
              // leave the slices zeroed: the integer path red.adds into this workspace
#pragma unroll
              for (int jj = 0; jj < kMaxC; ++jj)
#pragma unroll
                for (int t = 0; t < 8; ++t)
                  if (jj < nc && t0 + t < kCols)
                    __stcg(tile_ws + static_cast<int64_t>(jj) * MT * kTileN + (c0 + t0 + t) * kTileN + r, 0);
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                if (t0 + t < kCols) {
                  float acc = 0.0f;
#pragma unroll
                  for (int jj = 0; jj < kMaxC; ++jj)
                    if (jj < nc) acc += part[jj][t];
                  facc[t0 + t] = acc;
                }
              }
            }
          }
        }
      }
      if (ew == 0 && lane == 0) ISB_TRACE_CTA(23);
      if (finalize) {
        const int64_t n = static_cast<int64_t>(nt) * kTileN + r;
        if (n < p.N) {
#pragma unroll
          for (int t = 0; t < kCols; ++t) {
            const int64_t m = static_cast<int64_t>(mt) * MT + c0 + t;
            if (m < p.M) {
              const double s_a = __ldg(p.sa + m);
              double o;
              if (PATH == ISB_PATH_INTEGER_SCALE)
                o = __dmul_rn(static_cast<double>(iacc[t]) * p.inv_amp, s_a);  // /2^e exact
              else
                o = __dmul_rn(static_cast<double>(facc[t]), s_a);
              store_out(p.out, p.out_dtype, m * p.N + n, __double2float_rn(o));
            }
          }
        }
      }
      if (ew == 0 && lane == 0) ISB_TRACE_CTA(17);
      u += g1 - g0;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ISB_TRACE(6, 0);
  if (threadIdx.x == 0 && p.trace != nullptr) p.trace[15 * 512 + blockIdx.x] = globaltimer_();
  if (warp == 2) tmem_dealloc(tmem_base, C::kTmemCols);
}

// ---------------------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) fail(ISB_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_x_map(const int8_t* xq, int64_t m, int64_t k, int mt) {
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(m)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k)};
  const cuuint32_t box[2] = {128u, static_cast<cuuint32_t>(mt)};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = get_encode_fn()(
      &map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(xq), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ISB_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return map;
}

template <int MT, int PATH>
void launch_mt(const CUtensorMap& map, const Params& prm, int grid, cudaStream_t s) {
  using C = Cfg<MT>;
  auto kern = gemm_w4a8_tc<MT, PATH>;
  static_assert(C::kSmemBytes <= 227 * 1024, "smem");
  static bool attr_set = false;  // per instantiation; benign race (idempotent)
  if (!attr_set) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::kSmemBytes),
               "cudaFuncSetAttribute");
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, map, prm), "gemm_w4a8_tc launch");
  count_launch();
}

int pick_mt(int64_t m) {
  if (m <= 8) return 8;
  if (m <= 16) return 16;
  if (m <= 32) return 32;
  if (m <= 64) return 64;
  return 128;
}

int64_t cta_start(int64_t c, int64_t U, int P) { return (c * U) / P; }

int host_cta_of(int64_t u, int64_t U, int P) {
  int c = static_cast<int>((u * P) / U);
  while (c > 0 && cta_start(c, U, P) > u) --c;
  while (c + 1 < P && cta_start(c + 1, U, P) <= u) ++c;
  return c;
}

}  // namespace

int64_t* g_trace = nullptr;
int g_dbg = 0;
int g_trace_cta = 0;

GemmPlan plan_gemm(int64_t m, const isb_weight& w, int num_sms, int path) {
  GemmPlan pl;
  pl.mt = pick_mt(m);
  pl.m_tiles = static_cast<int>((m + pl.mt - 1) / pl.mt);
  pl.tiles = static_cast<int>(w.n_tiles) * pl.m_tiles;
  pl.units = static_cast<int64_t>(pl.tiles) * w.groups;
  pl.grid = static_cast<int>(std::min<int64_t>(num_sms, pl.units));
  auto max_contrib = [&](int grid) {
    int mc = 1;
    for (int t = 0; t < pl.tiles; ++t) {
      const int first = host_cta_of(static_cast<int64_t>(t) * w.groups, pl.units, grid);
      const int last = host_cta_of(static_cast<int64_t>(t) * w.groups + w.groups - 1, pl.units,
                                   grid);
      mc = std::max(mc, last - first + 1);
    }
    return mc;
  };
  pl.maxc = max_contrib(pl.grid);
  // The fp32 path reduces split tiles in fixed order from at most 8 slices.
  while (path == ISB_PATH_FLOAT_SCALE && pl.maxc > 8 && pl.grid > 1) {
    pl.grid = std::max(1, pl.grid * 8 / pl.maxc - 1);
    pl.maxc = max_contrib(pl.grid);
  }
  const int64_t counters = round_up(static_cast<int64_t>(pl.tiles) * 4, 256);
  const int64_t slices = pl.maxc <= 1 ? 0 : (path == ISB_PATH_INTEGER_SCALE ? 1 : pl.maxc);
  pl.workspace_bytes = counters + static_cast<int64_t>(pl.tiles) * slices * pl.mt * kTileN * 4;
  return pl;
}

void launch_gemm_tc(int path, const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                    void* out, int out_dtype, void* workspace, const GemmPlan& pl,
                    cudaStream_t s) {
  Params prm{};
  prm.packed = w.packed;
  prm.kscale = w.kscale_tiled;
  prm.fscale = w.fscale_tiled;
  prm.sa = sa;
  prm.out = out;
  prm.counters = static_cast<int32_t*>(workspace);
  prm.partials = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(workspace) +
                                            round_up(static_cast<int64_t>(pl.tiles) * 4, 256));
  prm.M = static_cast<int>(m);
  prm.N = static_cast<int>(w.n);
  prm.G = static_cast<int>(w.groups);
  prm.gb = static_cast<int>(w.group / kBlockK);
  prm.kblocks = static_cast<int>(w.kblocks);
  prm.m_tiles = pl.m_tiles;
  prm.tiles = pl.tiles;
  prm.maxc = path == ISB_PATH_INTEGER_SCALE ? 1 : pl.maxc;  // int path: one red.add slice
  prm.out_dtype = out_dtype;
  prm.units = pl.units;
  prm.inv_amp = std::ldexp(1.0, -w.exponent);
  prm.trace = g_trace;
  prm.trace_cta = g_trace_cta;
  prm.dbg = g_dbg;
  const CUtensorMap map = make_x_map(xq, m, w.k, pl.mt);
#define ISB_DISPATCH(MTV)                                                              \
  case MTV:                                                                            \
    if (path == ISB_PATH_INTEGER_SCALE)                                                \
      launch_mt<MTV, ISB_PATH_INTEGER_SCALE>(map, prm, pl.grid, s);                    \
    else                                                                               \
      launch_mt<MTV, ISB_PATH_FLOAT_SCALE>(map, prm, pl.grid, s);                      \
    break;
  switch (pl.mt) {
    ISB_DISPATCH(8)
    ISB_DISPATCH(16)
    ISB_DISPATCH(32)
    ISB_DISPATCH(64)
    ISB_DISPATCH(128)
    default: fail(ISB_ERROR, "bad tile");
  }
#undef ISB_DISPATCH
}

}  // namespace isb
