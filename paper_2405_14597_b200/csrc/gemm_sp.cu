// K3 prefill, integer scale folded into the int4 -> int8 weight expansion, on a CTA
// pair with TOKENS as the MMA M dimension — the default prefill kernel (M >= 256,
// k_g <= 16): single GEMM, or a layer's linears in one grouped launch.
//
// Reference: gemm_integer_scale (gemm.cpp:205-262), paper Eq. 2. As in gemm_fold.cu,
// sum_g k_g * P_g = sum_k x_k * (k_g(k) * w_k) and k_g * w fits int8 when k_g <= 16,
// so the tensor core accumulates the integer-scaled int32 accumulator over the whole
// K (bit-identical: every partial sum is within the static overflow bound, which the
// caller gates on).
//
// Why this shape (prefill): the 1-CTA kernel (gemm_fold.cu, 128
// channels x 256 tokens) is issue-bound — per 128-K block an SM must expand 128 x 128
// weights (~700 warp instructions) and convert 256 outputs per channel row. Here a
// pair tile is 512 tokens x 128 channels: the pair issues two M = 256 MMAs (token
// sub-tiles) per K-chunk against ONE folded weight operand (N = 128, each CTA
// expanding its 64 channels), so each expanded weight feeds 512 tokens — half the
// expansion work per MMA. The accumulator rows are tokens: an epilogue thread owns one
// token (one activation scale) and 32 consecutive channels per TMEM load, stored as
// 16-byte vectors.
//
// Pair tile (cluster of 2, tcgen05.mma.cta_group::2, M = 256, N = 128, K = 32):
//   CTA r: activation rows mt*512 + s*256 + r*128 .. +128 for sub-tiles s = 0, 1
//          (TMA, SWIZZLE_128B), weights for channels nt*128 + r*64 .. +64 (its half of
//          the N = 128 operand), D rows = its 128 tokens of each sub-tile.
//   TMEM per CTA: 2 buffers x 2 sub-tiles x 128 columns (double-buffered accumulators).
//
//   warp 0      producer W : per 128-K block 4 x 1 KiB packed rows + 256 B of k_g.
//   warp 1      MMA (leader CTA): 8 MMAs per block, commits multicast to both CTAs.
//   warp 2      TMEM allocator (cta_group::2).
//   warp 3      producer X : 2 TMA loads per block (both sub-tiles), signalling the leader.
//   warps 4..   transform  : NXW warps, one per block (block j -> warp j % NXW, which owns
//                            W slot and B slot j % NXW): 64 rows, 2 per lane, k_g * int4
//                            -> int8 into the swizzled B slot.
//   then        epilogue   : 2 warpgroups (sub-tile s), warp q drains TMEM lanes 32q.. (its
//                            tokens), 32 channels per load: out = float((double)acc *
//                            (s_a * 2^-e)), packed to bf16/f16, 16-byte stores.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "fold.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

constexpr int kSpMaxProb = 8;
constexpr int kSpT = 512;                    // tokens per pair tile (two M = 256 sub-tiles)
constexpr int kSpXSub = 128 * kBlockK;       // one sub-tile's 128 token rows x 128 K = 16 KiB
constexpr int kSpXStage = 2 * kSpXSub;       // per CTA per block
constexpr int kSpBBytes = 64 * kBlockK;      // folded weights, 64 channels x 128 K = 8 KiB
constexpr int kSpWBytes = kBlockBytes / 2;   // packed, 64 channels x 128 K = 4 KiB
constexpr int kSpSc = 64 * 4;                // k_g of 64 channels

struct SpProb {
  const uint8_t* packed;  // [n_tiles][kblocks][chunk 4][row 128][16 B]
  const int32_t* kscale;  // [n_tiles][G][128]
  const double* sa;       // [M]
  void* out;              // [M][N]
  double inv_amp;         // 2^-e
  int M, N, G, gb, kblocks, m_tiles, n_tiles, out_dtype;
};

struct SpMaps {
  CUtensorMap x[kSpMaxProb];  // int8 activations [M][K], box 128 (K) x 128 rows, SWIZZLE_128B
};

struct SpParams {
  SpProb prob[kSpMaxProb];
  int nprob;
  // Work list: cluster c runs items[off[c] .. off[c+1]) = (prob, n-tile, m-tile).
  // nullptr: one problem, unit u = c + i * #clusters -> (u / m_tiles, u % m_tiles).
  const int4* items;
  const int* item_off;
  int units;
  int dbg;  // isb_debug_set_flags measurement knobs: 1 no fold ALU, 4 no epilogue stores
  int64_t* trace;  // debug timeline (isb_debug_set_trace): [32][512] clock64, cluster 0
};

// Timeline tracing (scripts/trace_pair.py) is compiled in only with -DISB_SP_TRACE=1
// (scripts/build_sp_variant.sh): the checks cost the single-thread MMA issuer cycles.
#ifndef ISB_SP_TRACE
#define ISB_SP_TRACE 0
#endif
#ifndef ISB_SP_KNOBS
#define ISB_SP_KNOBS 0
#endif
__device__ __forceinline__ void trace_put_sp(const SpParams& p, int row, int idx, int64_t t) {
  if (ISB_SP_TRACE && p.trace != nullptr && idx < 512 && blockIdx.x < 2)
    p.trace[(row + 16 * static_cast<int>(blockIdx.x)) * 512 + idx] = t;
}
// globaltimer rows (ns, comparable across the pair's SMs): [32 + 2 * row + cta][512]
__device__ __forceinline__ void sp_gtrace(const SpParams& p, int row, int idx) {
  if (ISB_SP_TRACE && p.trace != nullptr && idx < 512 && blockIdx.x < 2)
    p.trace[(32 + 2 * row + static_cast<int>(blockIdx.x)) * 512 + idx] = globaltimer_();
}
__device__ __forceinline__ void sp_trace(const SpParams& p, int row, int idx) {
  if (ISB_SP_TRACE && p.trace != nullptr && idx < 512 && blockIdx.x < 2)
    p.trace[(row + 16 * static_cast<int>(blockIdx.x)) * 512 + idx] = clock64_();
}

template <int SX, int NXW, int EW, int WPB, int NW, int NB>
struct SpCfg {
  static constexpr int kXW = NXW * WPB;  // transform warps: WPB per block (block j -> warp j % NXW)
  // Packed-weight ring (NW blocks of lookahead) and folded-weight ring (NB slots): block j
  // uses W slot j % NW and B slot j % NB. Both rings are at least NXW deep, so a warp's
  // wait on a slot can never see a phase two uses old or new: its previous block's wait
  // already covered block j - NXW - NB (MMA and producers consume in order).
  static constexpr int kNW = NW;
  static_assert(NW >= NXW && NB >= NXW, "rings shallower than the transform warp count");
  static constexpr int kEW = EW;  // epilogue warpgroups: EW / 2 per token sub-tile
  static constexpr int kThreads = 128 + 32 * kXW + 128 * kEW;
  static constexpr int kStageTok = 16;                // tokens per staging round
  static constexpr int kStage = kStageTok * 64;       // per epilogue warp: 16 tokens x 32 bf16 channels
  static constexpr int kSmem = 1024 + SX * kSpXStage + NB * kSpBBytes + kNW * (kSpWBytes + kSpSc) +
                               4 * EW * kStage + 1024;
  static_assert(kSmem <= 227 * 1024, "smem");
  static_assert((4 + NXW) % 4 == 0 || true, "epilogue quadrant = warp % 4");
};

// mbarrier wait with a suspend-time hint: the waiting warp sleeps in try_wait until the
// phase completes instead of re-issuing TRYWAIT + BRA (knob 512: plain spin, A/B).
__device__ __forceinline__ void swait(uint64_t* bar, uint32_t parity, int dbg) {
  if (dbg & 512) {
    mbar_wait(bar, parity);
    return;
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
}

__device__ __forceinline__ void arrive_leader(uint64_t* bar, uint32_t rank) {
  // default semantics (release at CTA scope), as CUTLASS's ClusterBarrier::arrive; the
  // cluster-scope release form costs ~1000 cycles per arrive
  if (rank == 0)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
  else
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_u32(bar), 0))
                 : "memory");
}

__device__ __forceinline__ void mma2_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, uint32_t (&v)[32]) {
  tmem_ld_x16_(taddr, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
  tmem_ld_x16_(taddr + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
}

__device__ __forceinline__ void st_global_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  // streaming store: written once; must not evict the L2-resident activations
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d));
}


template <int SX, int NXW, int EW, int WPB, int NW, int NB>
__global__ void __launch_bounds__(SpCfg<SX, NXW, EW, WPB, NW, NB>::kThreads, 1)
    gemm_w4a8_sp(const __grid_constant__ SpMaps maps, const __grid_constant__ SpParams p) {
  using C = SpCfg<SX, NXW, EW, WPB, NW, NB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_x = smem;                                  // [SX][2 sub-tiles][128 x 128]
  uint8_t* smem_b = smem_x + SX * kSpXStage;               // [NB][64 x 128] folded weights
  uint8_t* smem_w = smem_b + NB * kSpBBytes;               // [kNW][4 chunks][64 rows][16 B]
  uint8_t* smem_sc = smem_w + C::kNW * kSpWBytes;          // [kNW][64] k_g
  uint8_t* smem_o = smem_sc + C::kNW * kSpSc;              // [epilogue warp][16 x 64 B] staging
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem_o + 4 * EW * C::kStage);  // local
  uint64_t* wempty = wfull + C::kNW;  // local (owning transform warp)
  uint64_t* xfull = wempty + C::kNW;  // leader: both CTAs' TMA bytes
  uint64_t* xempty = xfull + SX;    // local (multicast commit)
  uint64_t* bfull = xempty + SX;    // leader: both CTAs' transform warp
  uint64_t* bempty = bfull + NB;    // local (multicast commit)
  uint64_t* dfull = bempty + NB;    // local (multicast commit)
  uint64_t* dempty = dfull + 2;     // leader: both CTAs' epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);

  // Measurement knobs (isb_debug_set_flags) are compiled in only with -DISB_SP_KNOBS=1
  // (scripts/build_sp_variant.sh): their dead branches otherwise cost the product
  // epilogue registers (spills in the staged-store loop).
  const int dbg = ISB_SP_KNOBS ? p.dbg : 0;

  // fold constants for k_g = 0..16, built once: a row's constants are then one 16-byte
  // shared load instead of five conversions on the XU pipe the epilogue keeps busy
  __shared__ uint4 fold_tab[17];
  if (threadIdx.x < 17) {
    const FoldK f = fold_constants(static_cast<int32_t>(threadIdx.x));
    fold_tab[threadIdx.x] = make_uint4(f.k1, f.k16, f.cA, f.cB);
  }

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  // The MMA issuer is a single thread; it sits on warp 2 (knob 1 << 14: warp 1, A/B —
  // with six transform warps, two of them sharing warp 1's SMSP, warp 2 measured 5-6 %
  // fewer cycles per block).
  const uint32_t mma_warp = (dbg & (1 << 14)) ? 1u : 2u, alloc_warp = 3u - mma_warp;
  const int cid = static_cast<int>(blockIdx.x) / 2, ncl = static_cast<int>(gridDim.x) / 2;
  int it_begin, nunits;
  if (p.items) {
    it_begin = p.item_off[cid];
    nunits = p.item_off[cid + 1] - it_begin;
  } else {
    it_begin = 0;
    nunits = cid < p.units ? (p.units - cid + ncl - 1) / ncl : 0;
  }
  auto unit_of = [&](int it, int& pb, int& nt, int& mt) {
    if (p.items) {
      const int4 u = p.items[it_begin + it];
      pb = u.x;
      nt = u.y;
      mt = u.z;
    } else {
      const int u = cid + it * ncl;
      pb = 0;
      nt = u / p.prob[0].m_tiles;
      mt = u % p.prob[0].m_tiles;
    }
  };

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < p.nprob; ++i) prefetch_tensormap(&maps.x[i]);
    for (int i = 0; i < C::kNW; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], WPB);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&bfull[i], 2 * WPB);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < SX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&dempty[i], 2 * 4 * C::kEW);
    }
    fence_barrier_init();
  }
  if (warp == alloc_warp) {
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

  if (warp == 0) {
    // ------------------------------------------------ producer: packed weights + k_g
    if (elect_one()) {
      int j = 0;
      for (int it = 0; it < nunits; ++it) {
        int pb, nt, mt;
        unit_of(it, pb, nt, mt);
        const SpProb& q = p.prob[pb];
        for (int kb = 0; kb < q.kblocks; ++kb, ++j) {
          const int s = j % C::kNW;
          swait(&wempty[s], ((j / C::kNW) & 1) ^ 1, dbg);
          mbar_arrive_expect_tx(&wfull[s], kSpWBytes + kSpSc);
          const uint8_t* src = q.packed + (static_cast<int64_t>(nt) * q.kblocks + kb) * kBlockBytes +
                               rank * (kSpWBytes / 4);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            bulk_load(smem_w + s * kSpWBytes + c * (kSpWBytes / 4), src + c * (kBlockBytes / 4),
                      kSpWBytes / 4, &wfull[s]);
          bulk_load(smem_sc + s * kSpSc,
                    q.kscale + (static_cast<int64_t>(nt) * q.G + kb / q.gb) * kTileN + rank * 64,
                    kSpSc, &wfull[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ------------------------------------------------ producer: activation sub-tiles
    if (elect_one()) {
      const uint32_t xfull_leader = mapa_shared(smem_u32(xfull), 0);
      pdl_wait();
      int j = 0;
      for (int it = 0; it < nunits; ++it) {
        int pb, nt, mt;
        unit_of(it, pb, nt, mt);
        const int kbs = p.prob[pb].kblocks;
        for (int kb = 0; kb < kbs; ++kb, ++j) {
          const int s = j % SX;
          swait(&xempty[s], ((j / SX) & 1) ^ 1, dbg);
          // knob 1 << 13 (measurement): only sub-tile 0's activations are loaded (half the
          // L2 -> SM activation traffic; sub-tile 1 computes on stale data, wrong results)
          const int nsub = (dbg & (1 << 13)) ? 1 : 2;
          if (rank == 0) mbar_arrive_expect_tx(&xfull[s], nsub * kSpXStage);  // both CTAs
#pragma unroll
          for (int sub = 0; sub < nsub; ++sub)
            asm volatile(
                "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
                "bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_x + s * kSpXStage + sub * kSpXSub)),
                "l"(reinterpret_cast<uint64_t>(&maps.x[pb])),
                "r"(xfull_leader + static_cast<uint32_t>(s) * 8u), "r"(kb * kBlockK),
                "r"(mt * kSpT + sub * 256 + static_cast<int>(rank) * 128)
                : "memory");
        }
      }
    }
    __syncwarp();
  } else if (warp == mma_warp) {
    // ------------------------------------------------ MMA issuer (leader CTA)
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = make_idesc_i8(256, 128);
      const uint64_t adesc0 = make_sw128_kmajor_desc(smem_u32(smem_x));
      const uint64_t bdesc0 = make_sw128_kmajor_desc(smem_u32(smem_b));
      int j = 0, xs = 0, bs = 0;  // block, activation stage, folded-weight slot
      uint32_t xph = 0, bph = 0;  // their ring phases
      for (int it = 0; it < nunits; ++it) {
        int pb, nt, mt;
        unit_of(it, pb, nt, mt);
        const int kbs = p.prob[pb].kblocks;
        const int buf = it & 1;
        swait(&dempty[buf], ((it >> 1) & 1) ^ 1, dbg);
        tc_fence_after();
        const uint32_t d0 = tmem_base + buf * 256;
        for (int kb = 0; kb < kbs; ++kb, ++j) {
          swait(&bfull[bs], bph, dbg);
          sp_trace(p, 0, j);
          sp_gtrace(p, 0, j);
          swait(&xfull[xs], xph, dbg);
          sp_trace(p, 1, j);
          tc_fence_after();
          // descriptors by offset from the ring bases (start-address field = addr >> 4)
          const uint64_t bdesc = bdesc0 + static_cast<uint64_t>(bs * (kSpBBytes >> 4));
          const uint64_t adesc = adesc0 + static_cast<uint64_t>(xs * (kSpXStage >> 4));
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int sub = 0; sub < 2; ++sub)
              mma2_ss(d0 + sub * 128, adesc + static_cast<uint64_t>(sub * (kSpXSub >> 4) + c * 2),
                      bdesc + static_cast<uint64_t>(c * 2), idesc, (kb > 0 || c > 0) ? 1u : 0u);
          commit2_mc(&xempty[xs]);
          commit2_mc(&bempty[bs]);
          sp_trace(p, 2, j);
          sp_gtrace(p, 3, j);
          if (++xs == SX) { xs = 0; xph ^= 1u; }
          if (++bs == NB) { bs = 0; bph ^= 1u; }
        }
        commit2_mc(&dfull[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + C::kXW) {
    // ------------------------------------------------ transform: one warp per block
    const int xw = (static_cast<int>(warp) - 4) / WPB;     // blocks j with j % NXW == xw
    const int half = (static_cast<int>(warp) - 4) % WPB;   // which rows of the slot (WPB = 2)
    int total = 0;
    for (int it = 0; it < nunits; ++it) {
      int pb, nt, mt;
      unit_of(it, pb, nt, mt);
      total += p.prob[pb].kblocks;
    }
    const uint32_t w_base = smem_u32(smem_w);
    const uint32_t sc_base = smem_u32(smem_sc);
    for (int j = xw, u = 0; j < total; j += NXW, ++u) {
      const int ws = j % C::kNW, bs = j % NB;
      const uint32_t b_slot = smem_u32(smem_b + bs * kSpBBytes);
      const uint32_t w_slot = w_base + ws * kSpWBytes;
      const uint32_t sc_slot = sc_base + ws * kSpSc;
      const bool trx = ISB_SP_TRACE && lane == 0 && warp == 4 && p.trace != nullptr;
      const int64_t tx0 = trx ? clock64_() : 0;
      swait(&wfull[ws], (j / C::kNW) & 1, dbg);
      const int64_t tx1 = trx ? clock64_() : 0;
      swait(&bempty[bs], ((j / NB) & 1) ^ 1, dbg);
      if (lane == 0) sp_gtrace(p, 1, j);
      const int64_t tx2 = trx ? clock64_() : 0;
#pragma unroll
      for (int i = 0; i < 2 / WPB; ++i) {
        const uint32_t row = lane + 32 * (WPB == 1 ? i : half);  // channel row of this CTA's 64
        uint4 w4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) w4[c] = ld_shared_v4(w_slot + c * (kSpWBytes / 4) + row * 16);
        const int32_t k = static_cast<int32_t>(ld_shared_u32(sc_slot + row * 4));
        const uint4 fk = fold_tab[min(max(k, 0), 16)];  // k_g <= 16 on this path
        const FoldK f{fk.x, fk.y, fk.z, fk.w};
        uint32_t a[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t wv[4] = {w4[c].x, w4[c].y, w4[c].z, w4[c].w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            if (dbg & 1) {  // measurement: no fold ALU (wrong results)
              a[c * 8 + 2 * w] = wv[w] ^ f.k1;
              a[c * 8 + 2 * w + 1] = wv[w];
            } else {
              fold_word(wv[w], f.k1, f.k16, f.cA, f.cB, a[c * 8 + 2 * w], a[c * 8 + 2 * w + 1]);
            }
          }
        }
        // canonical SWIZZLE_128B K-major: 16-byte chunk c of row r at r*128 + (c ^ (r & 7))*16
        const uint32_t dst = b_slot + row * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + ((ch ^ (row & 7)) * 16)),
                       "r"(a[4 * ch]), "r"(a[4 * ch + 1]), "r"(a[4 * ch + 2]), "r"(a[4 * ch + 3])
                       : "memory");
      }
      // W-slot reads before its async refill; B-slot writes before the tensor core reads
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&wempty[ws]);
        arrive_leader(&bfull[bs], rank);
        sp_gtrace(p, 2, j);
        if (trx) {
          trace_put_sp(p, 12, u, tx0);
          trace_put_sp(p, 13, u, tx1);
          trace_put_sp(p, 14, u, tx2);
          trace_put_sp(p, 15, u, clock64_());
        }
        if (xw == 0 && half == 0) sp_trace(p, 5, u);
      }
    }
  } else if (warp >= 4 + C::kXW) {
    // ------------------------------------------------ epilogue
    const uint32_t ew = warp - (4 + C::kXW);
    constexpr int kWgPerSub = EW / 2;             // warpgroups sharing one sub-tile
    constexpr int kChunks = 4 / kWgPerSub;        // 32-channel chunks per warpgroup
    const int sub = static_cast<int>(ew / 4) / kWgPerSub;
    const int c0 = (static_cast<int>(ew / 4) % kWgPerSub) * kChunks;
    const uint32_t qd = warp % 4;  // a warp reaches TMEM lanes 32 * (warp % 4) ..
    const uint32_t lane_base = (qd * 32) << 16;
    pdl_wait();
    // this thread's token scale, fetched one tile ahead: under the prefill's L2 load a
    // demand load issued at the tile boundary stalled the first conversion ~5 k cycles
    auto token_of = [&](int it, int64_t& m, const SpProb*& qq) {
      int pb, nt, mt;
      unit_of(it, pb, nt, mt);
      qq = &p.prob[pb];
      m = static_cast<int64_t>(mt) * kSpT + sub * 256 + rank * 128 + qd * 32 + lane;
    };
    double sa_next = 0.0;
    if (nunits > 0) {
      int64_t m1;
      const SpProb* q1;
      token_of(0, m1, q1);
      sa_next = m1 < q1->M ? __ldg(q1->sa + m1) : 0.0;
    }
    for (int it = 0; it < nunits; ++it) {
      int pb, nt, mt;
      unit_of(it, pb, nt, mt);
      const SpProb& q = p.prob[pb];
      const int buf = it & 1;
      const int64_t m = static_cast<int64_t>(mt) * kSpT + sub * 256 + rank * 128 + qd * 32 + lane;
      const bool m_ok = m < q.M;
      const double sa2 = sa_next * q.inv_amp;  // s_a * 2^-e, exact (0 past M)
      if (it + 1 < nunits) {
        int64_t m1;
        const SpProb* q1;
        token_of(it + 1, m1, q1);
        sa_next = m1 < q1->M ? __ldg(q1->sa + m1) : 0.0;
      }
      swait(&dfull[buf], (it >> 1) & 1, dbg);
      if (ew == 0 && lane == 0) sp_trace(p, 6, it);
      tc_fence_after();
      const uint32_t taddr = tmem_base + lane_base + buf * 256 + sub * 128;
      const int64_t n0 = static_cast<int64_t>(nt) * kTileN;
      if (kChunks == 2 && (q.out_dtype == ISB_BF16 || q.out_dtype == ISB_F16) &&
          !(dbg & (4 | 8 | 128 | 256 | 1024 | 2048 | 4096))) {
        // bf16 / f16 output: both chunks' accumulators are loaded and the TMEM buffer is
        // released to the MMA before any conversion (the release gates the MMA of the
        // tile after next; 80 registers with 4 transform warps). Knob 2: the second
        // chunk loaded after the first one's conversion; knob 1024: the general loop.
        const bool bf = q.out_dtype == ISB_BF16;
        const double c52 = -sa2 * 4503599627370496.0;  // -2^52 * sa2, exact
        const bool dadd_form = dbg & 32;
        auto cvt_pack = [&](const uint32_t (&v)[32], uint32_t (&h)[16]) {
          if (dadd_form) {  // A/B: bias DADD + DMUL (the general loop's form)
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              const double d0 = __hiloint2double(0x43300000, static_cast<int>(v[2 * t] ^ 0x80000000u)) -
                                4503601774854144.0;
              const double d1 = __hiloint2double(0x43300000, static_cast<int>(v[2 * t + 1] ^ 0x80000000u)) -
                                4503601774854144.0;
              const float f0 = __double2float_rn(d0 * sa2), f1 = __double2float_rn(d1 * sa2);
              if (bf) {
                const __nv_bfloat162 b = __floats2bfloat162_rn(f0, f1);
                h[t] = *reinterpret_cast<const uint32_t*>(&b);
              } else {
                const __half2 b = __floats2half2_rn(f0, f1);
                h[t] = *reinterpret_cast<const uint32_t*>(&b);
              }
            }
            return;
          }
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float f0, f1;
            if (false) {
              const double d0 = __hiloint2double(0x43300000, static_cast<int>(v[2 * t] ^ 0x80000000u)) -
                                4503601774854144.0;
              const double d1 = __hiloint2double(0x43300000, static_cast<int>(v[2 * t + 1] ^ 0x80000000u)) -
                                4503601774854144.0;
              f0 = __double2float_rn(d0 * sa2);
              f1 = __double2float_rn(d1 * sa2);
            } else {
              // Eq. 2 exactly as gemm.cpp:252 in ONE FP64 op: D = 2^52 + |acc| (bit
              // construction), fma(D, sa2, -2^52 sa2) = RN64(|acc| * sa2) — the product is
              // exact inside the FMA and -2^52 sa2 is an exact power-of-two scaling — then
              // F2F and the sign (RN is odd-symmetric)
              const uint32_t a0 = v[2 * t], a1 = v[2 * t + 1];
              const uint32_t m0 = (a0 >> 31) ? 0u - a0 : a0, m1 = (a1 >> 31) ? 0u - a1 : a1;  // |acc|
              const double p0 = __fma_rn(__hiloint2double(0x43300000, static_cast<int>(m0)), sa2, c52);
              const double p1 = __fma_rn(__hiloint2double(0x43300000, static_cast<int>(m1)), sa2, c52);
              f0 = __uint_as_float(__float_as_uint(__double2float_rn(p0)) ^ (a0 & 0x80000000u));
              f1 = __uint_as_float(__float_as_uint(__double2float_rn(p1)) ^ (a1 & 0x80000000u));
            }
            if (bf) {
              const __nv_bfloat162 b = __floats2bfloat162_rn(f0, f1);
              h[t] = *reinterpret_cast<const uint32_t*>(&b);
            } else {
              const __half2 b = __floats2half2_rn(f0, f1);
              h[t] = *reinterpret_cast<const uint32_t*>(&b);
            }
          }
        };
        auto store_h = [&](const uint32_t (&h)[16], int cc) {
          const int64_t nb = n0 + cc * 32;
          const int nv = q.N - nb < 32 ? static_cast<int>(q.N - nb) : 32;
          if (nv <= 0) return;
          if (q.N % 8 == 0 && nb + 32 <= q.N) {
            const uint32_t stg = smem_u32(smem_o + ew * C::kStage);
            const int64_t mw = m - lane;
#pragma unroll
            for (int half = 0; half < 32 / C::kStageTok; ++half) {
              const int tl = static_cast<int>(lane) - half * C::kStageTok;
              if (tl >= 0 && tl < C::kStageTok) {
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                   stg + tl * 64 + (((qq + (tl >> 1)) & 3) * 16)),
                               "r"(h[4 * qq]), "r"(h[4 * qq + 1]), "r"(h[4 * qq + 2]),
                               "r"(h[4 * qq + 3])
                               : "memory");
              }
              __syncwarp();
#pragma unroll
              for (int i = 0; i < C::kStageTok / 8; ++i) {
                const uint32_t tk = 8 * i + lane / 4, pq = lane % 4;
                const uint4 d = ld_shared_v4(stg + tk * 64 + (((pq + (tk >> 1)) & 3) * 16));
                const int64_t tok = mw + half * C::kStageTok + tk;
                if (tok < q.M)
                  st_global_v4(static_cast<uint16_t*>(q.out) + tok * q.N + nb + pq * 8, d.x, d.y, d.z, d.w);
              }
              __syncwarp();
            }
          } else if (m_ok) {
            uint16_t* po = static_cast<uint16_t*>(q.out) + m * q.N + nb;
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (t < nv) po[t] = static_cast<uint16_t>(h[t / 2] >> (16 * (t & 1)));
          }
        };
        uint32_t v[32], h[16];
        if (!(dbg & 2)) {  // both chunks to registers, release, then convert (knob 2: A/B)
          uint32_t w[32];
          // timeline (trace builds): clock64 kept in registers, written after the tile
          const bool tr = ISB_SP_TRACE && ew == 0 && lane == 0 && p.trace != nullptr;
          int64_t ts[6] = {0, 0, 0, 0, 0, 0};
          if (tr) ts[0] = clock64_();
          tmem_ld_x32(taddr + c0 * 32, v);
          tmem_ld_x32(taddr + (c0 + 1) * 32, w);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&dempty[buf], rank);
          if (tr) ts[1] = clock64_() + (v[0] == 0x7fffffffu ? 1 : 0);
          cvt_pack(v, h);
          if (tr) ts[2] = clock64_() + (h[15] == 0x7fffffffu ? 1 : 0);
          store_h(h, c0);
          if (tr) ts[3] = clock64_();
          cvt_pack(w, h);
          if (tr) ts[4] = clock64_() + (h[15] == 0x7fffffffu ? 1 : 0);
          store_h(h, c0 + 1);
          if (tr) {
            ts[5] = clock64_();
            trace_put_sp(p, 8, it * 4, ts[0]);
            trace_put_sp(p, 9, it * 4, ts[1]);
            trace_put_sp(p, 10, it * 4, ts[2]);
            trace_put_sp(p, 11, it * 4, ts[3]);
            trace_put_sp(p, 8, it * 4 + 1, ts[4]);
            trace_put_sp(p, 9, it * 4 + 1, ts[5]);
          }
          continue;
        }
        tmem_ld_x32(taddr + c0 * 32, v);
        tmem_wait_ld();
        cvt_pack(v, h);
        tmem_ld_x32(taddr + (c0 + 1) * 32, v);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&dempty[buf], rank);
        store_h(h, c0);
        cvt_pack(v, h);
        store_h(h, c0 + 1);
        continue;
      }
#pragma unroll 1
      for (int cc = c0; cc < c0 + kChunks; ++cc) {
        uint32_t v[32];
        const bool tr = ISB_SP_TRACE && ew == 0 && lane == 0 && p.trace != nullptr;
        const int ti = it * 4 + cc;
        if (tr) sp_trace(p, 8, ti);
        tmem_ld_x32(taddr + cc * 32, v);
        tmem_wait_ld();
        if (tr) sp_trace(p, 9, ti + (v[0] == 0x7fffffffu ? 1 : 0));
        if (cc == c0 + kChunks - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&dempty[buf], rank);
          if (ew == 0 && lane == 0) sp_trace(p, 7, it);
        }
        if (dbg & 4) continue;  // (lanes past M stay: the staged store below is warp-wide)
        const int64_t nb = n0 + cc * 32;
        const int nv = q.N - nb < 32 ? static_cast<int>(q.N - nb) : 32;  // valid channels
        if (nv <= 0) continue;
        if (q.out_dtype == ISB_I32) {
          if (!m_ok) continue;
          int32_t* po = static_cast<int32_t*>(q.out) + m * q.N + nb;
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (t < nv) po[t] = static_cast<int32_t>(v[t]);
          continue;
        }
        // Eq. 2 exactly as gemm.cpp:252: (double)acc via the 2^52 + 2^31 bias (a DADD on
        // the FP64 pipe instead of an I2F.F64 conversion), one DMUL, one F2F.F32.F64
        float f[32];
        if (dbg & 8) {  // measurement: no conversion (wrong results)
#pragma unroll
          for (int t = 0; t < 32; ++t) f[t] = __int_as_float(v[t]);
        } else if (dbg & 256) {  // A/B: FP32 fast path with exact FP64 fallback (eq2_fast)
          float2 sf2;  // (hi, lo) float split of sa2; hi = NaN: always the exact path
          {
            const float hi = __double2float_rn(sa2);
            const bool ok = fabs(sa2) >= 0x1p-100 && fabs(sa2) <= 0x1p100;
            sf2 = make_float2(ok ? hi : __int_as_float(0x7FC00000),
                              __double2float_rn(sa2 - static_cast<double>(hi)));
          }
          uint32_t slow = 0;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            bool sl;
            f[t] = eq2_fast(static_cast<int32_t>(v[t]), sf2, sl);
            slow |= sl ? (1u << t) : 0u;
          }
          if (slow) {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if ((slow >> t) & 1)
                f[t] = __double2float_rn(static_cast<double>(static_cast<int32_t>(v[t])) * sa2);
          }
        } else if (dbg & 2048) {  // A/B: every int -> double on the XU pipe (I2F.F64)
#pragma unroll
          for (int t = 0; t < 32; ++t)
            f[t] = __double2float_rn(static_cast<double>(static_cast<int32_t>(v[t])) * sa2);
        } else if (dbg & 4096) {  // A/B: int -> double alternating XU (I2F.F64) / FP64 (bias DADD)
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const double d = (t & 1) ? static_cast<double>(static_cast<int32_t>(v[t]))
                                     : __hiloint2double(0x43300000, static_cast<int>(v[t] ^ 0x80000000u)) -
                                           4503601774854144.0;
            f[t] = __double2float_rn(d * sa2);
          }
        } else {
          // Eq. 2 exactly as gemm.cpp:252: (double)acc via the 2^52 + 2^31 bias (a DADD on
          // the FP64 pipe instead of an I2F.F64 conversion), one DMUL, one F2F.F32.F64
          // (scripts/cvt_bench.cu: ~16-21 outputs / clk / SM; integer re-rounding of the
          // double measured 4-6 / clk and the FP32 double-float path needs ~16 FMA-pipe ops)
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const double d = __hiloint2double(0x43300000, static_cast<int>(v[t] ^ 0x80000000u)) -
                             4503601774854144.0;
            f[t] = __double2float_rn(d * sa2);
          }
        }
        if (tr) sp_trace(p, 10, ti + (__float_as_uint(f[31]) == 0x7fffffffu ? 1 : 0));
        if (q.out_dtype == ISB_F32) {
          if (!m_ok) continue;
          float* po = static_cast<float*>(q.out) + m * q.N + nb;
          if (nv == 32 && (q.N % 4) == 0) {
#pragma unroll
            for (int t = 0; t < 32; t += 4)
              st_global_v4(po + t, __float_as_uint(f[t]), __float_as_uint(f[t + 1]),
                           __float_as_uint(f[t + 2]), __float_as_uint(f[t + 3]));
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (t < nv) po[t] = f[t];
          }
          continue;
        }
        uint32_t h[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          if (q.out_dtype == ISB_BF16) {
            const __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * t], f[2 * t + 1]);
            h[t] = *reinterpret_cast<const uint32_t*>(&b);
          } else {
            const __half2 b = __floats2half2_rn(f[2 * t], f[2 * t + 1]);
            h[t] = *reinterpret_cast<const uint32_t*>(&b);
          }
        }
        if (dbg & 128) {  // measurement: no stores (wrong results)
          if ((h[0] ^ h[7] ^ h[15]) == 0x12345u && m_ok) static_cast<uint16_t*>(q.out)[m * q.N + nb] = 0;
          continue;
        }
        if (q.N % 8 == 0 && nb + 32 <= q.N) {
          // Transpose through this warp's staging buffer so that each 16-byte store of a
          // warp covers 8 tokens x 64 contiguous bytes (instead of 32 scattered 16-byte
          // pieces): lane l writes token l's four 16-byte quads (rotated by l/2: bank-
          // conflict-free), then reads quad l%4 of token 8i + l/4.
          const uint32_t stg = smem_u32(smem_o + ew * C::kStage);
          const int64_t mw = m - lane;  // token of lane 0
#pragma unroll
          for (int half = 0; half < 32 / C::kStageTok; ++half) {
            const int tl = static_cast<int>(lane) - half * C::kStageTok;  // row in the buffer
            if (tl >= 0 && tl < C::kStageTok) {
#pragma unroll
              for (int qq = 0; qq < 4; ++qq)
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 stg + tl * 64 + (((qq + (tl >> 1)) & 3) * 16)),
                             "r"(h[4 * qq]), "r"(h[4 * qq + 1]), "r"(h[4 * qq + 2]),
                             "r"(h[4 * qq + 3])
                             : "memory");
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < C::kStageTok / 8; ++i) {
              const uint32_t tk = 8 * i + lane / 4, pq = lane % 4;
              const uint4 d = ld_shared_v4(stg + tk * 64 + (((pq + (tk >> 1)) & 3) * 16));
              const int64_t tok = mw + half * C::kStageTok + tk;
              if (tok < q.M)
                st_global_v4(static_cast<uint16_t*>(q.out) + tok * q.N + nb + pq * 8, d.x, d.y,
                             d.z, d.w);
            }
            __syncwarp();
          }
          if (tr) sp_trace(p, 11, ti);
        } else if (m_ok) {
          uint16_t* po = static_cast<uint16_t*>(q.out) + m * q.N + nb;
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (t < nv) po[t] = static_cast<uint16_t>(h[t / 2] >> (16 * (t & 1)));
        }
      }
    }
  }

  tc_fence_before();
  cluster_sync_all();  // no peer arrives on our barriers after this point
  if (warp == alloc_warp)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512)
                 : "memory");
}

#ifndef ISB_SP_NW
#define ISB_SP_NW 8
#endif
#ifndef ISB_SP_NB
#define ISB_SP_NB 8
#endif
#ifndef ISB_SP_NXW
#define ISB_SP_NXW 4
#endif
constexpr int kSpSX = 3, kSpNXW = ISB_SP_NXW, kSpEW = 4, kSpWPB = 1, kSpNW = ISB_SP_NW, kSpNB = ISB_SP_NB;
using SpC = SpCfg<kSpSX, kSpNXW, kSpEW, kSpWPB, kSpNW, kSpNB>;
#define ISB_SP_KERNEL gemm_w4a8_sp<kSpSX, kSpNXW, kSpEW, kSpWPB, kSpNW, kSpNB>

void launch_sp_raw(const SpMaps& maps, const SpParams& prm, int clusters, cudaStream_t s) {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(ISB_SP_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    SpC::kSmem),
               "cudaFuncSetAttribute(sp smem)");
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(SpC::kThreads);
  cfg.dynamicSmemBytes = SpC::kSmem;
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
  cuda_check(cudaLaunchKernelEx(&cfg, ISB_SP_KERNEL, maps, prm), "gemm_w4a8_sp launch");
  count_launch();
}

SpProb make_sp_prob(const int8_t* xq, const double* sa, int64_t m, const isb_weight& w, void* out,
                    int out_dtype, CUtensorMap* map) {
  SpProb q{};
  q.packed = w.packed;
  q.kscale = w.kscale_tiled;
  q.sa = sa;
  q.out = out;
  q.inv_amp = std::ldexp(1.0, -w.exponent);
  q.M = static_cast<int>(m);
  q.N = static_cast<int>(w.n);
  q.G = static_cast<int>(w.groups);
  q.gb = static_cast<int>(w.group / kBlockK);
  q.kblocks = static_cast<int>(w.kblocks);
  q.m_tiles = static_cast<int>((m + kSpT - 1) / kSpT);
  q.n_tiles = static_cast<int>(w.n_tiles);
  q.out_dtype = out_dtype;
  *map = make_x_map(xq, m, w.k, 128);
  return q;
}

}  // namespace

void launch_gemm_sp(const int8_t* xq, const double* sa, int64_t m, const isb_weight& w, void* out,
                    int out_dtype, int num_sms, cudaStream_t s) {
  SpMaps maps{};
  SpParams prm{};
  prm.prob[0] = make_sp_prob(xq, sa, m, w, out, out_dtype, &maps.x[0]);
  prm.nprob = 1;
  prm.units = prm.prob[0].n_tiles * prm.prob[0].m_tiles;
  prm.dbg = g_dbg;
  prm.trace = g_trace;
  launch_sp_raw(maps, prm, std::min(prm.units, num_sms / 2), s);
}

// ---------------------------------------------------------------------------
// Grouped prefill launch: the pair tiles of up to kSpMaxProb fold-eligible GEMMs (a
// layer's linears) in one persistent launch, dealt longest-first (K blocks) to the
// least-loaded cluster (LPT), so one GEMM's last wave fills with the next GEMM's tiles.
struct SpGroupPlan {
  SpMaps maps{};
  SpParams prm{};
  int clusters = 0;
  int4* d_items = nullptr;
  int* d_off = nullptr;
  int64_t makespan_blocks = 0, total_blocks = 0;
};

SpGroupPlan* sp_group_create(const isb_group_problem* probs, int nprob, int out_dtype, int num_sms) {
  if (nprob < 1 || nprob > kSpMaxProb) fail(ISB_PARAM, "grouped prefill: 1..8 problems");
  auto* pl = new SpGroupPlan();
  try {
    pl->clusters = num_sms / 2;
    struct Tile {
      int prob, nt, mt, cost;
    };
    std::vector<Tile> tiles;
    for (int i = 0; i < nprob; ++i) {
      const isb_group_problem& g = probs[i];
      pl->prm.prob[i] = make_sp_prob(g.xq, g.sa, g.m, *g.w, g.out, out_dtype, &pl->maps.x[i]);
      const SpProb& q = pl->prm.prob[i];
      for (int nt = 0; nt < q.n_tiles; ++nt)
        for (int mt = 0; mt < q.m_tiles; ++mt) tiles.push_back({i, nt, mt, q.kblocks});
    }
    pl->prm.nprob = nprob;
    std::stable_sort(tiles.begin(), tiles.end(),
                     [](const Tile& a, const Tile& b) { return a.cost > b.cost; });
    const int C = pl->clusters;
    std::vector<std::vector<int4>> per(C);
    std::vector<int64_t> load(C, 0);
    for (const Tile& t : tiles) {
      int best = 0;
      for (int c = 1; c < C; ++c)
        if (load[c] < load[best]) best = c;
      per[best].push_back(make_int4(t.prob, t.nt, t.mt, 0));
      load[best] += t.cost;
      pl->total_blocks += t.cost;
    }
    std::vector<int4> items;
    std::vector<int> off(C + 1, 0);
    for (int c = 0; c < C; ++c) {
      off[c] = static_cast<int>(items.size());
      items.insert(items.end(), per[c].begin(), per[c].end());
    }
    off[C] = static_cast<int>(items.size());
    pl->makespan_blocks = *std::max_element(load.begin(), load.end());
    cuda_check(cudaMalloc(&pl->d_items, std::max<size_t>(1, items.size()) * sizeof(int4)),
               "cudaMalloc(grouped prefill items)");
    cuda_check(cudaMalloc(&pl->d_off, off.size() * sizeof(int)), "cudaMalloc(grouped prefill off)");
    cuda_check(cudaMemcpy(pl->d_items, items.data(), items.size() * sizeof(int4),
                          cudaMemcpyHostToDevice),
               "cudaMemcpy(grouped prefill items)");
    cuda_check(cudaMemcpy(pl->d_off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice),
               "cudaMemcpy(grouped prefill off)");
    pl->prm.items = pl->d_items;
    pl->prm.item_off = pl->d_off;
  } catch (...) {
    sp_group_destroy(pl);
    throw;
  }
  return pl;
}

void sp_group_run(SpGroupPlan* pl, cudaStream_t s) {
  pl->prm.dbg = g_dbg;
  pl->prm.trace = g_trace;
  launch_sp_raw(pl->maps, pl->prm, pl->clusters, s);
}

double sp_group_balance(const SpGroupPlan* pl) {
  return pl->makespan_blocks > 0
             ? static_cast<double>(pl->total_blocks) / (pl->clusters * static_cast<double>(pl->makespan_blocks))
             : 0.0;
}

void sp_group_destroy(SpGroupPlan* pl) {
  if (!pl) return;
  cudaFree(pl->d_items);
  cudaFree(pl->d_off);
  delete pl;
}

}  // namespace isb
