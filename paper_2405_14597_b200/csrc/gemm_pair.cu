// K3 prefill on a CTA pair (tcgen05.mma.cta_group::2), integer scale folded into
// the int4 -> int8 weight expansion — the default prefill kernel (M >= 256,
// k_g <= 16), single GEMM or a whole layer's linears in one grouped launch.
//
// Reference: gemm_integer_scale (gemm.cpp:205-262), paper Eq. 2. As in
// gemm_fold.cu, sum_g k_g * P_g = sum_k x_k * (k_g(k) * w_k) and k_g * w fits
// int8 when k_g <= 16, so the tensor core accumulates the integer-scaled int32
// accumulator over the whole K (bit-identical: all partial sums are within the
// static overflow bound, which the caller gates on).
//
// Why a pair, with the weights in TMEM: a 1-CTA SS tile (gemm_fold.cu) moves per
// 128x256x32 MMA 12 KiB of operand reads + 8 KiB of activation TMA + 4 KiB of
// folded-weight stores + 4 KiB of packed-weight traffic through the SM's
// shared-memory port — more than the port carries in the MMA's 128 cycles
// (scripts/pair_bench.cu). Here the folded weights go to TMEM (tcgen05.st) and the
// pair shares the activation operand: per SM and MMA, 4 KiB of activation reads,
// 4 KiB of activation TMA and 4 KiB of packed weights.
//
// Pair tile: 256 output channels (CTA rank r owns channels 128r..128r+127 of the
// tile: its weights in its TMEM, its rows of D in its TMEM) x NT tokens (the MMA
// N; CTA r TMA-loads token rows [r*NT/2, (r+1)*NT/2) of the tile into its smem).
// TMEM per CTA: A ring NA x 32 columns + NACC x NT int32 accumulator columns.
//
//   warp 0      producer W : per 128-K block one bulk copy of the 8 KiB packed block
//                            + 512 B of k_g into this CTA's W ring.
//   warp 1      MMA (leader CTA only): 4 x tcgen05.mma.cta_group::2.kind::i8 per block,
//                            commits multicast to both CTAs.
//   warp 2      TMEM allocator (cta_group::2).
//   warp 3      producer X : TMA of this CTA's activation half (signals the leader).
//   warps 4..   transform  : XWG warpgroups; thread r expands channel r's block
//                            (k_g * int4 -> int8, fold.cuh) into the TMEM A ring.
//   then        epilogue   : EWG warpgroups; warp q of warpgroup g drains lanes
//                            32q..32q+31, tokens [g*NT/EWG, (g+1)*NT/EWG) into
//                            registers, releases the accumulator, then applies
//                            out = float(double(acc) * (s_a * 2^-e)) (one DMUL).
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

constexpr int kPairMaxProb = 8;

struct PairProb {
  const uint8_t* packed;  // [n_tiles][kblocks][8 KiB]
  const int32_t* kscale;  // [n_tiles][G][128]
  const double* sa;       // [M]
  void* out;              // [M][N]
  double inv_amp;         // 2^-e
  int M, N, G, gb, kblocks, m_tiles, n_tiles, out_dtype;
};

struct PairMaps {
  CUtensorMap x[kPairMaxProb];  // int8 activations, box 128 (K) x NT/2 rows, SWIZZLE_128B
};

struct PairParams {
  PairProb prob[kPairMaxProb];
  int nprob;
  // Work list: cluster c runs items[off[c] .. off[c+1]) = (prob, pair n-tile, m-tile).
  // nullptr: one problem, unit u = c + i * #clusters, (np, mt) = (u / m_tiles, u % m_tiles).
  const int4* items;
  const int* item_off;
  int units;  // single-problem mode
  int dbg;
  int64_t* trace;  // debug timeline (isb_debug_set_trace): [8][512] clock64 of cluster 0
};

// Debug timeline rows (cluster 0; clock64 of the recording SM).
__device__ __forceinline__ void trace_put(const PairParams& p, int row, int idx, int64_t t) {
  if (p.trace != nullptr && idx < 512 && blockIdx.x < 2)
    p.trace[(row + 16 * static_cast<int>(blockIdx.x)) * 512 + idx] = t;
}
__device__ __forceinline__ void trace_ev(const PairParams& p, int row, int idx) {
  if (p.trace != nullptr && idx < 512 && blockIdx.x < 2)
    p.trace[(row + 16 * static_cast<int>(blockIdx.x)) * 512 + idx] = clock64_();
}

template <int NT, int NACC, int NA, int SW, int SX, int XWG, int EWG, int XB, bool AS>
struct PairCfg {
  static constexpr int kXHalf = (NT / 2) * 128;  // activation half per CTA per 128-K block
  // transform warps: XWG warpgroups, or (XB == 0, one warp per block) XWG single warps
  static constexpr int kNXW = XB == 0 ? XWG : 4 * XWG;
  static constexpr int kThreads = 128 + 32 * kNXW + 128 * EWG;
  static constexpr int kABytes = AS ? 128 * 128 : 0;  // folded-weight slot in smem (SS form)
  static constexpr int kSmem = 1024 + NA * kABytes + SX * kXHalf +
                               SW * (kBlockBytes + kTileN * 4) + 2 * NT * 16 + 1024;
  static constexpr uint32_t kDCol = AS ? 0 : NA * 32;  // accumulators after the TMEM A ring
  static constexpr int kCols = NT / EWG;      // tokens per epilogue warpgroup
  static_assert(kXHalf % 1024 == 0, "SW128 tiles need 1 KiB alignment");
  static_assert(kDCol + NACC * NT <= 512, "TMEM");
  static_assert(kSmem <= 227 * 1024, "smem");
  static_assert(XB == 0 || (NA % (XWG * XB) == 0 && SW % (XWG * XB) == 0), "ring slots per transform warpgroup");
  static_assert(XB > 0 || (AS && SW > 0 && NA % XWG == 0 && SW % XWG == 0),
                "one warp per block: SS form, shared W ring, each ring slot owned by one warp "
                "(mbarrier parity tracks a lead of one phase only)");
  static_assert(kCols % 32 == 0 && (NACC > 1 || kCols <= 64), "epilogue share");
  static_assert(NT % 32 == 0 && NT <= 256, "UMMA N (cta_group::2: multiple of 16)");
};

// mbarrier wait that suspends the warp in try_wait (woken when the phase completes)
// instead of re-issuing TRYWAIT + BRA: ~20 waiting warps per SM otherwise burn ~15 % of
// the issue slots the transform and the epilogue need (ncu SASS profile: SYNCS + BRA).
__device__ __forceinline__ void pwait(uint64_t* bar, uint32_t parity, int dbg) {
  const uint32_t addr = smem_u32(bar);
  if (dbg & 512) {  // A/B: plain spin
    mbar_wait(bar, parity);
    return;
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity), "r"(0x100000)
      : "memory");
}

__device__ __forceinline__ void arrive_leader(uint64_t* bar, uint32_t rank, int cta_sem = 0) {
  if (cta_sem) {  // default semantics (release.cta), as CUTLASS's ClusterBarrier::arrive
    if (rank == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    else
      asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_u32(bar), 0))
                   : "memory");
    return;
  }
  if (rank == 0)
    asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  else
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                     mapa_shared(smem_u32(bar), 0))
                 : "memory");
}

__device__ __forceinline__ void mma2_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
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

__device__ __forceinline__ void store_one(void* out, int dtype, int64_t idx, int32_t acc,
                                          double scale) {
  if (dtype == ISB_I32) {
    static_cast<int32_t*>(out)[idx] = acc;
    return;
  }
  const float f = __double2float_rn(static_cast<double>(acc) * scale);
  if (dtype == ISB_F32)
    static_cast<float*>(out)[idx] = f;
  else if (dtype == ISB_BF16)
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
  else
    static_cast<__half*>(out)[idx] = __float2half_rn(f);
}

// Eq. 2 on the FP32 pipes: out = float((double)acc * sa2) with sa2 = s_a * 2^-e given as
// the float pair (hi, lo), hi + lo = sa2 to ~2^-48. For |acc| < 2^22, acc is exact in
// float, hi*acc is split exactly by FMA, and y = p1 + e approximates the exact product P
// to ~2^-46 relative; f = RN32(y) equals RN32(RN64(P)) (the reference's two roundings,
// gemm.cpp:252) unless P lies within ~2^-21 half-ulps of a float rounding midpoint.
// Those outputs (and |acc| >= 2^22, out-of-range magnitudes) are flagged `slow` and
// recomputed in FP64 by the caller — bit-identical either way, and the FP64 / conversion
// (XU) pipes stay free of the common case.
__device__ __forceinline__ float eq2_fast(int32_t acc, float2 s, bool& slow) {
  const float a = __int_as_float(0x4B400000 + acc) - 12582912.0f;  // exact for |acc| < 2^22
  const float p1 = __fmul_rn(a, s.x);
  const float e1 = __fmaf_rn(a, s.x, -p1);  // exact product error
  const float e = __fmaf_rn(a, s.y, e1);
  const float f = __fadd_rn(p1, e);
  const float rho = fabsf(__fsub_rn(e, __fsub_rn(f, p1)));  // |y - f|
  const uint32_t fb = __float_as_uint(f);
  const uint32_t E = fb & 0x7F800000u;
  const float hu = __uint_as_float(E - (24u << 23));       // ulp(f) / 2 (normal f)
  const float lim = (fb & 0x7FFFFFu) ? hu : 0.5f * hu;     // nearest midpoint (power of 2: below)
  slow = static_cast<uint32_t>(acc + (1 << 22)) >= (1u << 23) ||
         (E - (32u << 23)) > (220u << 23) || rho >= lim * (1.0f - 0x1p-18f);
  if (acc == 0) {  // (double)0 * sa2 = +0 exactly
    slow = false;
    return 0.0f;
  }
  return f;
}

template <int NT, int NACC, int NA, int SW, int SX, int XWG, int EWG, int XB, bool AS>
__global__ void __launch_bounds__(PairCfg<NT, NACC, NA, SW, SX, XWG, EWG, XB, AS>::kThreads, 1)
    gemm_w4a8_pair(const __grid_constant__ PairMaps maps, const __grid_constant__ PairParams p) {
  using C = PairCfg<NT, NACC, NA, SW, SX, XWG, EWG, XB, AS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;                                  // [NA][128 x 128] folded weights (AS)
  uint8_t* smem_x = smem_a + NA * C::kABytes;              // [SX][NT/2 x 128] activations
  uint8_t* smem_w = smem_x + SX * C::kXHalf;               // [SW][8 KiB] packed weights
  uint8_t* smem_sc = smem_w + SW * kBlockBytes;            // [SW][128] k_g
  double* sa_s = reinterpret_cast<double*>(smem_sc + SW * kTileN * 4);  // [2][NT] s_a * 2^-e
  float2* sf_s = reinterpret_cast<float2*>(sa_s + 2 * NT);             // [2][NT] its hi/lo floats
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sf_s + 2 * NT);     // local
  uint64_t* wempty = wfull + SW;                                    // local (transform)
  uint64_t* xfull = wempty + SW;   // leader: both halves (TMA complete_tx)
  uint64_t* xempty = xfull + SX;   // local (multicast commit)
  uint64_t* a_full = xempty + SX;  // leader: both CTAs' transform warps
  uint64_t* a_empty = a_full + NA; // local (multicast commit)
  uint64_t* d_full = a_empty + NA; // local (multicast commit)
  uint64_t* d_empty = d_full + NACC;  // leader: both CTAs' epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + NACC);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cid = static_cast<int>(blockIdx.x) / 2, ncl = static_cast<int>(gridDim.x) / 2;
  int it_begin, nunits;
  if (p.items) {
    it_begin = p.item_off[cid];
    nunits = p.item_off[cid + 1] - it_begin;
  } else {
    it_begin = 0;
    nunits = cid < p.units ? (p.units - cid + ncl - 1) / ncl : 0;
  }
  auto unit_of = [&](int it, int& pb, int& np, int& mt) {
    if (p.items) {
      const int4 u = p.items[it_begin + it];
      pb = u.x;
      np = u.y;
      mt = u.z;
    } else {
      const int u = cid + it * ncl;
      pb = 0;
      np = u / p.prob[0].m_tiles;
      mt = u % p.prob[0].m_tiles;
    }
  };

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < p.nprob; ++i) prefetch_tensormap(&maps.x[i]);
    for (int i = 0; i < SW; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], XB == 0 ? 1 : 4);
    }
    for (int i = 0; i < SX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(&a_full[i], XB == 0 ? 2 : 2 * 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 2 * 4 * EWG);
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

  if (warp == 0) {
    // ------------------------------------------------ producer: packed weights + k_g (TS)
    if (SW > 0 && elect_one()) {
      int j = 0;
      for (int it = 0; it < nunits; ++it) {
        int pb, np, mt;
        unit_of(it, pb, np, mt);
        const PairProb& q = p.prob[pb];
        const int nt = np * 2 + static_cast<int>(rank);
        for (int kb = 0; kb < q.kblocks; ++kb, ++j) {
          const int s = j % SW;
          pwait(&wempty[s], ((j / SW) & 1) ^ 1, p.dbg);
          if (nt < q.n_tiles && !(p.dbg & 32)) {
            mbar_arrive_expect_tx(&wfull[s], kBlockBytes + kTileN * 4);
            bulk_load(smem_w + s * kBlockBytes,
                      q.packed + (static_cast<int64_t>(nt) * q.kblocks + kb) * kBlockBytes,
                      kBlockBytes, &wfull[s]);
            bulk_load(smem_sc + s * kTileN * 4,
                      q.kscale + (static_cast<int64_t>(nt) * q.G + kb / q.gb) * kTileN,
                      kTileN * 4, &wfull[s]);
          } else {
            mbar_arrive(&wfull[s]);  // no channels here: the transform writes zeros
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ------------------------------------------------ producer: activation halves
    if (elect_one()) {
      const uint32_t xfull_leader = mapa_shared(smem_u32(xfull), 0);
      pdl_wait();
      int j = 0;
      for (int it = 0; it < nunits; ++it) {
        int pb, np, mt;
        unit_of(it, pb, np, mt);
        const int kbs = p.prob[pb].kblocks;
        for (int kb = 0; kb < kbs; ++kb, ++j) {
          const int s = j % SX;
          pwait(&xempty[s], ((j / SX) & 1) ^ 1, p.dbg);
          if (p.dbg & 16) {  // measurement: no activation traffic (wrong results)
            if (rank == 0) mbar_arrive(&xfull[s]);
            continue;
          }
          if (rank == 0) mbar_arrive_expect_tx(&xfull[s], 2 * C::kXHalf);  // both halves
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
              "bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_x + s * C::kXHalf)),
              "l"(reinterpret_cast<uint64_t>(&maps.x[pb])),
              "r"(xfull_leader + static_cast<uint32_t>(s) * 8u), "r"(kb * kBlockK),
              "r"(mt * NT + static_cast<int>(rank) * (NT / 2))
              : "memory");
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA)
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = make_idesc_i8(256, NT);
      const uint32_t x_base = smem_u32(smem_x);
      int j = 0;
      for (int it = 0; it < nunits; ++it) {
        int pb, np, mt;
        unit_of(it, pb, np, mt);
        const int kbs = p.prob[pb].kblocks;
        const int ds = it % NACC;
        if (!(p.dbg & 64)) pwait(&d_empty[ds], ((it / NACC) & 1) ^ 1, p.dbg);
        else mbar_wait_cluster(&d_empty[ds], ((it / NACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + C::kDCol + ds * NT;
        for (int kb = 0; kb < kbs; ++kb, ++j) {
          const int xs = j % SX, as = j % NA;
          if (!(p.dbg & 64)) pwait(&a_full[as], (j / NA) & 1, p.dbg);
          else mbar_wait_cluster(&a_full[as], (j / NA) & 1);
          trace_ev(p, 0, j);
          pwait(&xfull[xs], (j / SX) & 1, p.dbg);
          trace_ev(p, 1, j);
          tc_fence_after();
          const uint64_t bdesc = make_sw128_kmajor_desc(x_base + xs * C::kXHalf);
          if constexpr (AS) {
            const uint64_t adesc = make_sw128_kmajor_desc(smem_u32(smem_a + as * C::kABytes));
#pragma unroll
            for (int c = 0; c < 4; ++c)
              mma2_ss(d_tmem, adesc + static_cast<uint64_t>(c * 2), bdesc + static_cast<uint64_t>(c * 2),
                      idesc, (kb > 0 || c > 0) ? 1u : 0u);
          } else {
            const uint32_t a_tmem = tmem_base + as * 32;
#pragma unroll
            for (int c = 0; c < 4; ++c)
              mma2_ts(d_tmem, a_tmem + c * 8, bdesc + static_cast<uint64_t>(c * 2), idesc,
                      (kb > 0 || c > 0) ? 1u : 0u);
          }
          commit2_mc(&xempty[xs]);
          commit2_mc(&a_empty[as]);
          trace_ev(p, 2, j);
        }
        commit2_mc(&d_full[ds]);
      }
    }
    __syncwarp();
  } else if (XB == 0 && warp >= 4 && warp < 4 + C::kNXW) {
    // ------------------------------------------------ transform, one warp per block (SS
    // form): warp xw expands blocks j = xw (mod 4*XWG) — all 128 rows, 4 per lane — from
    // the shared W ring into the swizzled A ring; one proxy fence and one arrive per block
    // (releasing the W slot and publishing the A slot together).
    constexpr int kNXW = C::kNXW;
    const int xw = static_cast<int>(warp) - 4;
    int total = 0;
    for (int it = 0; it < nunits; ++it) {
      int pb, np, mt;
      unit_of(it, pb, np, mt);
      total += p.prob[pb].kblocks;
    }
    int cu = -1, cu_j0 = 0, cu_kbs = 0;
    bool valid = false;
    const uint32_t w_lane = smem_u32(smem_w) + lane * 16;
    const uint32_t sc_lane = smem_u32(smem_sc) + lane * 4;
    for (int j = xw; j < total; j += kNXW) {
      while (j >= cu_j0 + cu_kbs) {
        cu_j0 += cu_kbs;
        ++cu;
        int pb, np, mt;
        unit_of(cu, pb, np, mt);
        cu_kbs = p.prob[pb].kblocks;
        valid = np * 2 + static_cast<int>(rank) < p.prob[pb].n_tiles;
      }
      const int s = j % SW, as = j % NA;
      const bool tr = lane == 0 && warp == 4;
      int64_t t8 = tr ? clock64_() : 0;
      pwait(&wfull[s], (j / SW) & 1, p.dbg);
      pwait(&a_empty[as], ((j / NA) & 1) ^ 1, p.dbg);
      int64_t t9 = tr ? clock64_() : 0;
      const uint32_t a_slot = smem_u32(smem_a + as * C::kABytes);
#pragma unroll 1
      for (int i = 0; i < 4; ++i) {
        const uint32_t r = lane + 32 * i;
        uint32_t a[32];
        if (valid) {
          uint4 w4[4];
#pragma unroll
          for (int c = 0; c < 4; ++c)
            w4[c] = ld_shared_v4(w_lane + s * kBlockBytes + c * (kTileN * 16) + i * 512);
          const int32_t k = static_cast<int32_t>(ld_shared_u32(sc_lane + s * kTileN * 4 + i * 128));
          const FoldK f = fold_constants(k);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t wv[4] = {w4[c].x, w4[c].y, w4[c].z, w4[c].w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              if (p.dbg & 1) {  // measurement: no fold ALU (wrong results)
                a[c * 8 + 2 * w] = wv[w] ^ f.k1;
                a[c * 8 + 2 * w + 1] = wv[w];
              } else {
                fold_word(wv[w], f.k1, f.k16, f.cA, f.cB, a[c * 8 + 2 * w], a[c * 8 + 2 * w + 1]);
              }
            }
          }
        } else {
#pragma unroll
          for (int z = 0; z < 32; ++z) a[z] = 0u;
        }
        // canonical SWIZZLE_128B K-major: 16-byte chunk c of row r at r*128 + (c ^ (r & 7))*16
        const uint32_t dst = a_slot + r * 128;
        if (!(p.dbg & 2)) {
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + ((ch ^ (r & 7)) * 16)),
                         "r"(a[4 * ch]), "r"(a[4 * ch + 1]), "r"(a[4 * ch + 2]), "r"(a[4 * ch + 3])
                         : "memory");
        }
      }
      int64_t t10 = tr ? clock64_() : 0;
      // W-slot reads before its async refill; A-slot writes before the tensor core reads
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      int64_t t11 = tr ? clock64_() : 0;
      if (lane == 0) {
        mbar_arrive(&wempty[s]);
        arrive_leader(&a_full[as], rank, !(p.dbg & 64));
      }
      if (tr) {
        trace_put(p, 8, j / kNXW, t8);
        trace_put(p, 9, j / kNXW, t9);
        trace_put(p, 10, j / kNXW, t10);
        trace_put(p, 11, j / kNXW, t11);
        trace_put(p, 12, j / kNXW, clock64_());
        trace_ev(p, 5, j / kNXW);
      }
    }
  } else if (XB > 0 && AS && SW == 0 && warp >= 4 && warp < 4 + 4 * XWG) {
    // ------------------------------------------------ transform (SS form): the packed
    // weights go straight from L2 to registers (16-byte loads, one row per thread,
    // coalesced across the warp; the next block's loads are in flight while this one
    // is expanded), k_g * int4 -> int8 into the swizzled shared-memory A ring.
    const int xw = static_cast<int>(warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;  // A row == output channel of this CTA
    int total = 0;
    for (int it = 0; it < nunits; ++it) {
      int pb, np, mt;
      unit_of(it, pb, np, mt);
      total += p.prob[pb].kblocks;
    }
    int cu = -1, cu_j0 = 0, cu_kbs = 0, cu_nt = 0, cu_pb = 0;
    bool cu_valid = false;
    auto block_src = [&](int j, const uint4*& src, const int32_t*& ks) {
      while (j >= cu_j0 + cu_kbs) {
        cu_j0 += cu_kbs;
        ++cu;
        int np, mt;
        unit_of(cu, cu_pb, np, mt);
        cu_kbs = p.prob[cu_pb].kblocks;
        cu_nt = np * 2 + static_cast<int>(rank);
        cu_valid = cu_nt < p.prob[cu_pb].n_tiles;
      }
      const PairProb& q = p.prob[cu_pb];
      const int kb = j - cu_j0;
      src = cu_valid ? reinterpret_cast<const uint4*>(
                           q.packed + (static_cast<int64_t>(cu_nt) * q.kblocks + kb) * kBlockBytes) + r
                     : nullptr;
      ks = cu_valid ? q.kscale + (static_cast<int64_t>(cu_nt) * q.G + kb / q.gb) * kTileN + r : nullptr;
    };
    auto load = [&](const uint4* src, const int32_t* ks, uint4 (&w4)[4], int32_t& k) {
      if (src != nullptr && !(p.dbg & 32)) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w4[c].x), "=r"(w4[c].y), "=r"(w4[c].z), "=r"(w4[c].w)
                       : "l"(src + c * kTileN));
        asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(k) : "l"(ks));
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) w4[c] = make_uint4(0u, 0u, 0u, 0u);
        k = 0;  // k_g = 0 expands to zeros (no channels in this half of the pair tile)
      }
    };
    uint4 q4[4];
    int32_t kq = 0;
    if (xw < total) {
      const uint4* src;
      const int32_t* ks;
      block_src(xw, src, ks);
      load(src, ks, q4, kq);
    }
    const uint32_t a_row = smem_u32(smem_a) + r * 128;
    // Two blocks in flight per warp: the proxy fence below waits for every outstanding
    // memory operation of the thread, so a block's loads are issued only after the
    // previous block's fence and consumed one iteration later.
    uint4 qn[4];
    int32_t kn = 0;
    if (xw + XWG < total) {
      const uint4* src;
      const int32_t* ks;
      block_src(xw + XWG, src, ks);
      load(src, ks, qn, kn);
    }
    for (int j = xw; j < total; j += XWG) {
      uint32_t a[32];
      const FoldK f = fold_constants(kq);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t wv[4] = {q4[c].x, q4[c].y, q4[c].z, q4[c].w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          if (p.dbg & 1) {  // measurement: no fold ALU (wrong results)
            a[c * 8 + 2 * w] = wv[w] ^ f.k1;
            a[c * 8 + 2 * w + 1] = wv[w];
          } else {
            fold_word(wv[w], f.k1, f.k16, f.cA, f.cB, a[c * 8 + 2 * w], a[c * 8 + 2 * w + 1]);
          }
        }
      }
      const int as = j % NA;
      pwait(&a_empty[as], ((j / NA) & 1) ^ 1, p.dbg);
      // canonical SWIZZLE_128B K-major: 16-byte chunk c of row r at r*128 + (c ^ (r & 7))*16
      const uint32_t dst = a_row + as * C::kABytes;
      if (!(p.dbg & 2)) {
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + ((ch ^ (r & 7)) * 16)),
                       "r"(a[4 * ch]), "r"(a[4 * ch + 1]), "r"(a[4 * ch + 2]), "r"(a[4 * ch + 3])
                       : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        arrive_leader(&a_full[as], rank, !(p.dbg & 64));
        if (warp == 4) trace_ev(p, 5, j);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) q4[c] = qn[c];
      kq = kn;
      if (j + 2 * XWG < total) {
        const uint4* src;
        const int32_t* ks;
        block_src(j + 2 * XWG, src, ks);
        load(src, ks, qn, kn);
      }
    }
  } else if (XB > 0 && (!AS || SW > 0) && warp >= 4 && warp < 4 + 4 * XWG) {
    // ------------------------------------------------ transform: int4 -> k_g * w -> TMEM
    // Warpgroup xw expands groups of XB consecutive blocks (group index % XWG == xw):
    // one tcgen05.wait::st + fence + leader arrive per group, not per block.
    const int xw = static_cast<int>(warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;  // channel == TMEM lane
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t w_base = smem_u32(smem_w) + r * 16;
    const uint32_t sc_base = smem_u32(smem_sc) + r * 4;
    int total = 0;
    for (int it = 0; it < nunits; ++it) {
      int pb, np, mt;
      unit_of(it, pb, np, mt);
      total += p.prob[pb].kblocks;
    }
    int cu = -1, cu_j0 = 0, cu_kbs = 0;  // unit holding block j: [cu_j0, cu_j0 + cu_kbs)
    bool valid = false;
    for (int j0 = xw * XB; j0 < total; j0 += XWG * XB) {
      const int jn = min(j0 + XB, total);
      for (int j = j0; j < jn; ++j) {
        while (j >= cu_j0 + cu_kbs) {
          cu_j0 += cu_kbs;
          ++cu;
          int pb, np, mt;
          unit_of(cu, pb, np, mt);
          cu_kbs = p.prob[pb].kblocks;
          valid = np * 2 + static_cast<int>(rank) < p.prob[pb].n_tiles;
        }
        const int s = j % SW, as = j % NA;
        pwait(&wfull[s], (j / SW) & 1, p.dbg);
        const bool tr = lane == 0 && warp == 4;
        int64_t t8 = tr ? clock64_() : 0, t9 = 0, t10 = 0, t11 = 0;
        uint32_t a[32];
        if (valid) {
          uint4 w4[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) w4[c] = ld_shared_v4(w_base + s * kBlockBytes + c * (kTileN * 16));
          const int32_t k = static_cast<int32_t>(ld_shared_u32(sc_base + s * kTileN * 4));
          // generic-proxy reads of the slot ordered before its async-proxy refill
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&wempty[s]);
          if (tr) t9 = clock64_();
          const FoldK f = fold_constants(k);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t wv[4] = {w4[c].x, w4[c].y, w4[c].z, w4[c].w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              if (p.dbg & 1) {  // measurement: no fold ALU (wrong results)
                a[c * 8 + 2 * w] = wv[w] ^ f.k1;
                a[c * 8 + 2 * w + 1] = wv[w];
              } else {
                fold_word(wv[w], f.k1, f.k16, f.cA, f.cB, a[c * 8 + 2 * w], a[c * 8 + 2 * w + 1]);
              }
            }
          }
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(&wempty[s]);
#pragma unroll
          for (int z = 0; z < 32; ++z) a[z] = 0u;
        }
        if (tr) t10 = clock64_() + (a[0] == 0x12345678u ? 1 : 0);
        pwait(&a_empty[as], ((j / NA) & 1) ^ 1, p.dbg);
        if (tr) t11 = clock64_();
        if (tr) {
          trace_put(p, 8, j, t8);
          trace_put(p, 9, j, t9);
          trace_put(p, 10, j, t10);
          trace_put(p, 11, j, t11);
        }
        if constexpr (AS) {
          // canonical SWIZZLE_128B K-major: 16-byte chunk c of row r at r*128 + (c ^ (r & 7))*16
          const uint32_t dst = smem_u32(smem_a + as * C::kABytes) + r * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            if (!(p.dbg & 2))
              asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + ((ch ^ (r & 7)) * 16)),
                           "r"(a[4 * ch]), "r"(a[4 * ch + 1]), "r"(a[4 * ch + 2]), "r"(a[4 * ch + 3])
                           : "memory");
        } else {
          tc_fence_after();
          if (!(p.dbg & 2)) tmem_st_x32(tmem_base + lane_base + as * 32, a);  // knob 2: no stores
        }
      }
      if constexpr (AS) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
      } else {
        tmem_wait_st();
        tc_fence_before();
      }
      const int64_t t12 = clock64_();
      __syncwarp();
      if (lane == 0) {
        for (int j = j0; j < jn; ++j) arrive_leader(&a_full[j % NA], rank, !(p.dbg & 64));
        if (warp == 4) {
          trace_put(p, 12, j0, t12);
          trace_ev(p, 5, j0);
        }
      }
    }
  } else if (warp >= 4 + C::kNXW) {
    // ------------------------------------------------ epilogue
    constexpr int kCols = C::kCols;
    const uint32_t ew = warp - (4 + C::kNXW);
    const uint32_t qd = warp % 4, g = ew / 4;  // a warp reaches TMEM lanes 32 * (warp % 4) ..
    const int te = static_cast<int>(ew * 32 + lane);
    const uint32_t r = qd * 32 + lane;
    const uint32_t lane_base = (qd * 32) << 16;
    pdl_wait();
    auto sa_prefetch = [&](int it) {
      if (it < nunits) {
        int pb, np, mt;
        unit_of(it, pb, np, mt);
        const PairProb& q = p.prob[pb];
        for (int t = te; t < NT; t += 128 * EWG) {
          const int64_t m = static_cast<int64_t>(mt) * NT + t;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                           smem_u32(sa_s + (it & 1) * NT + t)),
                       "l"(q.sa + (m < q.M ? m : 0)), "r"(m < q.M ? 8 : 0)
                       : "memory");
        }
      }
      cp_async_commit();
    };
    sa_prefetch(0);
    for (int it = 0; it < nunits; ++it) {
      int pb, np, mt;
      unit_of(it, pb, np, mt);
      const PairProb& q = p.prob[pb];
      const int ds = it % NACC;
      sa_prefetch(it + 1);
      cp_async_wait<1>();
      // per token: sa2 = s_a * 2^-e (exact: a power-of-two scaling) and its (hi, lo)
      // float pair for eq2_fast (hi = NaN outside the fast path's range)
      double* sa_b = sa_s + (it & 1) * NT;
      float2* sf_b = sf_s + (it & 1) * NT;
      for (int t = te; t < NT; t += 128 * EWG) {
        const double v2 = sa_b[t] * q.inv_amp;
        sa_b[t] = v2;
        const float hi = __double2float_rn(v2);
        const float lo = __double2float_rn(v2 - static_cast<double>(hi));
        const bool ok = fabs(v2) >= 0x1p-100 && fabs(v2) <= 0x1p100;
        sf_b[t] = make_float2(ok ? hi : __int_as_float(0x7FC00000), lo);
      }
      named_bar_sync(1, 128 * EWG);
      pwait(&d_full[ds], (it / NACC) & 1, p.dbg);
      if (te == 0) trace_ev(p, 6, it);
      tc_fence_after();
      // One accumulator: drain this warp's whole share into registers, release it,
      // then convert. Two: drain and convert 32 columns at a time.
      constexpr int kCh = NACC == 1 ? kCols : 32;
      const uint32_t taddr = tmem_base + lane_base + C::kDCol + ds * NT + g * kCols;
      const int64_t n = static_cast<int64_t>(np * 2 + static_cast<int>(rank)) * kTileN + r;
      const bool n_ok = n < q.N && !(p.dbg & 4);
      // lane pairs (2i, 2i+1) store two adjacent channels as one 32-bit word
      const bool pairs = (q.out_dtype == ISB_BF16 || q.out_dtype == ISB_F16) && (q.N % 2 == 0) &&
                         static_cast<int64_t>(np * 2 + static_cast<int>(rank)) * kTileN + qd * 32 + 32 <= q.N;
#pragma unroll 1
      for (int cc = 0; cc < kCols; cc += kCh) {
        uint32_t v[kCh];
#pragma unroll
        for (int c = 0; c < kCh; c += 16)
          tmem_ld_x16_(taddr + cc + c, *reinterpret_cast<uint32_t(*)[16]>(&v[c]));
        tmem_wait_ld();
        if (cc + kCh >= kCols) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&d_empty[ds], rank, !(p.dbg & 64));
          if (te == 0) trace_ev(p, 7, it);
        }
        if (!n_ok) continue;
        const double* sa_t = sa_b + g * kCols + cc;
        const float2* sf_t = sf_b + g * kCols + cc;
        const int64_t m0 = static_cast<int64_t>(mt) * NT + g * kCols + cc;
        const int tv = q.M - m0 < kCh ? static_cast<int>(q.M - m0) : kCh;
        if (q.out_dtype == ISB_I32 || tv < kCh) {
#pragma unroll
          for (int t = 0; t < kCh; ++t)
            if (t < tv)
              store_one(q.out, q.out_dtype, (m0 + t) * q.N + n, static_cast<int32_t>(v[t]), sa_t[t]);
          continue;
        }
        float f[kCh];
        if (p.dbg & 8) {  // measurement: no conversion (wrong results)
#pragma unroll
          for (int t = 0; t < kCh; ++t) f[t] = __int_as_float(static_cast<int32_t>(v[t]));
        } else if (p.dbg & 256) {  // A/B: FP32 fast path with exact fallback (eq2_fast)
          uint64_t slow = 0;
#pragma unroll
          for (int t = 0; t < kCh; ++t) {
            bool sl;
            f[t] = eq2_fast(static_cast<int32_t>(v[t]), sf_t[t], sl);
            if (sl) slow |= 1ull << t;
          }
          if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
            for (int t = 0; t < kCh; ++t)
              if ((slow >> t) & 1)
                f[t] = __double2float_rn(static_cast<double>(static_cast<int32_t>(v[t])) * sa_t[t]);
          }
        } else {
          // Eq. 2 exactly as gemm.cpp:252: (double)acc via the 2^52 + 2^31 bias (one DADD on
          // the FP64 pipe instead of an I2F.F64 conversion), one DMUL, one F2F.F32.F64.
#pragma unroll
          for (int t = 0; t < kCh; ++t) {
            const double d = __hiloint2double(0x43300000, static_cast<int>(v[t] ^ 0x80000000u)) -
                             4503601774854144.0;
            f[t] = __double2float_rn(d * sa_t[t]);
          }
        }
        if (p.dbg & 128) {  // measurement: no stores (wrong results)
          uint32_t x = 0;
#pragma unroll
          for (int t = 0; t < kCh; ++t) x ^= __float_as_uint(f[t]);
          if (x == 0x12345u) static_cast<float*>(q.out)[0] = 0.f;
          continue;
        }
        if (q.out_dtype == ISB_F32) {
          float* po = static_cast<float*>(q.out) + m0 * q.N + n;
#pragma unroll
          for (int t = 0; t < kCh; ++t)
            asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(po + static_cast<int64_t>(t) * q.N), "f"(f[t]));
        } else if (pairs) {
          // even lane: token t, channels (n, n+1); odd lane: token t+1, channels (n-1, n)
          const bool odd = lane & 1;
          uint32_t* po = reinterpret_cast<uint32_t*>(static_cast<uint16_t*>(q.out) +
                                                     (m0 + (odd ? 1 : 0)) * q.N + (n - (odd ? 1 : 0)));
#pragma unroll
          for (int t = 0; t < kCh; t += 2) {
            const float x = __shfl_xor_sync(0xffffffffu, odd ? f[t] : f[t + 1], 1);
            const float lo = odd ? x : f[t], hi = odd ? f[t + 1] : x;
            uint32_t w;
            if (q.out_dtype == ISB_BF16) {
              const __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
              w = *reinterpret_cast<const uint32_t*>(&b);
            } else {
              const __half2 b = __floats2half2_rn(lo, hi);
              w = *reinterpret_cast<const uint32_t*>(&b);
            }
            asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(po + static_cast<int64_t>(t) * (q.N / 2)), "r"(w));
          }
        } else {
          uint16_t* po = static_cast<uint16_t*>(q.out) + m0 * q.N + n;
#pragma unroll
          for (int t = 0; t < kCh; ++t) {
            const uint16_t b = q.out_dtype == ISB_BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(f[t]))
                                                       : __half_as_ushort(__float2half_rn(f[t]));
            asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(po + static_cast<int64_t>(t) * q.N), "h"(b));
          }
        }
      }
      named_bar_sync(1, 128 * EWG);  // sa_b consumed before it is refilled
    }
  }

  tc_fence_before();
  cluster_sync_all();  // no peer arrives on our barriers after this point
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512)
                 : "memory");
}

// Configurations (ISB_PAIR_CFG): 256 (default) = 256-token tiles, folded weights in a
// shared-memory ring (SS form), double-buffered 256-column accumulators, 2 transform + 4
// epilogue warpgroups; 2562 = weights in TMEM (TS form), one accumulator; 192 = TS form,
// 192-token tiles, double-buffered accumulators.
using PairSS = PairCfg<256, 2, 6, 0, 6, 3, 2, 1, true>;
#define ISB_PAIRSS gemm_w4a8_pair<256, 2, 6, 0, 6, 3, 2, 1, true>
using Pair192 = PairCfg<192, 2, 4, 8, 8, 2, 2, 2, false>;
#define ISB_PAIR192 gemm_w4a8_pair<192, 2, 4, 8, 8, 2, 2, 2, false>
using Pair256x2 = PairCfg<256, 1, 8, 8, 6, 2, 4, 2, false>;
#define ISB_PAIR256X2 gemm_w4a8_pair<256, 1, 8, 8, 6, 2, 4, 2, false>

using PairSSR = PairCfg<256, 2, 4, 6, 4, 2, 4, 1, true>;
#define ISB_PAIRSSR gemm_w4a8_pair<256, 2, 4, 6, 4, 2, 4, 1, true>

using PairSSW = PairCfg<256, 2, 6, 6, 4, 6, 4, 0, true>;
#define ISB_PAIRSSW gemm_w4a8_pair<256, 2, 6, 6, 4, 6, 4, 0, true>

int pair_cfg() {
  static const int c = [] {
    const char* e = std::getenv("ISB_PAIR_CFG");
    return e ? std::atoi(e) : 256;
  }();
  return c;
}

template <typename K>
void set_smem_once(K kernel, int bytes, std::once_flag& once) {
  std::call_once(once, [&] {
    cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
               "cudaFuncSetAttribute(pair smem)");
  });
}

void launch_pair_raw(const PairMaps& maps, const PairParams& prm, int clusters, cudaStream_t s) {
  const int nt = pair_cfg();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters);
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
  if (nt == 2563) {
    static std::once_flag once;
    set_smem_once(ISB_PAIRSSW, PairSSW::kSmem, once);
    cfg.blockDim = dim3(PairSSW::kThreads);
    cfg.dynamicSmemBytes = PairSSW::kSmem;
    cuda_check(cudaLaunchKernelEx(&cfg, ISB_PAIRSSW, maps, prm), "gemm_w4a8_pair launch");
  } else if (nt == 2561) {
    static std::once_flag once;
    set_smem_once(ISB_PAIRSSR, PairSSR::kSmem, once);
    cfg.blockDim = dim3(PairSSR::kThreads);
    cfg.dynamicSmemBytes = PairSSR::kSmem;
    cuda_check(cudaLaunchKernelEx(&cfg, ISB_PAIRSSR, maps, prm), "gemm_w4a8_pair launch");
  } else if (nt == 2562) {
    static std::once_flag once;
    set_smem_once(ISB_PAIR256X2, Pair256x2::kSmem, once);
    cfg.blockDim = dim3(Pair256x2::kThreads);
    cfg.dynamicSmemBytes = Pair256x2::kSmem;
    cuda_check(cudaLaunchKernelEx(&cfg, ISB_PAIR256X2, maps, prm), "gemm_w4a8_pair launch");
  } else if (nt == 192) {
    static std::once_flag once;
    set_smem_once(ISB_PAIR192, Pair192::kSmem, once);
    cfg.blockDim = dim3(Pair192::kThreads);
    cfg.dynamicSmemBytes = Pair192::kSmem;
    cuda_check(cudaLaunchKernelEx(&cfg, ISB_PAIR192, maps, prm), "gemm_w4a8_pair launch");
  } else {
    static std::once_flag once;
    set_smem_once(ISB_PAIRSS, PairSS::kSmem, once);
    cfg.blockDim = dim3(PairSS::kThreads);
    cfg.dynamicSmemBytes = PairSS::kSmem;
    cuda_check(cudaLaunchKernelEx(&cfg, ISB_PAIRSS, maps, prm), "gemm_w4a8_pair launch");
  }
  count_launch();
}

PairProb make_prob(const int8_t* xq, const double* sa, int64_t m, const isb_weight& w, void* out,
                   int out_dtype, int nt, CUtensorMap* map) {
  PairProb q{};
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
  q.m_tiles = static_cast<int>((m + nt - 1) / nt);
  q.n_tiles = static_cast<int>(w.n_tiles);
  q.out_dtype = out_dtype;
  *map = make_x_map(xq, m, w.k, nt / 2);
  return q;
}

}  // namespace

int pair_tile_tokens() { return pair_cfg() == 192 ? 192 : 256; }

void launch_gemm_pair(const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                      void* out, int out_dtype, int num_sms, cudaStream_t s) {
  const int nt = pair_tile_tokens();
  PairMaps maps{};
  PairParams prm{};
  prm.prob[0] = make_prob(xq, sa, m, w, out, out_dtype, nt, &maps.x[0]);
  prm.nprob = 1;
  prm.items = nullptr;
  prm.item_off = nullptr;
  prm.units = static_cast<int>((w.n_tiles + 1) / 2) * prm.prob[0].m_tiles;
  prm.dbg = g_dbg;
  prm.trace = g_trace;
  launch_pair_raw(maps, prm, std::min(prm.units, num_sms / 2), s);
}

// ---------------------------------------------------------------------------
// Grouped prefill launch: the pair tiles of up to kPairMaxProb GEMMs (a layer's
// linears) in one persistent launch. Tiles are dealt longest-first (K blocks) to the
// least-loaded cluster (LPT), so the tail of one GEMM fills with the tiles of the
// next instead of idling a wave.
struct PairGroupPlan {
  PairMaps maps{};
  PairParams prm{};
  int clusters = 0;
  int4* d_items = nullptr;
  int* d_off = nullptr;
  double makespan_blocks = 0, mean_blocks = 0;
};

PairGroupPlan* pair_group_create(const isb_group_problem* probs, int nprob, int out_dtype,
                                 int num_sms) {
  if (nprob < 1 || nprob > kPairMaxProb) fail(ISB_PARAM, "pair group: 1..8 problems");
  const int nt = pair_tile_tokens();
  auto* pl = new PairGroupPlan();
  pl->clusters = num_sms / 2;
  struct Tile {
    int prob, np, mt, cost;
  };
  std::vector<Tile> tiles;
  for (int i = 0; i < nprob; ++i) {
    const isb_group_problem& g = probs[i];
    const isb_weight& w = *g.w;
    pl->prm.prob[i] = make_prob(static_cast<const int8_t*>(g.xq), g.sa, g.m, w, g.out,
                                out_dtype, nt, &pl->maps.x[i]);
    const PairProb& q = pl->prm.prob[i];
    for (int np = 0; np < (q.n_tiles + 1) / 2; ++np)
      for (int mt = 0; mt < q.m_tiles; ++mt) tiles.push_back({i, np, mt, q.kblocks});
  }
  pl->prm.nprob = nprob;
  // LPT: longest first; ties keep (prob, np, mt) order so neighbouring clusters share
  // weight tiles in L2.
  std::stable_sort(tiles.begin(), tiles.end(),
                   [](const Tile& a, const Tile& b) { return a.cost > b.cost; });
  const int C = pl->clusters;
  std::vector<std::vector<int4>> per(C);
  std::vector<int64_t> load(C, 0);
  int64_t total = 0;
  for (const Tile& t : tiles) {
    int best = 0;
    for (int c = 1; c < C; ++c)
      if (load[c] < load[best]) best = c;
    per[best].push_back(make_int4(t.prob, t.np, t.mt, 0));
    load[best] += t.cost;
    total += t.cost;
  }
  std::vector<int4> items;
  std::vector<int> off(C + 1, 0);
  for (int c = 0; c < C; ++c) {
    off[c] = static_cast<int>(items.size());
    items.insert(items.end(), per[c].begin(), per[c].end());
  }
  off[C] = static_cast<int>(items.size());
  pl->makespan_blocks = static_cast<double>(*std::max_element(load.begin(), load.end()));
  pl->mean_blocks = static_cast<double>(total) / C;
  cuda_check(cudaMalloc(&pl->d_items, std::max<size_t>(1, items.size()) * sizeof(int4)),
             "cudaMalloc(pair items)");
  cuda_check(cudaMalloc(&pl->d_off, off.size() * sizeof(int)), "cudaMalloc(pair off)");
  cuda_check(cudaMemcpy(pl->d_items, items.data(), items.size() * sizeof(int4),
                        cudaMemcpyHostToDevice),
             "cudaMemcpy(pair items)");
  cuda_check(cudaMemcpy(pl->d_off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice),
             "cudaMemcpy(pair off)");
  pl->prm.items = pl->d_items;
  pl->prm.item_off = pl->d_off;
  pl->prm.units = 0;
  return pl;
}

void pair_group_run(PairGroupPlan* pl, cudaStream_t s) {
  pl->prm.dbg = g_dbg;
  pl->prm.trace = g_trace;
  launch_pair_raw(pl->maps, pl->prm, pl->clusters, s);
}

double pair_group_efficiency(const PairGroupPlan* pl) {
  return pl->makespan_blocks > 0 ? pl->mean_blocks / pl->makespan_blocks : 0.0;
}

void pair_group_destroy(PairGroupPlan* pl) {
  if (!pl) return;
  cudaFree(pl->d_items);
  cudaFree(pl->d_off);
  delete pl;
}

}  // namespace isb
