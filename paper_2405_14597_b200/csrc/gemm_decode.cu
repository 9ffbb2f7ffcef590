// K3d / K4d — decode-shaped (M <= 32) W4A8 group GEMM: stream-K over all SMs,
// sized so two CTAs fit on one SM (the next launch's CTA co-resides with ours).
//
// Reference: gemm_integer_scale (gemm.cpp:205-262, paper Eq. 2) and
// gemm_float_scale (gemm.cpp:156-203, Eq. 1). Same arithmetic as gemm_tc.cu.
//
// Work split (stream-K). The work is U = n_tiles x G units (tile = 128 output
// channels, unit = one quantization group of one tile). CTA c of P owns units
// [c U/P, (c+1) U/P) in tile-major order, so every SM streams the same number of
// weight bytes (+-1 group) whatever N, K and the SM count are. A CTA's range
// splits at tile boundaries into segments (at most one leading and one trailing
// partial segment, full tiles in between). A full-tile segment finalises
// directly. A partial segment's int32 (Eq. 2) or fp32 (Eq. 1) accumulator is
// added into the tile's workspace accumulator with ONE bulk reduction
// (cp.reduce.async.bulk .add, performed in L2) by a fix-up warp, which then
// bumps the tile's arrival counter; the last arriver reads the accumulator back,
// applies the epilogue, stores the tile and re-zeroes accumulator and counter
// (the workspace is left clean for the next launch). Integer addition is
// associative, so the int32 accumulator is bit-exactly the reference's `acc`.
//
// Pipeline granularity. Measured on B200 (scripts/trace_decode.py, ncu source
// view): per-block barrier hand-offs cap a single-warpgroup pipeline near
// 5 TB/s, so everything moves in steps of S consecutive 128-K blocks of one
// segment: one bulk copy of the S packed-int4 blocks (contiguous in HBM), S
// activation TMA boxes and one bulk copy of the step's group scales, all
// completing on one barrier; one transform hand-off, one MMA batch, one
// epilogue hand-off per step.
//
// Residency. <= 113 KB shared memory, 256 TMEM columns and 384 threads x <= 80
// registers, so the NEXT kernel's CTA fits beside ours on every SM: with
// programmatic dependent launch it initialises and streams its first weight
// steps (static data, fetched before griddepcontrol.wait) under our tail.
//
// Roles (12 warps):
//   warp 0      producer
//   warp 1      MMA      : 4 x tcgen05.mma.kind::i8 (128 x MT x 32) per block, A from TMEM
//   warps 2-3   fix-up   : (warp 2 also allocates TMEM) partial segments
//   warps 4-7   transform: smem int4 -> TMEM int8 (16 x code), thread r = channel r
//   warps 8-11  epilogue : per group tcgen05.ld of 16 P_g, Eq. 2 acc += P_g k_g
//                          (int32 IMAD) or Eq. 1 acc += float(P_g) s_g (FFMA)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

#ifndef ISB_DEC_ONE
#define ISB_DEC_ONE 1
#endif
template <int MT>
struct DCfg {
#if ISB_DEC_ONE
  // One CTA per SM: the whole SM's shared memory / TMEM for a deep pipeline.
  static constexpr int kMinBlocks = 1;
  static constexpr int kXWG = 2;                           // transform warpgroups (alternate steps)
  static constexpr int S = 4;                              // 128-K blocks per step
  static constexpr int kStages = MT <= 16 ? 4 : 3;
  static constexpr int kNA = 2;
  static constexpr int kND = 2;
  static constexpr int kTmemCols = 512;
  static constexpr int kSmemMax = 227 * 1024;
#else
  static constexpr int kMinBlocks = 2;
  static constexpr int kXWG = 1;
  static constexpr int S = MT <= 16 ? 3 : 2;               // 128-K blocks per step
  static constexpr int kStages = 3;
  static constexpr int kNA = 2;                            // TMEM A ring (steps of S x 32 cols)
  static constexpr int kND = MT <= 16 ? 1 : 2;             // TMEM D ring (steps of S x MT cols)
  static constexpr int kTmemCols = 256;
  static constexpr int kSmemMax = 112 * 1024;
#endif
  static constexpr int kThreads = 128 + 128 * kXWG + 128;
  static constexpr int kXTile = MT * 128;                  // activation bytes per block
  static constexpr int kOffX = S * kBlockBytes;            // stage: [S W][S X] (1 KiB multiple)
  static constexpr int kStageAl = kOffX + S * kXTile;
  static_assert(kStageAl % 1024 == 0, "SW128 activation tiles need 1 KiB alignment");
  static constexpr int kScStage = S * kTileN * 4;          // the step's group scales (own ring)
  static constexpr int kPart = MT * kTileN * 4;            // one published partial
  static constexpr int kDCol = kNA * S * 32;
  static_assert(kNA * S * 32 + kND * S * MT <= kTmemCols, "TMEM budget");
  static constexpr int kOffSc = kStages * kStageAl;
  static constexpr int kOffPart = kOffSc + kStages * kScStage;
  static constexpr int kOffSa = kOffPart + 2 * kPart;
  static constexpr int kOffBar = kOffSa + MT * 8;
  static constexpr int kBars = 2 * kStages + 2 * kNA + 2 * kND + 4 + 1;
  static constexpr int kSmemBytes = 1024 + kOffBar + kBars * 8 + 16;
  static_assert(kSmemBytes <= kSmemMax, "shared memory budget");
};

struct DParams {
  const uint8_t* packed;   // [n_tiles][kblocks][8 KiB]
  const int32_t* scale;    // [n_tiles][G][128]: int32 k_g (Eq. 2) or float s_g/16 (Eq. 1)
  const double* sa;        // [M]
  void* out;               // [M][N]
  uint32_t* acc;           // workspace: [T][MT][128] tile accumulators (left zero)
  uint32_t* cnt;           // workspace: [T] arrival counters (left zero)
  int M, N, G, gb, kblocks, T, out_dtype, P;
  double inv_amp;          // 2^-e (exact)
  int late_shift;          // 16 * static bound fits int32: shift 16*acc once at the end
  int64_t* trace;          // optional debug timeline (isb_debug_set_trace)
  int trace_cta;
};

#define DTRACE(role, i)                                                \
  do {                                                                 \
    if (p.trace != nullptr && cta == p.trace_cta && (i) < 512)         \
      p.trace[(role) * 512 + (i)] = clock64_();                        \
  } while (0)

__device__ __forceinline__ void store_out_d(void* out, int dtype, int64_t idx, float f) {
  if (dtype == ISB_I32) return;  // raw accumulators are stored by store_acc_or_out
  if (dtype == ISB_F32)
    static_cast<float*>(out)[idx] = f;
  else if (dtype == ISB_BF16)
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
  else
    static_cast<__half*>(out)[idx] = __float2half_rn(f);
}

template <int PATH>
__device__ __forceinline__ float finish_d(uint32_t accbits, double sa, double inv_amp) {
  double o;
  if (PATH == ISB_PATH_INTEGER_SCALE)  // Eq. 2: (acc / 2^e) * s_a, /2^e exact
    o = __dmul_rn(static_cast<double>(static_cast<int32_t>(accbits)) * inv_amp, sa);
  else                                 // Eq. 1: acc already carries s_g
    o = __dmul_rn(static_cast<double>(__uint_as_float(accbits)), sa);
  return __double2float_rn(o);
}

// Eq. 2 / Eq. 1 epilogue store, or the raw int32 accumulator (ISB_I32, row-parallel TP).
template <int PATH>
__device__ __forceinline__ void store_acc_or_out(const DParams& p, int64_t idx, uint32_t accbits,
                                                 double sa) {
  if (PATH == ISB_PATH_INTEGER_SCALE && p.out_dtype == ISB_I32)
    static_cast<uint32_t*>(p.out)[idx] = accbits;
  else
    store_out_d(p.out, p.out_dtype, idx, finish_d<PATH>(accbits, sa, p.inv_amp));
}

// Number of CTAs whose range touches tile t (each contributes one segment).
__device__ __forceinline__ int expected_arrivals(const DParams& p, int t) {
  const int64_t U = static_cast<int64_t>(p.T) * p.G;
  const int64_t u0 = static_cast<int64_t>(t) * p.G, u1 = u0 + p.G - 1;
  return static_cast<int>(((u1 + 1) * p.P - 1) / U - ((u0 + 1) * p.P - 1) / U + 1);
}

// The CTA's segments (maximal runs of its unit range inside one tile), int32.
struct SegIter {
  int u, b, G;
  __device__ SegIter(const DParams& p, int cta) {
    const int64_t U = static_cast<int64_t>(p.T) * p.G;
    u = static_cast<int>(cta * U / p.P);
    b = static_cast<int>((cta + 1) * U / p.P);
    G = p.G;
  }
  __device__ bool next(int& t, int& g0, int& ng) {
    if (u >= b) return false;
    t = u / G;
    g0 = u - t * G;
    ng = min(G - g0, b - u);
    u += ng;
    return true;
  }
};

template <int MT, int PATH, bool GB1>
__global__ void __launch_bounds__(DCfg<MT>::kThreads, DCfg<MT>::kMinBlocks)
    gemm_w4a8_decode(const __grid_constant__ CUtensorMap x_map, const DParams p) {
  using Cf = DCfg<MT>;
  constexpr int S = Cf::S;
  constexpr int kStages = Cf::kStages;
  constexpr int kNA = Cf::kNA;
  constexpr int kND = Cf::kND;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* spart = smem + Cf::kOffPart;
  double* ssa = reinterpret_cast<double*>(smem + Cf::kOffSa);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cf::kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* a_full = empty + kStages;
  uint64_t* a_empty = a_full + kNA;
  uint64_t* d_full = a_empty + kNA;
  uint64_t* d_empty = d_full + kND;
  uint64_t* ps_full = d_empty + kND;
  uint64_t* ps_empty = ps_full + 2;
  uint64_t* sa_full = ps_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sa_full + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int cta = static_cast<int>(blockIdx.x);
  const int gb = GB1 ? 1 : p.gb;

  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&x_map);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 4 + 1 + 4);  // transform warps (W), MMA commit (X), epilogue (scales)
    }
    for (int i = 0; i < kNA; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kND; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ps_full[i], 4);
      mbar_init(&ps_empty[i], 1);
    }
    mbar_init(sa_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cf::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (elect_one()) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      SegIter it(p, cta);
      int t = 0, g0 = 0, ng = 0, bi = 0, nb = 0, js = 0;
      // Weights + scales of a step (static data).
      auto issue_static = [&](int stage, int kb, int n) {
        const int ga = kb / gb, gz = (kb + n - 1) / gb;
        uint8_t* st = smem + stage * Cf::kStageAl;
        mbar_arrive_expect_tx(&full[stage],
                              n * (kBlockBytes + Cf::kXTile) + (gz - ga + 1) * kTileN * 4);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(st)),
            "l"(p.packed + (static_cast<int64_t>(t) * p.kblocks + kb) * kBlockBytes),
            "r"(n * kBlockBytes), "r"(smem_u32(&full[stage])), "l"(policy)
            : "memory");
        bulk_load(smem + Cf::kOffSc + stage * Cf::kScStage, p.scale + (static_cast<int64_t>(t) * p.G + ga) * kTileN,
                  (gz - ga + 1) * kTileN * 4, &full[stage]);
      };
      // Steps of the first kStages: weights before the wait, activations after.
      int pre_kb[kStages], pre_n[kStages], npre = 0;
      while (true) {
        if (bi == nb) {
          if (!it.next(t, g0, ng)) break;
          bi = 0;
          nb = ng * gb;
        }
        const int n = min(S, nb - bi);
        const int kb = g0 * gb + bi;
        const int stage = js % kStages;
        if (js < kStages) {
          issue_static(stage, kb, n);
          pre_kb[js] = kb;
          pre_n[js] = n;
          npre = js + 1;
          if (js + 1 == kStages) {
            pdl_wait();
            for (int q = 0; q < npre; ++q)
              for (int i = 0; i < pre_n[q]; ++i)
                tma_load_2d(smem + q * Cf::kStageAl + Cf::kOffX + i * Cf::kXTile, &x_map,
                            &full[q], (pre_kb[q] + i) * kBlockK, 0);
          }
        } else {
          mbar_wait(&empty[stage], ((js / kStages) & 1) ^ 1);
          issue_static(stage, kb, n);
          for (int i = 0; i < n; ++i)
            tma_load_2d(smem + stage * Cf::kStageAl + Cf::kOffX + i * Cf::kXTile, &x_map,
                        &full[stage], (kb + i) * kBlockK, 0);
        }
        DTRACE(0, js);
        bi += n;
        ++js;
      }
      if (npre < kStages) {  // fewer steps than stages: activations of all of them now
        pdl_wait();
        for (int q = 0; q < npre; ++q)
          for (int i = 0; i < pre_n[q]; ++i)
            tma_load_2d(smem + q * Cf::kStageAl + Cf::kOffX + i * Cf::kXTile, &x_map, &full[q],
                        (pre_kb[q] + i) * kBlockK, 0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc_i8(128, MT);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    SegIter it(p, cta);
    int js = 0, t, g0, ng;
    while (it.next(t, g0, ng)) {
      const int nb = ng * gb;
      for (int i0 = 0; i0 < nb; i0 += S, ++js) {
        const int n = min(S, nb - i0);
        const int stage = js % kStages, as = js % kNA, ds = js % kND;
        mbar_wait(&a_full[as], (js / kNA) & 1);  // transform saw full[stage]: X landed too
        mbar_wait(&d_empty[ds], ((js / kND) & 1) ^ 1);
        tc_fence_after();
        const uint32_t xs = smem_u32(smem + stage * Cf::kStageAl + Cf::kOffX);
#pragma unroll
        for (int i = 0; i < S; ++i) {
          if (i < n) {
            const uint64_t bdesc = make_sw128_kmajor_desc(xs + i * Cf::kXTile);
            const uint32_t d_tmem = tbase + Cf::kDCol + (ds * S + i) * MT;
            const uint32_t a_tmem = tbase + (as * S + i) * 32;
#pragma unroll
            for (int c = 0; c < 4; ++c)
              mma_i8_ts_warp(d_tmem, a_tmem + c * 8, bdesc + static_cast<uint64_t>(c * 2), idesc,
                             c > 0 ? 1u : 0u);
          }
        }
        mma_commit_warp(&empty[stage]);
        mma_commit_warp(&a_empty[as]);
        mma_commit_warp(&d_full[ds]);
        if (lane == 0) DTRACE(2, js);
      }
    }
  } else if (warp >= 4 && warp < 4 + 4 * Cf::kXWG) {
    // ------------------------------------------------------------------ transform
    const int xw = static_cast<int>(warp - 4) / 4;  // warpgroup xw takes steps js % kXWG == xw
    const uint32_t r = (warp % 4) * 32 + lane;      // output channel within the tile == TMEM lane
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    SegIter it(p, cta);
    int js = 0, t, g0, ng;
    while (it.next(t, g0, ng)) {
      const int nb = ng * gb;
      for (int i0 = 0; i0 < nb; i0 += S, ++js) {
        if (js % Cf::kXWG != xw) continue;
        const int n = min(S, nb - i0);
        const int stage = js % kStages, as = js % kNA;
        mbar_wait(&full[stage], (js / kStages) & 1);
        if (lane == 0 && warp == 4) DTRACE(7, js);
        const uint32_t w_base = smem_u32(smem + stage * Cf::kStageAl) + r * 16;
        uint4 qv[S][4];
#pragma unroll
        for (int i = 0; i < S; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (i < n) qv[i][c] = ld_shared_v4(w_base + i * kBlockBytes + c * (kTileN * 16));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the async refill
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        mbar_wait(&a_empty[as], ((js / kNA) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < S; ++i) {
          if (i < n) {
            uint32_t a[32];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t w4[4] = {qv[i][c].x, qv[i][c].y, qv[i][c].z, qv[i][c].w};
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                a[c * 8 + 2 * w] = (w4[w] << 4) & 0xF0F0F0F0u;  // 16 * code(k0 .. k0+3)
                a[c * 8 + 2 * w + 1] = w4[w] & 0xF0F0F0F0u;     // 16 * code(k0+4 .. k0+7)
              }
            }
            tmem_st_x32(tmem_base + lane_base + (as * S + i) * 32, a);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[as]);
        if (lane == 0 && warp == 4) DTRACE(1, js);
      }
    }
  } else if (warp >= 4 + 4 * Cf::kXWG) {
    // ------------------------------------------------------------------ epilogue
    const uint32_t ew = warp - (4 + 4 * Cf::kXWG);
    const uint32_t r = ew * 32 + lane;  // TMEM lane == output channel within the tile
    const uint32_t lane_base = (ew * 32) << 16;
    const bool late = p.late_shift != 0;
    SegIter it(p, cta);
    int js = 0, pidx = 0, t, g0, ng;
    while (it.next(t, g0, ng)) {
      const bool whole = g0 == 0 && ng == p.G;
      int32_t iacc[MT], gsum[MT];  // gsum: 16 * P_g of the open group (g > 128 spans blocks)
      float facc[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        iacc[m] = 0;
        facc[m] = 0.0f;
      }
      const int nb = ng * gb;
      for (int i0 = 0; i0 < nb; i0 += S, ++js) {
        const int n = min(S, nb - i0);
        const int stage = js % kStages, ds = js % kND;
        const int ga = (g0 * gb + i0) / gb;  // first group of the step (its scales' base)
        mbar_wait(&d_full[ds], (js / kND) & 1);
        tc_fence_after();
        const uint32_t sc_base = smem_u32(smem + Cf::kOffSc + stage * Cf::kScStage) + r * 4;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          if (i >= n) break;
          const int kb = g0 * gb + i0 + i;
          const bool gfirst = GB1 || (kb % gb == 0);
          const bool glast = GB1 || (kb % gb == gb - 1);
          uint32_t v[MT];
#pragma unroll
          for (int cc = 0; cc < MT; cc += 16)
            tmem_ld_x16_(tmem_base + lane_base + Cf::kDCol + (ds * S + i) * MT + cc,
                         *reinterpret_cast<uint32_t(*)[16]>(&v[cc]));
          tmem_wait_ld();
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            int32_t d = static_cast<int32_t>(v[m]);  // 16 * (partial of this block), exact
            if (!gfirst) d += gsum[m];
            gsum[m] = d;
          }
          if (glast) {
            const uint32_t sraw = ld_shared_u32(sc_base + (kb / gb - ga) * (kTileN * 4));
            const int32_t kg = static_cast<int32_t>(sraw);
            const float sg = __uint_as_float(sraw);
#pragma unroll
            for (int m = 0; m < MT; ++m) {
              if (PATH == ISB_PATH_INTEGER_SCALE) {
                if (late) iacc[m] += gsum[m] * kg;  // Eq. 2 in int32 (x16 removed at the end)
                else iacc[m] += (gsum[m] >> 4) * kg;
              } else {
                facc[m] = fmaf(static_cast<float>(gsum[m]), sg, facc[m]);  // Eq. 1, s_g/16
              }
            }
          }
        }
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // scale reads before refill
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&d_empty[ds]);
          mbar_arrive(&empty[stage]);
        }
        if (r == 0) DTRACE(3, js);
      }
      // ---- segment complete
      if (PATH == ISB_PATH_INTEGER_SCALE && late) {
#pragma unroll
        for (int m = 0; m < MT; ++m) iacc[m] >>= 4;  // exact: 16 | acc
      }
      if (whole) {
        mbar_wait(sa_full, 0);
        const int64_t nn = static_cast<int64_t>(t) * kTileN + r;
        if (nn < p.N) {
#pragma unroll
          for (int m = 0; m < MT; ++m)
            if (m < p.M)
              store_acc_or_out<PATH>(p, static_cast<int64_t>(m) * p.N + nn,
                                     PATH == ISB_PATH_INTEGER_SCALE
                                         ? static_cast<uint32_t>(iacc[m])
                                         : __float_as_uint(facc[m]),
                                     ssa[m]);
        }
      } else {
        // Publish [MT][128] x 32-bit into staging slot pidx & 1 (owned by fix-up
        // warp 2 + (pidx & 1)), which bulk-reduces it into the tile accumulator.
        const int w = pidx & 1, k = pidx >> 1;
        mbar_wait(&ps_empty[w], (k & 1) ^ 1);
        const uint32_t pb = smem_u32(spart + w * Cf::kPart) + r * 4;
#pragma unroll
        for (int m = 0; m < MT; ++m)
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(pb + m * (kTileN * 4)),
                       "r"(PATH == ISB_PATH_INTEGER_SCALE ? static_cast<uint32_t>(iacc[m])
                                                          : __float_as_uint(facc[m]))
                       : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&ps_full[w]);
        ++pidx;
      }
    }
  } else {
    // ------------------------------------------------------------------ fix-up (warps 2, 3)
    const int fw = static_cast<int>(warp) - 2;
    pdl_wait();  // s_a, the output and the workspace may be in use by the preceding grid
    if (fw == 0) {
      for (int i = lane; i < MT; i += 32) ssa[i] = i < p.M ? p.sa[i] : 0.0;
      __syncwarp();
      if (lane == 0) mbar_arrive(sa_full);
    }
    mbar_wait(sa_full, 0);
    SegIter it(p, cta);
    int pidx = 0, t, g0, ng;
    while (it.next(t, g0, ng)) {
      if (g0 == 0 && ng == p.G) continue;  // whole tile: finalised by the epilogue
      const int mine = pidx++;
      if ((mine & 1) != fw) continue;
      const int k = mine >> 1;
      mbar_wait(&ps_full[fw], k & 1);
      uint32_t* acc_t = p.acc + static_cast<int64_t>(t) * (MT * kTileN);
      uint32_t* cnt_t = p.cnt + t;
      int old = 0;
      if (lane == 0) {
        const uint32_t src = smem_u32(spart + fw * Cf::kPart);
        if (PATH == ISB_PATH_INTEGER_SCALE)
          asm volatile(
              "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.s32 [%0], [%1], %2;" ::"l"(
                  acc_t),
              "r"(src), "r"(Cf::kPart)
              : "memory");
        else
          asm volatile(
              "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                  acc_t),
              "r"(src), "r"(Cf::kPart)
              : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        mbar_arrive(&ps_empty[fw]);  // staging slot reusable
        asm volatile("fence.proxy.async.global;" ::: "memory");  // async-proxy writes -> generic
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;"
                     : "=r"(old)
                     : "l"(cnt_t)
                     : "memory");
      }
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old + 1 != expected_arrivals(p, t)) continue;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");  // every lane reads after the acquire
      // Last arriver: the accumulator is complete. Finalise and re-zero, 8 token
      // rows per round trip (all loads of a chunk in flight before first use).
      const int64_t n0 = static_cast<int64_t>(t) * kTileN + lane * 4;
      constexpr int kCh = 8;
#pragma unroll 1
      for (int i0 = 0; i0 < MT; i0 += kCh) {
        uint4 v[kCh];
#pragma unroll
        for (int i = 0; i < kCh; ++i)
          v[i] = __ldcg(reinterpret_cast<const uint4*>(acc_t + (i0 + i) * kTileN + lane * 4));
#pragma unroll
        for (int i = 0; i < kCh; ++i)
          __stcg(reinterpret_cast<uint4*>(acc_t + (i0 + i) * kTileN + lane * 4),
                 make_uint4(0u, 0u, 0u, 0u));
#pragma unroll
        for (int i = 0; i < kCh; ++i) {
          if (i0 + i < p.M) {
            const uint32_t vv[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (n0 + e < p.N)
                store_acc_or_out<PATH>(p, static_cast<int64_t>(i0 + i) * p.N + n0 + e, vv[e],
                                       ssa[i0 + i]);
          }
        }
      }
      if (lane == 0)
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(cnt_t), "r"(0u) : "memory");
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, Cf::kTmemCols);
}

template <int MT, int PATH, bool GB1>
void launch_decode_mt(const CUtensorMap& map, const DParams& prm, cudaStream_t s) {
  using Cf = DCfg<MT>;
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemm_w4a8_decode<MT, PATH, GB1>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmemBytes),
               "cudaFuncSetAttribute(decode smem)");
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(prm.P);
  cfg.blockDim = dim3(Cf::kThreads);
  cfg.dynamicSmemBytes = Cf::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_decode<MT, PATH, GB1>, map, prm),
             "gemm_w4a8_decode launch");
  count_launch();
}

int decode_mt(int64_t m) { return m <= 16 ? 16 : 32; }

}  // namespace

bool decode_eligible(int64_t m, const isb_weight& w) {
  // int32 unit indices: tiles x groups must fit comfortably.
  return m >= 1 && m <= kDecodeMaxM && w.tensor_core_ok() &&
         w.n_tiles * w.groups < (int64_t{1} << 30);
}

int64_t decode_workspace_bytes(int64_t m, const isb_weight& w) {
  const int mt = decode_mt(m);
  return w.n_tiles * (mt * kTileN * 4 + 4) + 256;
}

void launch_gemm_decode(int path, const int8_t* xq, const double* sa, int64_t m,
                        const isb_weight& w, void* out, int out_dtype, void* workspace,
                        int num_sms, cudaStream_t s) {
  const int mt = decode_mt(m);
  DParams prm{};
  prm.packed = w.packed;
  prm.scale = path == ISB_PATH_INTEGER_SCALE ? w.kscale_tiled
                                             : reinterpret_cast<const int32_t*>(w.fscale_tiled);
  prm.sa = sa;
  prm.out = out;
  prm.M = static_cast<int>(m);
  prm.N = static_cast<int>(w.n);
  prm.G = static_cast<int>(w.groups);
  prm.gb = static_cast<int>(w.group / kBlockK);
  prm.kblocks = static_cast<int>(w.kblocks);
  prm.T = static_cast<int>(w.n_tiles);
  prm.out_dtype = out_dtype;
  prm.P = static_cast<int>(std::min<int64_t>(num_sms, static_cast<int64_t>(prm.T) * prm.G));
  prm.acc = static_cast<uint32_t*>(workspace);
  prm.cnt = prm.acc + static_cast<int64_t>(prm.T) * mt * kTileN;
  prm.inv_amp = std::ldexp(1.0, -w.exponent);
  prm.late_shift = (path == ISB_PATH_INTEGER_SCALE && w.static_bound > 0 &&
                    w.static_bound <= (int64_t{1} << 27) - 1) ? 1 : 0;
  prm.trace = g_trace;
  prm.trace_cta = g_trace_cta;
  const CUtensorMap map = make_x_map(xq, m, w.k, mt);
  const bool gb1 = prm.gb == 1;
#define ISB_DECODE_LAUNCH(MTV, PV)                         \
  if (gb1) launch_decode_mt<MTV, PV, true>(map, prm, s);   \
  else launch_decode_mt<MTV, PV, false>(map, prm, s);
  if (mt == 16) {
    if (path == ISB_PATH_INTEGER_SCALE) { ISB_DECODE_LAUNCH(16, ISB_PATH_INTEGER_SCALE) }
    else { ISB_DECODE_LAUNCH(16, ISB_PATH_FLOAT_SCALE) }
  } else {
    if (path == ISB_PATH_INTEGER_SCALE) { ISB_DECODE_LAUNCH(32, ISB_PATH_INTEGER_SCALE) }
    else { ISB_DECODE_LAUNCH(32, ISB_PATH_FLOAT_SCALE) }
  }
#undef ISB_DECODE_LAUNCH
}

}  // namespace isb
