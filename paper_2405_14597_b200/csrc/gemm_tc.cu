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

constexpr int kStages = 4;

template <int MT>
struct Cfg {
  static constexpr int kEpiWG = MT >= 128 ? 2 : 1;           // epilogue warpgroups
  static constexpr int kCols = MT / kEpiWG;                   // D columns per epilogue WG
  static constexpr int kThreads = 256 + 128 * kEpiWG;
  static constexpr int kNA = 4;                               // TMEM A stages (32 cols each)
  static constexpr int kND = MT >= 128 ? 3 : (MT >= 64 ? 4 : (MT >= 16 ? 4 : 8));
  static constexpr int kTmemUsed = kNA * 32 + kND * MT;
  static constexpr int kTmemCols = kTmemUsed <= 32 ? 32 : kTmemUsed <= 64 ? 64
                                   : kTmemUsed <= 128 ? 128 : kTmemUsed <= 256 ? 256 : 512;
  static_assert(kTmemUsed <= 512, "TMEM overflow");
  static constexpr int kXBytes = MT * 128;
  static constexpr int kStageBytes = kBlockBytes + kXBytes;
  static constexpr int kSmemBytes = 1024 + kStages * (kBlockBytes + (kXBytes < 1024 ? 1024 : kXBytes)) + 512;
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
};

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
  constexpr int kXSlot = C::kXBytes < 1024 ? 1024 : C::kXBytes;
  uint8_t* smem_w = smem;                                  // kStages x 8 KiB
  uint8_t* smem_x = smem + kStages * kBlockBytes;          // kStages x kXSlot (1 KiB aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_x + kStages * kXSlot);
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

  const int P = gridDim.x;
  const int64_t U = p.units;
  const int64_t u0 = (static_cast<int64_t>(blockIdx.x) * U) / P;
  const int64_t u1 = (static_cast<int64_t>(blockIdx.x + 1) * U) / P;
  const int G = p.G, gb = p.gb;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = u0; u < u1;) {
        const int tile = static_cast<int>(u / G);
        const int g0 = static_cast<int>(u % G);
        const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
        const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
        for (int kb = g0 * gb; kb < g1 * gb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kBlockBytes + C::kXBytes);
          bulk_load_evict_first(smem_w + stage * kBlockBytes,
                                p.packed + (static_cast<int64_t>(nt) * p.kblocks + kb) * kBlockBytes,
                                kBlockBytes, &full[stage]);
          tma_load_2d(smem_x + stage * kXSlot, &x_map, &full[stage], kb * kBlockK, mt * MT);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        u += g1 - g0;
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = make_idesc_i8(128, MT);
    int stage = 0, as = 0, ds = 0;
    uint32_t phase = 0, aphase = 0, dphase = 0;
    for (int64_t u = u0; u < u1;) {
      const int g0 = static_cast<int>(u % G);
      const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
      for (int g = g0; g < g1; ++g) {
        mbar_wait(&d_empty[ds], dphase ^ 1);
        const uint32_t d_tmem = tmem_base + C::kNA * 32 + ds * MT;
        for (int b = 0; b < gb; ++b) {
          mbar_wait(&full[stage], phase);
          mbar_wait(&a_full[as], aphase);
          tc_fence_after();
          if (lane == 0) {
            const uint64_t bdesc = make_sw128_kmajor_desc(smem_u32(smem_x + stage * kXSlot));
#pragma unroll
            for (int c = 0; c < 4; ++c)
              mma_i8_ts(d_tmem, tmem_base + as * 32 + c * 8, bdesc + static_cast<uint64_t>(c * 2),
                        idesc, (b > 0 || c > 0) ? 1u : 0u);
            mma_commit(&empty[stage]);
            mma_commit(&a_empty[as]);
            if (b == gb - 1) mma_commit(&d_full[ds]);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
          if (++as == C::kNA) { as = 0; aphase ^= 1; }
        }
        if (++ds == C::kND) { ds = 0; dphase ^= 1; }
      }
      u += g1 - g0;
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------------- transform
    const uint32_t r = (warp - 4) * 32 + lane;  // output channel within the tile == TMEM lane
    const uint32_t lane_base = ((warp - 4) * 32) << 16;
    int stage = 0, as = 0;
    uint32_t phase = 0, aphase = 0;
    for (int64_t u = u0; u < u1;) {
      const int g0 = static_cast<int>(u % G);
      const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
      for (int kb = g0 * gb; kb < g1 * gb; ++kb) {
        mbar_wait(&full[stage], phase);
        uint4 q[4];
        const uint8_t* src = smem_w + stage * kBlockBytes + r * 16;
#pragma unroll
        for (int c = 0; c < 4; ++c) q[c] = *reinterpret_cast<const uint4*>(src + c * (kTileN * 16));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
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
        mbar_wait(&a_empty[as], aphase ^ 1);
        tc_fence_after();
        tmem_st_x32(tmem_base + lane_base + as * 32, a);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[as]);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        if (++as == C::kNA) { as = 0; aphase ^= 1; }
      }
      u += g1 - g0;
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t ew = warp - 8;             // 0 .. 4*kEpiWG-1
    const uint32_t wg = ew / 4;               // which column half
    const uint32_t r = (ew % 4) * 32 + lane;  // TMEM lane == output channel in tile
    const uint32_t lane_base = ((ew % 4) * 32) << 16;
    const int c0 = wg * C::kCols;
    constexpr int kCols = C::kCols;
    int ds = 0;
    uint32_t dphase = 0;
    for (int64_t u = u0; u < u1;) {
      const int tile = static_cast<int>(u / G);
      const int g0 = static_cast<int>(u % G);
      const int g1 = static_cast<int>((G < g0 + (u1 - u) ? static_cast<int64_t>(G) : g0 + (u1 - u)));
      const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
      int32_t iacc[kCols];
      float facc[kCols];
#pragma unroll
      for (int t = 0; t < kCols; ++t) { iacc[t] = 0; facc[t] = 0.0f; }
      for (int g = g0; g < g1; ++g) {
        const int64_t sidx = (static_cast<int64_t>(nt) * G + g) * kTileN + r;
        int32_t kg = 0;
        float sg = 0.0f;
        if (PATH == ISB_PATH_INTEGER_SCALE) kg = __ldg(p.kscale + sidx);
        else sg = __ldg(p.fscale + sidx);
        mbar_wait(&d_full[ds], dphase);
        tc_fence_after();
        uint32_t v[kCols];
        const uint32_t taddr = tmem_base + lane_base + C::kNA * 32 + ds * MT + c0;
#pragma unroll
        for (int c = 0; c < kCols; c += 8)
          tmem_ld_x8(taddr + c, *reinterpret_cast<uint32_t(*)[8]>(&v[c]));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[ds]);
        if (++ds == C::kND) { ds = 0; dphase ^= 1; }
#pragma unroll
        for (int t = 0; t < kCols; ++t) {
          const int32_t d = static_cast<int32_t>(v[t]);  // 16 * P_g, exact
          if (PATH == ISB_PATH_INTEGER_SCALE)
            iacc[t] += (d >> 4) * kg;                      // Eq. 2: int32 scaled accumulation
          else
            facc[t] = fmaf(static_cast<float>(d), sg, facc[t]);  // Eq. 1, Atom-style fp32
        }
      }
      // ------------------------------------------------ tile completion
      const bool whole = (g0 == 0 && g1 == G);
      bool finalize = whole;
      if (!whole) {
        const int first = cta_of(static_cast<int64_t>(tile) * G, U, P);
        const int last = cta_of(static_cast<int64_t>(tile) * G + G - 1, U, P);
        const int j = blockIdx.x - first;
        int32_t* slice = p.partials + (static_cast<int64_t>(tile) * p.maxc + j) * MT * kTileN;
#pragma unroll
        for (int t = 0; t < kCols; ++t)
          slice[(c0 + t) * kTileN + r] =
              PATH == ISB_PATH_INTEGER_SCALE ? iacc[t] : __float_as_int(facc[t]);
        __threadfence();
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
        if (finalize) {
          __threadfence();
          const int nc = last - first + 1;
#pragma unroll
          for (int t = 0; t < kCols; ++t) { iacc[t] = 0; facc[t] = 0.0f; }
          for (int jj = 0; jj < nc; ++jj) {
            const int32_t* sl = p.partials + (static_cast<int64_t>(tile) * p.maxc + jj) * MT * kTileN;
#pragma unroll
            for (int t = 0; t < kCols; ++t) {
              const int32_t x = __ldcg(sl + (c0 + t) * kTileN + r);
              if (PATH == ISB_PATH_INTEGER_SCALE) iacc[t] += x;
              else facc[t] += __int_as_float(x);
            }
          }
        }
      }
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
      u += g1 - g0;
    }
  }

  tc_fence_before();
  __syncthreads();
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
  static bool attr_set = false;  // per instantiation; benign race (idempotent)
  if (!attr_set) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::kSmemBytes),
               "cudaFuncSetAttribute");
    attr_set = true;
  }
  kern<<<grid, C::kThreads, C::kSmemBytes, s>>>(map, prm);
  cuda_check(cudaGetLastError(), "gemm_w4a8_tc launch");
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

GemmPlan plan_gemm(int64_t m, const isb_weight& w, int num_sms) {
  GemmPlan pl;
  pl.mt = pick_mt(m);
  pl.m_tiles = static_cast<int>((m + pl.mt - 1) / pl.mt);
  pl.tiles = static_cast<int>(w.n_tiles) * pl.m_tiles;
  pl.units = static_cast<int64_t>(pl.tiles) * w.groups;
  pl.grid = static_cast<int>(std::min<int64_t>(num_sms, pl.units));
  pl.maxc = 1;
  for (int t = 0; t < pl.tiles; ++t) {
    const int first = host_cta_of(static_cast<int64_t>(t) * w.groups, pl.units, pl.grid);
    const int last = host_cta_of(static_cast<int64_t>(t) * w.groups + w.groups - 1, pl.units,
                                 pl.grid);
    pl.maxc = std::max(pl.maxc, last - first + 1);
  }
  const int64_t counters = round_up(static_cast<int64_t>(pl.tiles) * 4, 256);
  const int64_t partials = pl.maxc > 1
                               ? static_cast<int64_t>(pl.tiles) * pl.maxc * pl.mt * kTileN * 4
                               : 0;
  pl.workspace_bytes = counters + partials;
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
  prm.maxc = pl.maxc;
  prm.out_dtype = out_dtype;
  prm.units = pl.units;
  prm.inv_amp = std::ldexp(1.0, -w.exponent);
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
