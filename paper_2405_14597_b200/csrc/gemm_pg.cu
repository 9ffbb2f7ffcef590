// Prefill-M W4A8 group GEMM with a per-group epilogue on the shared-memory
// (SS) tcgen05 skeleton: the general integer-scale path (any k_g, e.g. alpha =
// 8192 where k_g reaches ~124 and cannot be folded into the int8 weight operand)
// and the float-scale path K4 — the paper's comparison, on the same producers,
// transform and SWIZZLE_128B rings as the folded prefill kernel (gemm_fold.cu).
//
// Reference: gemm_integer_scale (gemm.cpp:205-262): acc += P_g * k_g in integer,
// out = float((double(acc) / 2^e) * s_a); gemm_float_scale (gemm.cpp:156-203) in
// the Atom-style fp32 form: acc += float(P_g) * float(s_g), out = float(acc * s_a).
//
// Tile: 128 output channels x 128 tokens. Per 128-K block (one group, g = 128) the
// tensor core writes the group's int32 partial into one of kNP TMEM slots; four
// epilogue warpgroups (32 tokens each, one TMEM lane = one channel per thread) drain
// it and accumulate in registers
//   integer:  acc += P_g * k_g   (one IMAD; the transform expands the int4 codes
//                                 themselves, so the partial is P_g)
//   float:    acc  = fma(float(P16), s_g / 16, acc)   (I2F + FFMA; the transform
//                                 expands 16*code, two ops per word, P16 = 16 P_g)
// while the MMA fills the next slots. Roles:
//   warp 0        packed int4 weights -> W ring (bulk copies)
//   warp 1        MMA issuer (tcgen05.mma.cta_group::1.kind::i8, SS)
//   warp 2        TMEM owner + group scales -> scale ring (one slot per partial)
//   warp 3        int8 activation tiles -> X ring (TMA, SWIZZLE_128B)
//   warps 4-7     transform: int4 -> int8 (code / 16*code) into the SW128 A ring
//   warps 8-23    epilogue
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

constexpr int kPgMT = 128;                      // tokens per tile (UMMA N)
constexpr int kPgXBytes = kPgMT * 128;          // 16 KiB activation tile per block
constexpr int kPgABytes = 128 * 128;            // 16 KiB expanded weights per block
constexpr int kPgSW = 6;                        // packed-weight ring
constexpr int kPgSX = 4;                        // activation ring
constexpr int kPgNA = 4;                        // expanded-weight ring
constexpr int kPgNP = 4;                        // TMEM partial slots (128 columns each)
constexpr int kPgEW = 4;                        // epilogue warpgroups (MT / kPgEW tokens each)
constexpr int kPgThreads = 128 + 128 + 128 * kPgEW;
constexpr int kPgSmem = 1024 + kPgNA * kPgABytes + kPgSX * kPgXBytes + kPgSW * kBlockBytes +
                        kPgNP * kTileN * 4 + 4 * kPgMT * 8 + 1024;
static_assert(kPgSmem <= 227 * 1024, "smem");
static_assert(kPgNP * kPgMT <= 512, "TMEM");

struct PgParams {
  const uint8_t* packed;  // [n_tiles][kblocks][8 KiB]
  const int32_t* scale;   // [n_tiles][G][128]: int32 k_g (integer) or float s_g/16 bits
  const double* sa;       // [M]
  void* out;              // [M][N]
  int M, N, G, kblocks, m_tiles, tiles, out_dtype, late_shift;
  int kb0, kbw;  // first 128-K block of this launch, the weight's block count (K-chunked calls)
  double inv_amp;
};

__device__ __forceinline__ void pg_store(void* out, int dtype, int64_t idx, float f) {
  if (dtype == ISB_F32)
    static_cast<float*>(out)[idx] = f;
  else if (dtype == ISB_BF16)
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
  else
    static_cast<__half*>(out)[idx] = __float2half_rn(f);
}

template <int PATH>
__global__ void __launch_bounds__(kPgThreads, 1)
    gemm_w4a8_pg(const __grid_constant__ CUtensorMap x_map, const PgParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;                                  // [NA][128 x 128] int8, SW128
  uint8_t* smem_x = smem_a + kPgNA * kPgABytes;            // [SX][128 x 128] int8, SW128
  uint8_t* smem_w = smem_x + kPgSX * kPgXBytes;            // [SW][8 KiB] packed int4
  uint8_t* smem_sc = smem_w + kPgSW * kBlockBytes;         // [NP][128] group scales
  double* sa_s = reinterpret_cast<double*>(smem_sc + kPgNP * kTileN * 4);  // [2][MT]
  double* c52_s = sa_s + 2 * kPgMT;  // [2][MT] integer path: -2^52 * s_a * 2^-e per token
  uint64_t* wfull = reinterpret_cast<uint64_t*>(c52_s + 2 * kPgMT);
  uint64_t* wempty = wfull + kPgSW;
  uint64_t* xfull = wempty + kPgSW;
  uint64_t* xempty = xfull + kPgSX;
  uint64_t* a_full = xempty + kPgSX;
  uint64_t* a_empty = a_full + kPgNA;
  uint64_t* d_full = a_empty + kPgNA;
  uint64_t* d_empty = d_full + kPgNP;
  uint64_t* s_full = d_empty + kPgNP;
  uint64_t* s_empty = s_full + kPgNP;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + kPgNP);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int ntiles = static_cast<int>(blockIdx.x) < p.tiles
                         ? (p.tiles - static_cast<int>(blockIdx.x) + gridDim.x - 1) / gridDim.x
                         : 0;
  const int total = ntiles * p.kblocks;

  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&x_map);
    for (int i = 0; i < kPgSW; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], 4);
    }
    for (int i = 0; i < kPgSX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < kPgNA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kPgNP; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4 * kPgEW);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4 * kPgEW);
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
    // ------------------------------------------------ producer: packed weights
    if (elect_one()) {
      for (int j = 0; j < total; ++j) {
        const int s = j % kPgSW;
        mbar_wait(&wempty[s], ((j / kPgSW) & 1) ^ 1);
        int nt, mt;
        tile_of(j / p.kblocks, nt, mt);
        mbar_arrive_expect_tx(&wfull[s], kBlockBytes);
        bulk_load_evict_first(smem_w + s * kBlockBytes,
                              p.packed + (static_cast<int64_t>(nt) * p.kbw + p.kb0 + j % p.kblocks) *
                                             kBlockBytes,
                              kBlockBytes, &wfull[s]);
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ------------------------------------------------ producer: group scales (one per partial)
    if (elect_one()) {
      for (int j = 0; j < total; ++j) {
        const int s = j % kPgNP;
        mbar_wait(&s_empty[s], ((j / kPgNP) & 1) ^ 1);
        int nt, mt;
        tile_of(j / p.kblocks, nt, mt);
        mbar_arrive_expect_tx(&s_full[s], kTileN * 4);
        bulk_load(smem_sc + s * kTileN * 4,
                  p.scale + (static_cast<int64_t>(nt) * p.G + p.kb0 + j % p.kblocks) * kTileN, kTileN * 4,
                  &s_full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ------------------------------------------------ producer: activation tiles
    if (elect_one()) {
      pdl_wait();
      for (int j = 0; j < total; ++j) {
        const int s = j % kPgSX;
        mbar_wait(&xempty[s], ((j / kPgSX) & 1) ^ 1);
        int nt, mt;
        tile_of(j / p.kblocks, nt, mt);
        mbar_arrive_expect_tx(&xfull[s], kPgXBytes);
        tma_load_2d(smem_x + s * kPgXBytes, &x_map, &xfull[s], (p.kb0 + j % p.kblocks) * kBlockK,
                    mt * kPgMT);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer: one partial per group
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_i8(128, kPgMT);
      for (int j = 0; j < total; ++j) {
        const int xs = j % kPgSX, as = j % kPgNA, ds = j % kPgNP;
        mbar_wait(&d_empty[ds], ((j / kPgNP) & 1) ^ 1);
        mbar_wait(&a_full[as], (j / kPgNA) & 1);
        mbar_wait(&xfull[xs], (j / kPgSX) & 1);
        tc_fence_after();
        const uint64_t adesc = make_sw128_kmajor_desc(smem_u32(smem_a + as * kPgABytes));
        const uint64_t bdesc = make_sw128_kmajor_desc(smem_u32(smem_x + xs * kPgXBytes));
        const uint32_t d_tmem = tmem_base + ds * kPgMT;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          mma_i8_ss(d_tmem, adesc + static_cast<uint64_t>(c * 2), bdesc + static_cast<uint64_t>(c * 2),
                    idesc, c > 0 ? 1u : 0u);
        mma_commit(&xempty[xs]);
        mma_commit(&a_empty[as]);
        mma_commit(&d_full[ds]);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------ transform: int4 -> 16*code, SW128
    const uint32_t r = (warp % 4) * 32 + lane;  // output channel == A row
    const uint32_t w_base = smem_u32(smem_w) + r * 16;
    const uint32_t a_row = smem_u32(smem_a) + r * 128;
    for (int j = 0; j < total; ++j) {
      const int s = j % kPgSW, as = j % kPgNA;
      mbar_wait(&wfull[s], (j / kPgSW) & 1);
      uint4 q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c] = ld_shared_v4(w_base + s * kBlockBytes + c * (kTileN * 16));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the refill
      __syncwarp();
      if (lane == 0) mbar_arrive(&wempty[s]);
      uint32_t a[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t w4[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          if constexpr (PATH == ISB_PATH_INTEGER_SCALE) {
            // code itself (sign-extended nibble per byte: ((n ^ 8) + 0x78) ^ 0x80, no
            // carry leaves a byte), so the epilogue's partial is P_g and acc += P_g * k_g
            // is one IMAD per value (no >> 4)
            a[c * 8 + 2 * w] = (((w4[w] & 0x0F0F0F0Fu) ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
            a[c * 8 + 2 * w + 1] =
                ((((w4[w] >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
          } else {
            a[c * 8 + 2 * w] = (w4[w] << 4) & 0xF0F0F0F0u;  // 16*code(k0..k0+3)
            a[c * 8 + 2 * w + 1] = w4[w] & 0xF0F0F0F0u;     // 16*code(k0+4..k0+7)
          }
        }
      }
      mbar_wait(&a_empty[as], ((j / kPgNA) & 1) ^ 1);
      const uint32_t dst = a_row + as * kPgABytes;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + ((ch ^ (r & 7)) * 16)),
                     "r"(a[4 * ch]), "r"(a[4 * ch + 1]), "r"(a[4 * ch + 2]), "r"(a[4 * ch + 3])
                     : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
      named_bar_sync(2, 128);  // the whole warpgroup's rows are written and fenced
      if (warp == 4 && lane == 0) mbar_arrive(&a_full[as]);
    }
  } else {
    // ------------------------------------------------ epilogue: per-group scaling
    constexpr int kCols = kPgMT / kPgEW;             // tokens per thread
    const uint32_t ew = warp - 8;                     // 0 .. 4 * kPgEW - 1
    const uint32_t q = ew % 4, g = ew / 4;
    const int te = static_cast<int>(ew * 32 + lane);
    const uint32_t r = q * 32 + lane;                 // TMEM lane == channel in tile
    const uint32_t lane_base = (q * 32) << 16;
    pdl_wait();
    auto sa_prefetch = [&](int it) {
      if (it < ntiles) {
        int nt, mt;
        tile_of(it, nt, mt);
        if (te < kPgMT) {
          const int64_t m = static_cast<int64_t>(mt) * kPgMT + te;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                           smem_u32(sa_s + (it & 1) * kPgMT + te)),
                       "l"(p.sa + (m < p.M ? m : 0)), "r"(m < p.M ? 8 : 0)
                       : "memory");
        }
      }
      cp_async_commit();
    };
    sa_prefetch(0);
    int j = 0;
    for (int it = 0; it < ntiles; ++it) {
      int nt, mt;
      tile_of(it, nt, mt);
      sa_prefetch(it + 1);
      int32_t iacc[kCols];
      float facc[kCols];
#pragma unroll
      for (int t = 0; t < kCols; ++t) { iacc[t] = 0; facc[t] = 0.0f; }
      for (int kb = 0; kb < p.kblocks; ++kb, ++j) {
        const int ds = j % kPgNP;
        mbar_wait(&s_full[ds], (j / kPgNP) & 1);
        mbar_wait(&d_full[ds], (j / kPgNP) & 1);
        tc_fence_after();
        const uint32_t sraw = ld_shared_u32(smem_u32(smem_sc + ds * kTileN * 4) + r * 4);
        const uint32_t taddr = tmem_base + lane_base + ds * kPgMT + g * kCols;
        const int32_t k = static_cast<int32_t>(sraw);
        const float s16 = __uint_as_float(sraw);
        // 16 columns at a time: 64 accumulators + 16 loaded values stay in registers
#pragma unroll
        for (int cc = 0; cc < kCols; cc += 16) {
          uint32_t v[16];
          tmem_ld_x16_(taddr + cc, v);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int32_t d = static_cast<int32_t>(v[t]);  // P_g (integer) / 16 * P_g (float)
            if (PATH == ISB_PATH_INTEGER_SCALE)
              iacc[cc + t] += d * k;
            else
              facc[cc + t] = fmaf(static_cast<float>(d), s16, facc[cc + t]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&d_empty[ds]);
          mbar_arrive(&s_empty[ds]);
        }
      }
      // tile done: Eq. 2 / Eq. 1 per output
      cp_async_wait<1>();
      // integer path: s_a * 2^-e once per token (exact), not once per output
      // and the DFMA's addend -2^52 * sa2, also once per token (exponent arithmetic on
      // the ALU; a DMUL only for zero / subnormal / huge sa2) instead of per output
      if (PATH == ISB_PATH_INTEGER_SCALE && te < kPgMT) {
        const double sa2 = sa_s[(it & 1) * kPgMT + te] * p.inv_amp;
        sa_s[(it & 1) * kPgMT + te] = sa2;
        const int sh = __double2hiint(sa2);
        c52_s[(it & 1) * kPgMT + te] =
            (sh & 0x7FF00000) != 0 && (sh & 0x7FF00000) < 0x7C000000
                ? __hiloint2double((sh + (52 << 20)) ^ static_cast<int>(0x80000000u), __double2loint(sa2))
                : -sa2 * 4503599627370496.0;
      }
      named_bar_sync(1, 128 * kPgEW);  // sa_s[it & 1] landed (and scaled) for every thread
      const double* sa_t = sa_s + (it & 1) * kPgMT + g * kCols;
      const double* c52_t = c52_s + (it & 1) * kPgMT + g * kCols;
      const int64_t n = static_cast<int64_t>(nt) * kTileN + r;
      const int64_t m0 = static_cast<int64_t>(mt) * kPgMT + g * kCols;
      if (n < p.N) {
#pragma unroll
        for (int t = 0; t < kCols; ++t) {
          const int64_t m = m0 + t;
          if (m < p.M) {
            const int64_t idx = m * p.N + n;
            if (PATH == ISB_PATH_INTEGER_SCALE) {
              if (p.out_dtype == ISB_I32) {
                static_cast<int32_t*>(p.out)[idx] = iacc[t];
              } else {
                // Eq. 2 in one FP64 op (the FP64 pipe is the epilogue's scarce resource
                // while the tensor core streams): D = 2^52 + |acc| by bit construction,
                // fma(D, sa2, -2^52 sa2) = RN64(|acc| * sa2) exactly, sign after F2F
                const uint32_t a = static_cast<uint32_t>(iacc[t]);
                const uint32_t mag = (a >> 31) ? 0u - a : a;
                const double o =
                    __fma_rn(__hiloint2double(0x43300000, static_cast<int>(mag)), sa_t[t], c52_t[t]);
                pg_store(p.out, p.out_dtype, idx,
                         __uint_as_float(__float_as_uint(__double2float_rn(o)) ^ (a & 0x80000000u)));
              }
            } else {
              const double o = __dmul_rn(static_cast<double>(facc[t]), sa_t[t]);
              pg_store(p.out, p.out_dtype, idx, __double2float_rn(o));
            }
          }
        }
      }
      named_bar_sync(1, 128 * kPgEW);  // done with sa_s[it & 1] before it is refilled
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

template <int PATH>
void launch_pg(const CUtensorMap& map, const PgParams& prm, int grid, cudaStream_t s) {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemm_w4a8_pg<PATH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kPgSmem),
               "cudaFuncSetAttribute(pg smem)");
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPgThreads);
  cfg.dynamicSmemBytes = kPgSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_pg<PATH>, map, prm), "gemm_w4a8_pg launch");
  count_launch();
}

}  // namespace

bool pg_eligible(int64_t m, const isb_weight& w) {
  return w.tensor_core_ok() && w.group == kBlockK && m >= kPgMinM;
}

void launch_gemm_pg(int path, const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                    void* out, int out_dtype, int num_sms, cudaStream_t s, int64_t kb0, int64_t kbn) {
  if (kbn < 0) kbn = w.kblocks - kb0;
  PgParams prm{};
  prm.packed = w.packed;
  prm.scale = path == ISB_PATH_INTEGER_SCALE ? w.kscale_tiled
                                             : reinterpret_cast<const int32_t*>(w.fscale_tiled);
  prm.sa = sa;
  prm.out = out;
  prm.M = static_cast<int>(m);
  prm.N = static_cast<int>(w.n);
  prm.G = static_cast<int>(w.groups);
  prm.kblocks = static_cast<int>(kbn);
  prm.kb0 = static_cast<int>(kb0);
  prm.kbw = static_cast<int>(w.kblocks);
  prm.m_tiles = static_cast<int>((m + kPgMT - 1) / kPgMT);
  prm.tiles = static_cast<int>(w.n_tiles) * prm.m_tiles;
  prm.out_dtype = out_dtype;
  prm.late_shift = (path == ISB_PATH_INTEGER_SCALE && w.static_bound > 0 &&
                    w.static_bound <= (int64_t{1} << 27) - 1 && kbn == w.kblocks) ? 1 : 0;
  prm.inv_amp = std::ldexp(1.0, -w.exponent);
  const CUtensorMap map = make_x_map(xq, m, w.k, kPgMT);
  const int grid = std::min(prm.tiles, num_sms);
  if (path == ISB_PATH_INTEGER_SCALE)
    launch_pg<ISB_PATH_INTEGER_SCALE>(map, prm, grid, s);
  else
    launch_pg<ISB_PATH_FLOAT_SCALE>(map, prm, grid, s);
}

}  // namespace isb
