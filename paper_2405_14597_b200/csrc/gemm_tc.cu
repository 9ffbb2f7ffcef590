// K3 (integer scale) and K4 (float scale) — fused W4A8 group GEMM on tcgen05.
//
// Reference: gemm_integer_scale (gemm.cpp:205-262) and gemm_float_scale
// (gemm.cpp:156-203); paper Eq. 2 / Eq. 1 (PAPER.md:149 / :80).
//
// "Swap-AB" shape: output channels are the UMMA M dimension (128 per tile), tokens
// are UMMA N (MT = 16..128), so decode-sized M still issues full-width MMAs.
//
// Work split: thread-block clusters of C CTAs own whole output tiles (persistent,
// tile += #clusters); CTA rank q of a cluster takes quantization groups
// [q*G/C, (q+1)*G/C) of every tile it visits (split-K on group boundaries). The
// C int32 partials of a tile are reduced through distributed shared memory
// (no global atomics, no fences in HBM) and each rank finalises MT/C tokens.
//
// Per CTA, warp-specialised, synchronising once per "step" of S consecutive
// 128-K blocks (S = 4 at decode) so the fixed cost of each mbarrier hop is
// amortised over 32 KiB of weights:
//   warp 0      producer : one cp.async.bulk of the step's S x 8 KiB packed-int4
//                          blocks (contiguous in HBM) + S TMA (SWIZZLE_128B) loads
//                          of the MT x 128 int8 activation tiles. The first steps'
//                          weights are fetched before griddepcontrol.wait (PDL).
//   warps 4..   transform: smem int4 -> int8 (x16) expansion into the TMEM A ring
//                          (thread r owns output channel r); 2 warpgroups alternate
//                          steps at decode.
//   warp 1      MMA      : 4 x tcgen05.mma.kind::i8 (K=32) per 128-K block, one TMEM
//                          accumulator block per 128-K block.
//   warps ..    epilogue : tcgen05.ld of each block's int32 16*P (summed over the
//                          blocks of a group when g > 128), then
//                          integer path  acc += (P16 >> 4) * k_g   (int32, IMAD)
//                          float path    acc += float(P16) * (s_g/16) (I2F + FFMA)
//                          and one conversion per output (Eq. 2).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"
#include "quant.cuh"
#include "tc_decode.cuh"

namespace isb {

int64_t* g_trace = nullptr;
int g_trace_cta = 0;
int g_dbg = 0;

namespace {


struct Params {
  const uint8_t* packed;
  const int32_t* kscale;  // [n_tiles][G][128]
  const float* fscale;    // [n_tiles][G][128], s/16
  const double* sa;       // [M]
  void* out;              // [M][N]
  int M, N, G, gb, kblocks, m_tiles, tiles, out_dtype;
  int C, NC;              // cluster size, number of clusters
  double inv_amp;         // 2^-e (exact)
  int late_shift;         // 16 * static bound fits int32: accumulate 16*P*k, shift once
  int64_t* trace;         // optional debug timeline (see ISB_TRACE)
  int trace_cta;
  int dbg;                // debug knobs: 1 skip A st, 2 skip D ld, 4 skip MMA issue
  const void* xf;         // XQ: float32 / bf16 activations [M][K]
  int x_dtype;
  int K;
  double* sa_out;         // XQ: optional per-token scales out [M] (written by rank 0)
  const double* wscale_d; // coarse path: per-channel weight scales s_w[N] (double)
};

// Debug timeline: trace[role * 512 + i] = globaltimer at event i of that role.
#define ISB_TRACE(role, i)                                                              \
  do {                                                                                  \
    if (p.trace != nullptr && static_cast<int>(blockIdx.x) == p.trace_cta && (i) < 512) \
      p.trace[(role) * 512 + (i)] = globaltimer_();                                     \
  } while (0)
#define ISB_TRACE_CTA(role)                                                        \
  do {                                                                             \
    if (p.trace != nullptr) p.trace[(role) * 512 + blockIdx.x] = globaltimer_(); \
  } while (0)

// The CTA's view of the work: tiles cid, cid+NC, ...; groups [g0, g1) of each.
struct Work {
  int cid, rank, g0, g1, kb0, kb1, nsteps_tile, ntiles;
  __device__ Work(const Params& p, int S) {
    cid = blockIdx.x / p.C;
    rank = blockIdx.x % p.C;
    g0 = rank * p.G / p.C;
    g1 = (rank + 1) * p.G / p.C;
    kb0 = g0 * p.gb;
    kb1 = g1 * p.gb;
    nsteps_tile = (kb1 - kb0 + S - 1) / S;
    ntiles = cid < p.tiles ? (p.tiles - cid + p.NC - 1) / p.NC : 0;
  }
  __device__ int tile(int it, const Params& p) const { return cid + it * p.NC; }
};

template <int MT, int PATH, bool GB1, bool XQ>
__global__ void __launch_bounds__(Cfg<MT, XQ>::kThreads, 1)
    gemm_w4a8_tc(const __grid_constant__ CUtensorMap x_map, const Params p) {
  using Cf = Cfg<MT, XQ>;
  constexpr int S = Cf::S;
  constexpr int kStages = Cf::kStages;
  constexpr int kXSlot = Cf::kXSlot;
  constexpr int kCols = Cf::kCols;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_xres = smem;                                     // XQ: [kb][MT rows][128 B]
  uint8_t* smem_w = smem + Cf::kXRes;                            // [stage][S][8 KiB]
  uint8_t* smem_x = smem_w + kStages * S * kBlockBytes;          // [stage][S][kXSlot]
  uint8_t* smem_sc = smem_x + kStages * S * kXSlot;              // [stage][S][128] scales
  uint8_t* pbuf = smem_sc + kStages * Cf::kScBytes;              // [kPbufs][MT][128] partials
  double* sa_s = reinterpret_cast<double*>(pbuf + Cf::kPbufBytes);  // [2][MT]
  float* amx_peer = reinterpret_cast<float*>(pbuf + Cf::kPbufBytes + Cf::kSaBytes);  // XQ [8][MT]
  float* amx_loc = amx_peer + 8 * MT;                                 // XQ [MT]
  double* sa_f = reinterpret_cast<double*>(amx_loc + MT);             // XQ [MT] fused s_a
  uint64_t* bars = reinterpret_cast<uint64_t*>(pbuf + Cf::kPbufBytes + Cf::kSaBytes +
                                               Cf::kAmaxBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* a_full = empty + kStages;
  uint64_t* a_empty = a_full + Cf::kNA;
  uint64_t* d_full = a_empty + Cf::kNA;
  uint64_t* d_empty = d_full + Cf::kND;
  uint64_t* sc_empty = d_empty + Cf::kND;
  uint64_t* pb_full = sc_empty + kStages;   // [2] epilogue -> reduction warps (local)
  uint64_t* red_full = pb_full + 2;         // [2] all ranks' partials published (cluster)
  uint64_t* red_empty = red_full + 2;       // [2] all ranks done reading ours (cluster)
  uint64_t* x_ready = red_empty + 2;        // XQ: resident codes + s_a written (local)
  uint64_t* amax_bar = x_ready + 1;         // XQ: all ranks' partial row maxima in (cluster)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(amax_bar + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const Work wk(p, S);
  const int nsteps = wk.nsteps_tile * wk.ntiles;

  if (warp == 0 && lane == 0) {
    if (!XQ) prefetch_tensormap(&x_map);
    mbar_init(x_ready, 1);
    mbar_init(amax_bar, p.C);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1 + 4);
      mbar_init(&sc_empty[i], 4 * Cf::kEpiWG);
    }
    for (int i = 0; i < Cf::kNA; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < Cf::kND; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4 * Cf::kEpiWG);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pb_full[i], 4 * Cf::kEpiWG);
      mbar_init(&red_full[i], 2 * p.C);
      mbar_init(&red_empty[i], 2 * p.C);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cf::kTmemCols);
  tc_fence_before();
  if (p.C > 1) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) pdl_launch_dependents();
  if (threadIdx.x == 0) ISB_TRACE_CTA(14);

  // kblock range of step j (global step index over this CTA's tiles)
  auto step_range = [&](int j, int& tile, int& kb, int& nkb) {
    const int it = j / wk.nsteps_tile;
    const int sj = j - it * wk.nsteps_tile;
    tile = wk.tile(it, p);
    kb = wk.kb0 + sj * S;
    nkb = min(S, wk.kb1 - kb);
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      // Weights do not depend on the preceding kernel: stream the first kStages
      // steps before griddepcontrol.wait so their HBM latency hides behind the
      // previous grid (PDL). Activations are loaded after the wait.
      const int32_t* scale_src = PATH == ISB_PATH_INTEGER_SCALE
                                     ? p.kscale : reinterpret_cast<const int32_t*>(p.fscale);
      // weights + group scales of step j into stage j % kStages (both static data)
      auto load_static = [&](int j, int stage) {
        int tile, kb, nkb;
        step_range(j, tile, kb, nkb);
        const int nt = tile / p.m_tiles;
        const int ga = kb / p.gb, gz = (kb + nkb - 1) / p.gb;
        mbar_arrive_expect_tx(&full[stage], nkb * (kBlockBytes + (XQ ? 0 : Cf::kXBytes)) +
                                                (gz - ga + 1) * kTileN * 4);
        bulk_load_evict_first(smem_w + stage * S * kBlockBytes,
                              p.packed + (static_cast<int64_t>(nt) * p.kblocks + kb) * kBlockBytes,
                              nkb * kBlockBytes, &full[stage]);
        bulk_load(smem_sc + stage * Cf::kScBytes,
                  scale_src + (static_cast<int64_t>(nt) * p.G + ga) * kTileN,
                  (gz - ga + 1) * kTileN * 4, &full[stage]);
      };
      const int pre = min(nsteps, kStages);
      for (int j = 0; j < pre; ++j) load_static(j, j);
      pdl_wait();
      for (int j = 0; j < nsteps; ++j) {
        const int stage = j % kStages;
        int tile, kb, nkb;
        step_range(j, tile, kb, nkb);
        const int mt = tile % p.m_tiles;
        if (j >= pre) {
          mbar_wait(&empty[stage], ((j / kStages) & 1) ^ 1);
          mbar_wait(&sc_empty[stage], ((j / kStages) & 1) ^ 1);
          load_static(j, stage);
        }
        if (!XQ)
          for (int i = 0; i < nkb; ++i)
            tma_load_2d(smem_x + (stage * S + i) * kXSlot, &x_map, &full[stage],
                        (kb + i) * kBlockK, mt * MT);
        (void)mt;
        ISB_TRACE(0, j);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp)
    constexpr uint32_t idesc = make_idesc_i8(128, MT);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t x_base = smem_u32(smem_x);
    const uint32_t xres_base = smem_u32(smem_xres);
    if (XQ && nsteps > 0) mbar_wait(x_ready, 0);  // resident quantized activations written
    for (int j = 0; j < nsteps; ++j) {
      const int stage = j % kStages, as = j % Cf::kNA, ds = j % Cf::kND;
      int tile, kb, nkb;
      step_range(j, tile, kb, nkb);
      // a_full implies full: the transform warps observed full[stage] before arriving.
      mbar_wait(&a_full[as], (j / Cf::kNA) & 1);
      mbar_wait(&d_empty[ds], ((j / Cf::kND) & 1) ^ 1);
      tc_fence_after();
      ISB_TRACE(2, j);
#pragma unroll
      for (int i = 0; i < S; ++i) {
        if (i < nkb) {
          const uint64_t bdesc = make_sw128_kmajor_desc(
              XQ ? xres_base + (kb + i - wk.kb0) * Cf::kXTile : x_base + (stage * S + i) * kXSlot);
          const uint32_t d_tmem = tbase + Cf::kNA * Cf::kACols + ds * Cf::kDCols + i * MT;
          const uint32_t a_tmem = tbase + as * Cf::kACols + i * 32;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (!(p.dbg & 4))
              mma_i8_ts_warp(d_tmem, a_tmem + c * 8, bdesc + static_cast<uint64_t>(c * 2), idesc,
                             c > 0 ? 1u : 0u);
        }
      }
      mma_commit_warp(&empty[stage]);
      mma_commit_warp(&a_empty[as]);
      mma_commit_warp(&d_full[ds]);
    }
  } else if (warp >= 4 && warp < 4 + 4 * Cf::kXformWG) {
    // ---------------------------------------------------------------- transform
    const int xw = static_cast<int>(warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;  // output channel within the tile == TMEM lane
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t w_base = smem_u32(smem_w) + r * 16;
    for (int j = xw; j < nsteps; j += Cf::kXformWG) {
      const int stage = j % kStages, as = j % Cf::kNA;
      int tile, kb, nkb;
      step_range(j, tile, kb, nkb);
      mbar_wait(&full[stage], (j / kStages) & 1);
      ISB_TRACE(1, j);
      uint4 q[S][4];
#pragma unroll
      for (int i = 0; i < S; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (i < nkb)
            q[i][c] = ld_shared_v4(w_base + (stage * S + i) * kBlockBytes + c * (kTileN * 16));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the async refill
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      mbar_wait(&a_empty[as], ((j / Cf::kNA) & 1) ^ 1);
      tc_fence_after();
#pragma unroll
      for (int i = 0; i < S; ++i) {
        if (i < nkb) {
          uint32_t a[32];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t w4[4] = {q[i][c].x, q[i][c].y, q[i][c].z, q[i][c].w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              a[c * 8 + 2 * w] = (w4[w] << 4) & 0xF0F0F0F0u;  // 16*code(k0..k0+3)
              a[c * 8 + 2 * w + 1] = w4[w] & 0xF0F0F0F0u;     // 16*code(k0+4..k0+7)
            }
          }
          if (!(p.dbg & 1)) tmem_st_x32(tmem_base + lane_base + as * Cf::kACols + i * 32, a);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[as]);
      ISB_TRACE(3, j);
    }
  } else if (warp >= 4 + 4 * Cf::kXformWG) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t ew = warp - (4 + 4 * Cf::kXformWG);  // 0 .. 4*kEpiWG-1
    const uint32_t wg = ew / 4;                          // which token half
    const uint32_t r = (ew % 4) * 32 + lane;             // TMEM lane == output channel in tile
    const uint32_t lane_base = ((ew % 4) * 32) << 16;
    const int c0 = wg * kCols;
    pdl_wait();  // sa and the output may be touched by the preceding grid
    const uint32_t pbuf_local = smem_u32(pbuf);
    const bool late = p.late_shift != 0;
    int j = 0;   // global step index
    for (int it = 0; it < wk.ntiles; ++it) {
      const int tile = wk.tile(it, p);
      const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
      if constexpr (Cf::kPbufs == 0) {
        if (ew == 0) {  // token scales of this tile -> sa_s[it & 1] (read at finalise)
          for (int t = lane; t < MT; t += 32) {
            const int64_t m = static_cast<int64_t>(mt) * MT + t;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                             smem_u32(sa_s + (it & 1) * MT + t)),
                         "l"(p.sa + (m < p.M ? m : 0)), "r"(m < p.M ? 8 : 0)
                         : "memory");
          }
          cp_async_commit();
        }
      }
      int32_t iacc[kCols];
      float facc[kCols];
      int32_t gsum[GB1 ? 1 : kCols];
#pragma unroll
      for (int t = 0; t < kCols; ++t) { iacc[t] = 0; facc[t] = 0.0f; }
      for (int sj = 0; sj < wk.nsteps_tile; ++sj, ++j) {
        const int ds = j % Cf::kND, stage = j % kStages;
        const int kb = wk.kb0 + sj * S;
        const int nkb = min(S, wk.kb1 - kb);
        mbar_wait(&d_full[ds], (j / Cf::kND) & 1);
        mbar_wait(&full[stage], (j / kStages) & 1);  // scales of this step landed (cheap: done)
        tc_fence_after();
        ISB_TRACE(4, j);
        const uint32_t sc_base = smem_u32(smem_sc + stage * Cf::kScBytes) + r * 4;
        const int ga = kb / p.gb;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          if (i < nkb) {
            const bool g_first = GB1 || ((kb + i) % p.gb == 0);
            const bool g_last = GB1 || ((kb + i) % p.gb == p.gb - 1);
            int32_t kg = 0;
            float sg = 0.0f;
            if (g_last) {
              const uint32_t sraw = ld_shared_u32(sc_base + ((kb + i) / p.gb - ga) * (kTileN * 4));
              kg = PATH == ISB_PATH_COARSE ? 1 : static_cast<int32_t>(sraw);
              sg = __uint_as_float(sraw);
            }
            const uint32_t taddr =
                tmem_base + lane_base + Cf::kNA * Cf::kACols + ds * Cf::kDCols + i * MT + c0;
            constexpr int kChunk = kCols < 16 ? kCols : 16;
#pragma unroll
            for (int cc = 0; cc < kCols; cc += kChunk) {
              uint32_t v[16];
              if (!(p.dbg & 2)) {
                if constexpr (kChunk == 16) {
                  tmem_ld_x16_(taddr + cc, v);
                } else {
                  tmem_ld_x8(taddr + cc, *reinterpret_cast<uint32_t(*)[8]>(&v[0]));
                }
              } else {
#pragma unroll
                for (int z = 0; z < 16; ++z) v[z] = z;
              }
              tmem_wait_ld();
#pragma unroll
              for (int t = 0; t < kChunk; ++t) {
                int32_t d = static_cast<int32_t>(v[t]);  // 16 * P over this 128-K block, exact
                if constexpr (!GB1) {
                  d = g_first ? d : gsum[cc + t] + d;
                  gsum[cc + t] = d;
                }
                if (g_last) {
                  if (PATH != ISB_PATH_FLOAT_SCALE) {
                    // Eq. 2: int32 scaled accumulation. With 16x headroom under the
                    // static bound the x16 of the nibble expansion is removed once at
                    // the end (one IMAD per value instead of SHF + IMAD).
                    if (late) iacc[cc + t] += d * kg;
                    else iacc[cc + t] += (d >> 4) * kg;
                  } else {
                    facc[cc + t] = fmaf(static_cast<float>(d), sg, facc[cc + t]);  // Eq. 1, fp32
                  }
                }
              }
            }
          }
        }
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // scale reads before refill
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&d_empty[ds]);
          mbar_arrive(&sc_empty[stage]);
        }
      }
      if (PATH != ISB_PATH_FLOAT_SCALE && late) {
#pragma unroll
        for (int t = 0; t < kCols; ++t) iacc[t] >>= 4;  // exact: 16 | acc16
      }
      // ------------------------------------------------ tile completion
      if (ew == 0 && lane == 0) ISB_TRACE(8, it);
      if constexpr (Cf::kPbufs > 0) {
        // Hand the partial to the reduction warps and move on to the next tile.
        const int buf = it % Cf::kPbufs;
        mbar_wait_cluster(&red_empty[buf], ((it / Cf::kPbufs) & 1) ^ 1);
        const uint32_t pb = pbuf_local + buf * (MT * kTileN * 4);
#pragma unroll
        for (int t = 0; t < kCols; ++t)
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(pb + ((c0 + t) * kTileN + r) * 4),
                       "r"(PATH != ISB_PATH_FLOAT_SCALE ? static_cast<uint32_t>(iacc[t])
                                                          : __float_as_uint(facc[t]))
                       : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&pb_full[buf]);
      } else {
        // Direct finalise from registers (MT = 128): token scales were prefetched
        // into sa_s at the start of the tile.
        if (ew == 0) cp_async_wait<0>();
        named_bar_sync(1, 128 * Cf::kEpiWG);
        const double* sa_t = sa_s + (it & 1) * MT;
        const int64_t n = static_cast<int64_t>(nt) * kTileN + r;
        if (n < p.N) {
          const double s_w = PATH == ISB_PATH_COARSE ? p.wscale_d[n] : 0.0;
#pragma unroll
          for (int t = 0; t < kCols; ++t) {
            const int64_t m = static_cast<int64_t>(mt) * MT + c0 + t;
            if (m < p.M) {
              if (PATH == ISB_PATH_INTEGER_SCALE && p.out_dtype == ISB_I32)
                static_cast<int32_t*>(p.out)[m * p.N + n] = iacc[t];
              else
                store_out(p.out, p.out_dtype, m * p.N + n,
                          finish<PATH>(iacc[t], facc[t], sa_t[c0 + t], p.inv_amp, s_w));
            }
          }
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------------------------------------------------------- reduction warps
    // Cluster split-K: every rank reduces tokens [rank*MT/C, (rank+1)*MT/C) of the
    // tile over all ranks' published partials (DSMEM reads in fixed rank order =>
    // deterministic), applies Eq. 2 / Eq. 1 and writes them. C = 1 reads locally.
    if constexpr (Cf::kPbufs > 0) {
      pdl_wait();  // sa and the output
      const uint32_t u = (warp - 2) * 32 + lane;  // rows u and u + 64
      const uint32_t pbuf_local = smem_u32(pbuf);
      // Token scales of tile `it` land in sa_s[it & 1] via cp.async issued one tile
      // ahead, so the finalise never waits on an L2/HBM round trip.
      auto sa_prefetch = [&](int it) {
        if (it < wk.ntiles && u < static_cast<uint32_t>(MT)) {
          const int64_t m = static_cast<int64_t>(wk.tile(it, p) % p.m_tiles) * MT + u;
          const uint32_t dst = smem_u32(sa_s + (it & 1) * MT + u);
          const double* src = p.sa + (m < p.M ? m : 0);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                       "r"(m < p.M ? 8 : 0)
                       : "memory");
        }
        cp_async_commit();
      };
      if (!XQ) sa_prefetch(0);
      if (XQ && wk.ntiles > 0) mbar_wait(x_ready, 0);  // fused s_a in sa_f
      for (int it = 0; it < wk.ntiles; ++it) {
        const int buf = it % Cf::kPbufs;
        const uint32_t ph = (it / Cf::kPbufs) & 1;
        const int tile = wk.tile(it, p);
        const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
        if (!XQ) {
          sa_prefetch(it + 1);
          cp_async_wait<1>();
          named_bar_sync(2, 64);  // sa_s[it & 1] visible to both reduction warps
        }
        const double* sa_t = XQ ? sa_f : sa_s + (it & 1) * MT;
        mbar_wait(&pb_full[buf], ph);
        if (p.C > 1) {
          if (lane < static_cast<uint32_t>(p.C))
            mbar_arrive_remote_release(mapa_shared(smem_u32(&red_full[buf]), lane));
          mbar_wait_cluster(&red_full[buf], ph);
        }
        if (warp == 2 && lane == 0) ISB_TRACE(6, it);
        const uint32_t pb = pbuf_local + buf * (MT * kTileN * 4);
        switch (p.C) {
          case 1: reduce_tile<MT, 1, PATH>(p, pb, sa_t, wk.rank, nt, mt, u); break;
          case 2: reduce_tile<MT, 2, PATH>(p, pb, sa_t, wk.rank, nt, mt, u); break;
          case 3: reduce_tile<MT, 3, PATH>(p, pb, sa_t, wk.rank, nt, mt, u); break;
          case 4: reduce_tile<MT, 4, PATH>(p, pb, sa_t, wk.rank, nt, mt, u); break;
          default: reduce_tile<MT, 8, PATH>(p, pb, sa_t, wk.rank, nt, mt, u); break;
        }
        if (!XQ) named_bar_sync(2, 64);  // done with sa_s[it & 1] before it is refilled
        if (warp == 2 && lane == 0) ISB_TRACE(7, it);
        if (p.C > 1) {
          if (lane < static_cast<uint32_t>(p.C))
            mbar_arrive_remote(mapa_shared(smem_u32(&red_empty[buf]), lane));
        } else if (lane == 0) {
          mbar_arrive(&red_empty[buf]);
        }
      }
      // Do not retire while peers may still read our partials.
      for (int it = max(0, wk.ntiles - Cf::kPbufs); it < wk.ntiles; ++it)
        mbar_wait_cluster(&red_empty[it % Cf::kPbufs], (it / Cf::kPbufs) & 1);
    }
  }

  // Peers never touch this CTA's smem after its red_empty completes (waited above),
  // so a CTA-local barrier suffices before releasing TMEM.
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ISB_TRACE_CTA(15);
  if (warp == 2) tmem_dealloc(tmem_base, Cf::kTmemCols);
}

template <int MT, int PATH, bool GB1, bool XQ>
void prepare_kernel() {
  static std::once_flag once;
  std::call_once(once, [] {
    auto kern = gemm_w4a8_tc<MT, PATH, GB1, XQ>;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Cfg<MT, XQ>::kSmemBytes),
               "cudaFuncSetAttribute(smem)");
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
               "cudaFuncSetAttribute(cluster)");
  });
}

// Max co-resident clusters of size C for this kernel (driver occupancy query).
template <int MT, int PATH, bool GB1, bool XQ>
int max_active_clusters(int C) {
  prepare_kernel<MT, PATH, GB1, XQ>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C * 64);
  cfg.blockDim = dim3(Cfg<MT, XQ>::kThreads);
  cfg.dynamicSmemBytes = Cfg<MT, XQ>::kSmemBytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_w4a8_tc<MT, PATH, GB1, XQ>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

template <int MT, int PATH, bool GB1, bool XQ>
void launch_mt(const CUtensorMap& map, const Params& prm, int grid, cudaStream_t s) {
  using Cf = Cfg<MT, XQ>;
  prepare_kernel<MT, PATH, GB1, XQ>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cf::kThreads);
  cfg.dynamicSmemBytes = Cf::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = prm.C;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_tc<MT, PATH, GB1, XQ>, map, prm),
             "gemm_w4a8_tc launch");
  count_launch();
}

int pick_mt(int64_t m) {
  static const bool mt64 = [] {  // ISB_MT64=1: the single 64-token tile for 32 < M <= 64 (A/B)
    const char* e = std::getenv("ISB_MT64");
    return e && e[0] == '1';
  }();
  if (m <= 16) return 16;
  if (m <= 32) return 32;
  if (m <= 64) return mt64 ? 64 : 32;  // two 32-token tiles: MT=64 spills its accumulators
  return 128;
}

int cluster_capacity(int mt, int C, bool xq) {
  // Co-resident clusters per device; cached per (mt, C, fused).
  static std::mutex mu;
  static int cache[2][4][9] = {};
  const int mi = mt == 16 ? 0 : mt == 32 ? 1 : mt == 64 ? 2 : 3;
  std::lock_guard<std::mutex> lk(mu);
  int& slot = cache[xq ? 1 : 0][mi][C];
  if (!slot) {
    int n = 0;
    if (xq) {
      switch (mt) {
        case 16: n = max_active_clusters<16, ISB_PATH_INTEGER_SCALE, true, true>(C); break;
        case 32: n = max_active_clusters<32, ISB_PATH_INTEGER_SCALE, true, true>(C); break;
        default: n = max_active_clusters<64, ISB_PATH_INTEGER_SCALE, true, true>(C); break;
      }
    } else {
      switch (mt) {
        case 16: n = max_active_clusters<16, ISB_PATH_INTEGER_SCALE, true, false>(C); break;
        case 32: n = max_active_clusters<32, ISB_PATH_INTEGER_SCALE, true, false>(C); break;
        case 64: n = max_active_clusters<64, ISB_PATH_INTEGER_SCALE, true, false>(C); break;
        default: n = max_active_clusters<128, ISB_PATH_INTEGER_SCALE, true, false>(C); break;
      }
    }
    slot = n > 0 ? n : -1;
  }
  return slot;
}

int xres_blocks(int mt) {
  return mt == 16 ? Cfg<16, true>::kXResBlocks
                  : mt == 32 ? Cfg<32, true>::kXResBlocks : Cfg<64, true>::kXResBlocks;
}

}  // namespace

// ---------------------------------------------------------------------------- host side (shared)
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


GemmPlan plan_gemm(int64_t m, const isb_weight& w, int num_sms, int path, bool fused) {
  (void)path;
  GemmPlan pl;
  pl.mt = pick_mt(m);
  pl.m_tiles = static_cast<int>((m + pl.mt - 1) / pl.mt);
  pl.tiles = static_cast<int>(w.n_tiles) * pl.m_tiles;
  pl.units = static_cast<int64_t>(pl.tiles) * w.groups;
  pl.fused = fused;
  // Choose the cluster size C (split-K ways): makespan ~ rounds * (steps per CTA
  // + per-tile overhead), rounds = ceil(tiles / co-resident clusters). Fused
  // activation quantization also needs every rank's K slice to fit the resident
  // budget.
  const int S = pl.mt <= 32 ? 4 : (pl.mt == 64 ? 2 : 1);
  const int64_t gb = w.group / kBlockK;
  double best = 1e30;
  pl.cluster = 0;
  pl.grid = 1;
  static const int force_c = [] {  // ISB_FORCE_C=<1|2|4|8>: A/B of the split-K width
    const char* e = std::getenv("ISB_FORCE_C");
    return e ? std::atoi(e) : 0;
  }();
  for (int C : {1, 2, 3, 4, 8}) {
    if (C > w.groups) break;
    if (C == 3 && (fused || force_c != 3)) continue;  // C = 3 (uneven token split): opt-in
    if (C > 1 && pl.mt >= 128) break;  // two epilogue warpgroups: no cluster split-K
    if (force_c && C != force_c) continue;
    const int64_t groups_cta = (w.groups + C - 1) / C;
    if (fused && groups_cta * gb > xres_blocks(pl.mt)) continue;
    int cap = cluster_capacity(pl.mt, C, fused);
    if (cap <= 0) continue;
    cap = std::min(cap, num_sms / C);
    const int nc = std::min(cap, pl.tiles);
    const int rounds = (pl.tiles + nc - 1) / nc;
    const int64_t kb_cta = groups_cta * gb;
    const double steps = std::ceil(static_cast<double>(kb_cta) / S);
    // Per-tile cost beyond streaming: ~half a step (the next tile's loads are already
    // in flight), plus the cluster reduction. Fitted on the LLaMA-2-7B decode shapes
    // (profiles/r01_decode_planner.txt): a grid that leaves SMs idle (few tiles, C=1)
    // loses to more rounds of a wider split.
    double cost = rounds * (steps + 0.5 + (C > 1 ? 0.25 : 0.0));
    // fused: every CTA first reads its float activation slice (4 B / element),
    // counted in units of one step's 32 KiB of weights.
    if (fused) cost += static_cast<double>(pl.mt) * kb_cta * kBlockK * 4.0 / (4.0 * kBlockBytes);
    if (cost < best - 1e-9) {
      best = cost;
      pl.cluster = C;
      pl.grid = nc * C;
    }
  }
  if (pl.cluster == 0) {  // fused: no cluster size fits the resident slice
    if (fused) fail(ISB_PARAM, "fused activation quantization: K slice too large");
    pl.cluster = 1;
  }
  pl.maxc = pl.cluster;
  pl.workspace_bytes = 0;  // split-K reduces through DSMEM: no global workspace
  return pl;
}

bool act_fused_eligible(int64_t m, int64_t k, const isb_weight& w) {
  if (m < 1 || m > 64 || !w.tensor_core_ok() || k != w.k) return false;
  const int mt = pick_mt(m);
  if (mt < m) return false;  // the resident slice holds one token tile
  const int64_t gb = w.group / kBlockK;
  for (int C : {1, 2, 4, 8})
    if (C <= w.groups && ((w.groups + C - 1) / C) * gb <= xres_blocks(mt)) return true;
  return false;
}

void launch_gemm_tc(int path, const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                    void* out, int out_dtype, void* workspace, const GemmPlan& pl,
                    cudaStream_t s, const void* xf, int x_dtype, double* sa_out) {
  (void)workspace;
  Params prm{};
  prm.packed = w.packed;
  prm.kscale = w.kscale_tiled;
  prm.fscale = w.fscale_tiled;
  prm.sa = sa;
  prm.out = out;
  prm.M = static_cast<int>(m);
  prm.N = static_cast<int>(w.n);
  prm.G = static_cast<int>(w.groups);
  prm.gb = static_cast<int>(w.group / kBlockK);
  prm.kblocks = static_cast<int>(w.kblocks);
  prm.m_tiles = pl.m_tiles;
  prm.tiles = pl.tiles;
  prm.out_dtype = out_dtype;
  prm.C = pl.cluster;
  prm.NC = pl.grid / pl.cluster;
  prm.inv_amp = std::ldexp(1.0, -w.exponent);
  prm.trace = g_trace;
  prm.trace_cta = g_trace_cta;
  prm.dbg = g_dbg;
  prm.late_shift = (path == ISB_PATH_INTEGER_SCALE && w.static_bound > 0 &&
                    w.static_bound <= (int64_t{1} << 27) - 1) ? 1 : 0;
  if (path == ISB_PATH_COARSE) {
    // exact int32 sum of 16 * x * w over the whole K: |.| <= 16 * K * 127 * 8
    if (16 * w.k * 127 * 8 > (int64_t{1} << 31) - 1) fail(ISB_PARAM, "coarse path: K too large");
    prm.late_shift = 1;
  }
  prm.wscale_d = w.scales;
  prm.xf = xf;
  prm.x_dtype = x_dtype;
  prm.K = static_cast<int>(w.k);
  prm.sa_out = sa_out;
  CUtensorMap map{};
  if (!pl.fused) map = make_x_map(xq, m, w.k, pl.mt);
  const bool gb1 = prm.gb == 1;
#define ISB_DISPATCH_P(MTV, PV, XQV)                                          \
  if (gb1) launch_mt<MTV, PV, true, XQV>(map, prm, pl.grid, s);               \
  else launch_mt<MTV, PV, false, XQV>(map, prm, pl.grid, s);
#define ISB_DISPATCH(MTV, XQV)                                                \
  case MTV:                                                                   \
    if (path == ISB_PATH_INTEGER_SCALE) { ISB_DISPATCH_P(MTV, ISB_PATH_INTEGER_SCALE, XQV) } \
    else { ISB_DISPATCH_P(MTV, ISB_PATH_FLOAT_SCALE, XQV) }                   \
    break;
#define ISB_DISPATCH_COARSE(MTV)                                              \
  case MTV:                                                                   \
    launch_mt<MTV, ISB_PATH_COARSE, false, false>(map, prm, pl.grid, s);     \
    break;
  if (path == ISB_PATH_COARSE) {  // per-channel weights: one group spanning K
    switch (pl.mt) {
      ISB_DISPATCH_COARSE(16)
      ISB_DISPATCH_COARSE(32)
      ISB_DISPATCH_COARSE(64)
      ISB_DISPATCH_COARSE(128)
      default: fail(ISB_ERROR, "bad tile");
    }
  } else if (pl.fused) {
    // The single-GEMM fused-quantization variant (XQ, removed) measured slower than K1 +
    // K3 (scripts/fused_timing.py, M = 16: 15.2 vs 8.3 us at 4096 x 4096): the fused form
    // is the grouped launch (gemm_group.cu); isb_gemm_act_fused runs K1 + K3.
    fail(ISB_ERROR, "no single-GEMM fused-quantization kernel");
  } else {
    switch (pl.mt) {
      ISB_DISPATCH(16, false)
      ISB_DISPATCH(32, false)
      ISB_DISPATCH(64, false)
      ISB_DISPATCH(128, false)
      default: fail(ISB_ERROR, "bad tile");
    }
  }
#undef ISB_DISPATCH
#undef ISB_DISPATCH_P
#undef ISB_DISPATCH_COARSE
}

}  // namespace isb
