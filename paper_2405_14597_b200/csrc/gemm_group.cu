// Grouped decode kernel ("layer launch"): several integer-scale (K3) or
// float-scale (K4) W4A8 GEMMs — the linears of one decoder layer, or the experts
// of a MoE layer — in ONE persistent launch, with the per-token activation
// quantizer (K1) folded in.
//
// Reference: gemm_integer_scale / gemm_float_scale (gemm.cpp:205-262 / :156-203)
// per problem, quantize(x, 8, symmetric, per_token) (quantize.cpp:93-145) for
// each problem's activation. Results are bit-identical to K1 followed by the
// single-GEMM kernel (gemm_tc.cu) for every problem.
//
// Why: at decode M every single-GEMM launch pays a fixed ~5 us (CTA setup,
// first-byte latency, split-K tail) that the weight stream cannot hide, and the
// K1 launches in front of each GEMM are pure latency. Here the SMs
// stream the weights of all problems back to back; the tiles of all problems
// are scheduled over the clusters longest-first (host LPT), so the tail is paid
// once per layer instead of once per GEMM.
//
// Per CTA the pipeline is the single-GEMM decode pipeline (gemm_tc.cu): producer
// warp (bulk copy of packed int4 weights + int32 k_g, TMA of int8 activation
// tiles), two transform warpgroups (int4 -> TMEM int8), MMA warp
// (tcgen05.mma.kind::i8, TMEM accumulators), epilogue warpgroup (per-group
// IMAD / FFMA), two reduction warps (cluster split-K over DSMEM + Eq. 2). What
// differs is the work list (a per-cluster schedule of (problem, tile) entries)
// and the activation hand-off:
//
//   quantize phase  the epilogue warpgroup of CTA b quantizes token rows b,
//                   b + grid, ... of the concatenated problems (exact K1
//                   arithmetic, quant.cuh) into the problem's int8 code buffer
//                   and double scales, then publishes the row with a
//                   gpu-scope release add on the problem's readiness counter;
//   consumers       the producer (before the first TMA of a problem's codes)
//                   and the reduction warps (before reading its token scales)
//                   acquire-poll the counter until all M rows are in. The weight
//                   stream never waits: the first kStages steps are in flight
//                   before griddepcontrol.wait, and weight loads of later steps
//                   are issued ahead of the activation loads.
//   reset           the last CTA to retire (acq_rel counter) zeroes the
//                   counters, so the plan can be replayed (CUDA graphs) with no
//                   memset node. All CTAs are co-resident (grid <= the
//                   occupancy-derived cluster capacity), so the polls cannot
//                   deadlock.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <numeric>
#include <queue>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"
#include "quant.cuh"
#include "tc_decode.cuh"

namespace isb {
namespace {

constexpr int kMaxGroup = ISB_GROUP_MAX_PROBLEMS;
constexpr int kSyncDone = kMaxGroup;      // CTAs retired
constexpr int kSyncBad = kMaxGroup + 1;   // non-finite activation seen (sticky)
constexpr int kSyncWords = kMaxGroup + 2;

struct GProb {
  const uint8_t* packed;
  const int32_t* kscale;   // [n_tiles][G][128]
  const float* fscale;     // [n_tiles][G][128] (s / 16)
  const double* sa;        // token scales [M] (written by the quantize phase when xf)
  void* out;               // [M][N]
  const void* xf;          // float32 / bf16 [M][K] quantized in-kernel, or nullptr
  int8_t* xq;              // int8 codes [M][K] (TMA source)
  double* sa_w;            // == sa when quantizing in-kernel
  const double* wscale_d;  // unused here (reduce_tile's coarse branch)
  double inv_amp;
  int M, N, G, K, kblocks, m_tiles, out_dtype, late_shift, x_dtype;
};

struct GParams {
  GProb prob[kMaxGroup];
  int qoff[kMaxGroup + 1];  // prefix sums of M over problems (quantize row tasks)
  int nprob, C, NC, quantize, qtasks, sched_stride;
  const int* sched;         // [NC][sched_stride]: (problem << 24) | tile
  const int* sched_len;     // [NC]
  unsigned* sync;           // [kSyncWords]
};

struct alignas(64) GMaps {
  CUtensorMap m[kMaxGroup];
};

ISB_DEVICE unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

ISB_DEVICE void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

ISB_DEVICE unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
               : "memory");
  return old;
}

ISB_DEVICE void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Spin (with back-off) until all `target` rows of a problem are published.
ISB_DEVICE void wait_rows(const unsigned* ctr, unsigned target) {
  while (ld_acquire_gpu(ctr) < target) __nanosleep(32);
}

// The CTA's walk over its cluster's schedule, one step (S 128-K blocks of one
// tile) at a time. Rank q of the cluster owns groups [q G / C, (q+1) G / C) of
// every tile (g = 128: one group per 128-K block).
template <int S>
struct GCur {
  const GParams* P;
  int cid, rank, it, ntiles, sj, nst, pi, nt, mt, kb0, kb1;
  __device__ void init(const GParams& prm, int cid_, int rank_) {
    P = &prm;
    cid = cid_;
    rank = rank_;
    it = 0;
    sj = 0;
    ntiles = cid < prm.NC ? prm.sched_len[cid] : 0;
    if (ntiles > 0) load();
  }
  __device__ void load() {
    const int e = P->sched[cid * P->sched_stride + it];
    pi = e >> 24;
    const int t = e & 0xFFFFFF;
    const GProb& q = P->prob[pi];
    nt = t / q.m_tiles;
    mt = t - nt * q.m_tiles;
    kb0 = rank * q.G / P->C;
    kb1 = (rank + 1) * q.G / P->C;
    nst = (kb1 - kb0 + S - 1) / S;
  }
  __device__ bool valid() const { return it < ntiles; }
  __device__ int kb() const { return kb0 + sj * S; }
  __device__ int nkb() const { return min(S, kb1 - kb()); }
  __device__ bool last_step() const { return sj == nst - 1; }
  __device__ void next() {
    if (++sj == nst) {
      sj = 0;
      if (++it < ntiles) load();
    }
  }
};

// K1 on one token row by a 128-thread warpgroup: exact quantize.cpp:93-145
// arithmetic (float absmax, s = double(amax) / 127, codes via quant_one), i.e.
// bit-identical to quantize_rows_* in quant.cu.
template <typename T>
__device__ __forceinline__ void quant_row(const T* __restrict__ xr, int K, int8_t* __restrict__ cr,
                                          double* s_out, float* red, uint32_t tid,
                                          unsigned* bad) {
  constexpr int U = 4;
  const int nv = K >> 2;  // float4 / 4-element groups (K % 128 == 0)
  float mx = 0.0f;
  bool fin = true;
  for (int v0 = static_cast<int>(tid); v0 < nv; v0 += 128 * U) {
    float v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 128 < nv) load4<T>(xr + 4 * (v0 + u * 128), v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 128 < nv)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          fin = fin && isfinite(v[u][e]);
          mx = fmaxf(mx, fabsf(v[u][e]));
        }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) red[tid / 32] = mx;
  if (!fin) atomicOr(bad, 1u);
  named_bar_sync(4, 128);
  mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  const double s = mx == 0.0f ? 1.0 : static_cast<double>(mx) / 127.0;  // quantize.cpp:120-125
  const double r = 1.0 / s;
  if (tid == 0) *s_out = s;
  for (int v0 = static_cast<int>(tid); v0 < nv; v0 += 128 * U) {
    float v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 128 < nv) load4<T>(xr + 4 * (v0 + u * 128), v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 128 < nv) {
        uint32_t packed = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          packed |= (static_cast<uint32_t>(quant_one(v[u][e], s, r, -128, 127)) & 0xFFu)
                    << (8 * e);
        *reinterpret_cast<uint32_t*>(cr + 4 * (v0 + u * 128)) = packed;
      }
  }
}

template <int MT, int PATH>
__global__ void __launch_bounds__(Cfg<MT, false>::kThreads, 1)
    gemm_w4a8_group(const __grid_constant__ GMaps maps, const __grid_constant__ GParams p) {
  using Cf = Cfg<MT, false>;
  static_assert(Cf::kXformWG == 2 && Cf::kEpiWG == 1 && Cf::kPbufs > 0, "decode tiles only");
  constexpr int S = Cf::S;
  constexpr int kStages = Cf::kStages;
  constexpr int kXSlot = Cf::kXSlot;
  constexpr int kCols = Cf::kCols;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_w = smem;                                        // [stage][S][8 KiB]
  uint8_t* smem_x = smem_w + kStages * S * kBlockBytes;          // [stage][S][kXSlot]
  uint8_t* smem_sc = smem_x + kStages * S * kXSlot;              // [stage][S][128] scales
  uint8_t* pbuf = smem_sc + kStages * Cf::kScBytes;              // [kPbufs][MT][128] partials
  double* sa_s = reinterpret_cast<double*>(pbuf + Cf::kPbufBytes);  // [2][MT]
  uint64_t* bars = reinterpret_cast<uint64_t*>(pbuf + Cf::kPbufBytes + Cf::kSaBytes);
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
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_empty + 2);
  float* qred = reinterpret_cast<float*>(bars + 64);  // quantize-phase block max [4]

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int cid = static_cast<int>(blockIdx.x) / p.C;
  const int rank = static_cast<int>(blockIdx.x) % p.C;

  if (warp == 0 && lane == 0) {
    if (p.quantize == 0)
      for (int i = 0; i < p.nprob; ++i) prefetch_tensormap(&maps.m[i]);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1 + 4);
      mbar_init(&sc_empty[i], 4);
    }
    for (int i = 0; i < Cf::kNA; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < Cf::kND; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pb_full[i], 4);
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

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      auto load_static = [&](const GCur<S>& c, int stage) {
        const GProb& q = p.prob[c.pi];
        const int kb = c.kb(), nkb = c.nkb();
        const int32_t* src = PATH == ISB_PATH_INTEGER_SCALE
                                 ? q.kscale : reinterpret_cast<const int32_t*>(q.fscale);
        mbar_arrive_expect_tx(&full[stage], nkb * (kBlockBytes + Cf::kXBytes + kTileN * 4));
        bulk_load_evict_first(smem_w + stage * S * kBlockBytes,
                              q.packed + (static_cast<int64_t>(c.nt) * q.kblocks + kb) * kBlockBytes,
                              nkb * kBlockBytes, &full[stage]);
        bulk_load(smem_sc + stage * Cf::kScBytes,
                  src + (static_cast<int64_t>(c.nt) * q.G + kb) * kTileN, nkb * kTileN * 4,
                  &full[stage]);
      };
      // Weights and scales do not depend on the preceding grid or on the
      // quantize phase: the first kStages steps go out before griddepcontrol.wait.
      GCur<S> a;
      a.init(p, cid, rank);
      int pre = 0;
      for (; pre < kStages && a.valid(); ++pre, a.next()) load_static(a, pre);
      pdl_wait();
      uint32_t seen = 0;
      GCur<S> cur;
      cur.init(p, cid, rank);
      for (int j = 0; cur.valid(); ++j, cur.next()) {
        const int stage = j % kStages;
        if (j >= pre) {
          mbar_wait(&empty[stage], ((j / kStages) & 1) ^ 1);
          mbar_wait(&sc_empty[stage], ((j / kStages) & 1) ^ 1);
          load_static(cur, stage);
        }
        if (p.quantize && !((seen >> cur.pi) & 1u)) {
          // codes of this problem written by the quantize phase (generic proxy,
          // other SMs): acquire the row count, then order the TMA reads after it
          wait_rows(&p.sync[cur.pi], static_cast<unsigned>(p.prob[cur.pi].M));
          fence_proxy_async_global();
          prefetch_tensormap(&maps.m[cur.pi]);
          seen |= 1u << cur.pi;
        }
        const int kb = cur.kb(), nkb = cur.nkb();
        for (int i = 0; i < nkb; ++i)
          tma_load_2d(smem_x + (stage * S + i) * kXSlot, &maps.m[cur.pi], &full[stage],
                      (kb + i) * kBlockK, cur.mt * MT);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp)
    constexpr uint32_t idesc = make_idesc_i8(128, MT);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t x_base = smem_u32(smem_x);
    GCur<S> cur;
    cur.init(p, cid, rank);
    for (int j = 0; cur.valid(); ++j, cur.next()) {
      const int stage = j % kStages, as = j % Cf::kNA, ds = j % Cf::kND;
      const int nkb = cur.nkb();
      mbar_wait(&a_full[as], (j / Cf::kNA) & 1);  // implies full[stage] (transform saw it)
      mbar_wait(&d_empty[ds], ((j / Cf::kND) & 1) ^ 1);
      tc_fence_after();
#pragma unroll
      for (int i = 0; i < S; ++i) {
        if (i < nkb) {
          const uint64_t bdesc = make_sw128_kmajor_desc(x_base + (stage * S + i) * kXSlot);
          const uint32_t d_tmem = tbase + Cf::kNA * Cf::kACols + ds * Cf::kDCols + i * MT;
          const uint32_t a_tmem = tbase + as * Cf::kACols + i * 32;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            mma_i8_ts_warp(d_tmem, a_tmem + c * 8, bdesc + static_cast<uint64_t>(c * 2), idesc,
                           c > 0 ? 1u : 0u);
        }
      }
      mma_commit_warp(&empty[stage]);
      mma_commit_warp(&a_empty[as]);
      mma_commit_warp(&d_full[ds]);
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------------------------------------------------------- transform
    const int xw = static_cast<int>(warp - 4) / 4;
    const uint32_t r = (warp % 4) * 32 + lane;  // output channel within the tile == TMEM lane
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t w_base = smem_u32(smem_w) + r * 16;
    GCur<S> cur;
    cur.init(p, cid, rank);
    for (int j = 0; cur.valid(); ++j, cur.next()) {
      if ((j & 1) != xw) continue;
      const int stage = j % kStages, as = j % Cf::kNA;
      const int nkb = cur.nkb();
      mbar_wait(&full[stage], (j / kStages) & 1);
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
          tmem_st_x32(tmem_base + lane_base + as * Cf::kACols + i * 32, a);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[as]);
    }
  } else if (warp >= 12) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t tid = threadIdx.x - 384;
    const uint32_t r = (warp % 4) * 32 + lane;  // TMEM lane == output channel in tile
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    pdl_wait();  // activations / counters / outputs may belong to the preceding grid
    if (p.quantize) {
      // ---- quantize phase: token rows blockIdx.x, blockIdx.x + gridDim.x, ...
      for (int t = blockIdx.x; t < p.qtasks; t += gridDim.x) {
        int pi = 0;
        while (t >= p.qoff[pi + 1]) ++pi;
        const GProb& q = p.prob[pi];
        const int row = t - p.qoff[pi];
        int8_t* cr = q.xq + static_cast<int64_t>(row) * q.K;
        if (q.x_dtype == ISB_F32)
          quant_row<float>(static_cast<const float*>(q.xf) + static_cast<int64_t>(row) * q.K, q.K,
                           cr, q.sa_w + row, qred, tid, &p.sync[kSyncBad]);
        else
          quant_row<__nv_bfloat16>(
              static_cast<const __nv_bfloat16*>(q.xf) + static_cast<int64_t>(row) * q.K, q.K, cr,
              q.sa_w + row, qred, tid, &p.sync[kSyncBad]);
        fence_proxy_async_global();  // codes are read by TMA (async proxy) on other SMs
        named_bar_sync(4, 128);      // whole row written (and qred consumed)
        if (tid == 0) red_release_gpu_add(&p.sync[pi], 1u);
      }
    }
    const uint32_t pbuf_local = smem_u32(pbuf);
    GCur<S> cur;
    cur.init(p, cid, rank);
    int j = 0;
    for (int it = 0; cur.valid(); ++it) {
      const bool late = p.prob[cur.pi].late_shift != 0;
      int32_t iacc[kCols];
      float facc[kCols];
#pragma unroll
      for (int t = 0; t < kCols; ++t) { iacc[t] = 0; facc[t] = 0.0f; }
      bool last;
      do {
        const int ds = j % Cf::kND, stage = j % kStages;
        const int nkb = cur.nkb();
        mbar_wait(&d_full[ds], (j / Cf::kND) & 1);
        mbar_wait(&full[stage], (j / kStages) & 1);  // scales of this step landed
        tc_fence_after();
        const uint32_t sc_base = smem_u32(smem_sc + stage * Cf::kScBytes) + r * 4;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          if (i < nkb) {
            const uint32_t sraw = ld_shared_u32(sc_base + i * (kTileN * 4));
            const int32_t kg = static_cast<int32_t>(sraw);
            const float sg = __uint_as_float(sraw);
            const uint32_t taddr =
                tmem_base + lane_base + Cf::kNA * Cf::kACols + ds * Cf::kDCols + i * MT;
            constexpr int kChunk = kCols < 16 ? kCols : 16;
#pragma unroll
            for (int cc = 0; cc < kCols; cc += kChunk) {
              uint32_t v[16];
              if constexpr (kChunk == 16) tmem_ld_x16_(taddr + cc, v);
              else tmem_ld_x8(taddr + cc, *reinterpret_cast<uint32_t(*)[8]>(&v[0]));
              tmem_wait_ld();
#pragma unroll
              for (int t = 0; t < kChunk; ++t) {
                const int32_t d = static_cast<int32_t>(v[t]);  // 16 * P_g, exact
                if (PATH == ISB_PATH_INTEGER_SCALE) {
                  if (late) iacc[cc + t] += d * kg;            // shift once at the end
                  else iacc[cc + t] += (d >> 4) * kg;
                } else {
                  facc[cc + t] = fmaf(static_cast<float>(d), sg, facc[cc + t]);  // Eq. 1, fp32
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
        last = cur.last_step();
        ++j;
        cur.next();
      } while (!last);
      if (PATH == ISB_PATH_INTEGER_SCALE && late) {
#pragma unroll
        for (int t = 0; t < kCols; ++t) iacc[t] >>= 4;  // exact: 16 | acc16
      }
      // hand the tile's partial to the reduction warps
      const int buf = it % Cf::kPbufs;
      mbar_wait_cluster(&red_empty[buf], ((it / Cf::kPbufs) & 1) ^ 1);
      const uint32_t pb = pbuf_local + buf * (MT * kTileN * 4);
#pragma unroll
      for (int t = 0; t < kCols; ++t)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(pb + (t * kTileN + r) * 4),
                     "r"(PATH == ISB_PATH_INTEGER_SCALE ? static_cast<uint32_t>(iacc[t])
                                                        : __float_as_uint(facc[t]))
                     : "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&pb_full[buf]);
    }
  } else {
    // ---------------------------------------------------------------- reduction warps (2, 3)
    pdl_wait();
    const uint32_t u = (warp - 2) * 32 + lane;  // rows u and u + 64
    const uint32_t pbuf_local = smem_u32(pbuf);
    const int ntiles = cid < p.NC ? p.sched_len[cid] : 0;
    const int* sched = p.sched + cid * p.sched_stride;
    uint32_t seen = 0;
    auto sa_prefetch = [&](int it) {
      if (it < ntiles) {
        const int e = sched[it];
        const int pi = e >> 24;
        const GProb& q = p.prob[pi];
        if (p.quantize && !((seen >> pi) & 1u)) {
          wait_rows(&p.sync[pi], static_cast<unsigned>(q.M));
          seen |= 1u << pi;
        }
        if (u < static_cast<uint32_t>(MT)) {
          const int64_t m = static_cast<int64_t>((e & 0xFFFFFF) % q.m_tiles) * MT + u;
          const uint32_t dst = smem_u32(sa_s + (it & 1) * MT + u);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst),
                       "l"(q.sa + (m < q.M ? m : 0)), "r"(m < q.M ? 8 : 0)
                       : "memory");
        }
      }
      cp_async_commit();
    };
    sa_prefetch(0);
    for (int it = 0; it < ntiles; ++it) {
      const int buf = it % Cf::kPbufs;
      const uint32_t ph = (it / Cf::kPbufs) & 1;
      const int e = sched[it];
      const GProb& q = p.prob[e >> 24];
      const int nt = (e & 0xFFFFFF) / q.m_tiles, mt = (e & 0xFFFFFF) % q.m_tiles;
      sa_prefetch(it + 1);
      cp_async_wait<1>();
      named_bar_sync(2, 64);  // sa_s[it & 1] visible to both reduction warps
      const double* sa_t = sa_s + (it & 1) * MT;
      mbar_wait(&pb_full[buf], ph);
      if (p.C > 1) {
        if (lane < static_cast<uint32_t>(p.C))
          mbar_arrive_remote_release(mapa_shared(smem_u32(&red_full[buf]), lane));
        mbar_wait_cluster(&red_full[buf], ph);
      }
      const uint32_t pb = pbuf_local + buf * (MT * kTileN * 4);
      switch (p.C) {
        case 1: reduce_tile<MT, 1, PATH>(q, pb, sa_t, rank, nt, mt, u); break;
        case 2: reduce_tile<MT, 2, PATH>(q, pb, sa_t, rank, nt, mt, u); break;
        case 4: reduce_tile<MT, 4, PATH>(q, pb, sa_t, rank, nt, mt, u); break;
        default: reduce_tile<MT, 8, PATH>(q, pb, sa_t, rank, nt, mt, u); break;
      }
      named_bar_sync(2, 64);  // done with sa_s[it & 1] before it is refilled
      if (p.C > 1) {
        if (lane < static_cast<uint32_t>(p.C))
          mbar_arrive_remote(mapa_shared(smem_u32(&red_empty[buf]), lane));
      } else if (lane == 0) {
        mbar_arrive(&red_empty[buf]);
      }
    }
    // Do not retire while peers may still read our partials.
    for (int it = max(0, ntiles - Cf::kPbufs); it < ntiles; ++it)
      mbar_wait_cluster(&red_empty[it % Cf::kPbufs], (it / Cf::kPbufs) & 1);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, Cf::kTmemCols);
  if (p.quantize && threadIdx.x == 0) {
    // every CTA's polls are behind it: the last one to retire re-arms the counters
    const unsigned prev = atom_add_acq_rel_gpu(&p.sync[kSyncDone], 1u);
    if (prev == gridDim.x - 1) {
      for (int i = 0; i < p.nprob; ++i) p.sync[i] = 0u;
      p.sync[kSyncDone] = 0u;
    }
  }
}

template <int MT, int PATH>
void prepare_group_kernel() {
  static std::once_flag once;
  std::call_once(once, [] {
    auto kern = gemm_w4a8_group<MT, PATH>;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Cfg<MT, false>::kSmemBytes),
               "cudaFuncSetAttribute(smem)");
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
               "cudaFuncSetAttribute(cluster)");
  });
}

template <int MT, int PATH>
int group_capacity(int C) {
  prepare_group_kernel<MT, PATH>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C * 64);
  cfg.blockDim = dim3(Cfg<MT, false>::kThreads);
  cfg.dynamicSmemBytes = Cfg<MT, false>::kSmemBytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_w4a8_group<MT, PATH>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int group_capacity_cached(int mt, int path, int C) {
  static std::mutex mu;
  static int cache[2][2][9] = {};
  std::lock_guard<std::mutex> lk(mu);
  int& slot = cache[mt == 16 ? 0 : 1][path == ISB_PATH_INTEGER_SCALE ? 1 : 0][C];
  if (!slot) {
    int n = 0;
    if (mt == 16)
      n = path == ISB_PATH_INTEGER_SCALE ? group_capacity<16, ISB_PATH_INTEGER_SCALE>(C)
                                         : group_capacity<16, ISB_PATH_FLOAT_SCALE>(C);
    else
      n = path == ISB_PATH_INTEGER_SCALE ? group_capacity<32, ISB_PATH_INTEGER_SCALE>(C)
                                         : group_capacity<32, ISB_PATH_FLOAT_SCALE>(C);
    slot = n > 0 ? n : -1;
  }
  return slot;
}

template <int MT, int PATH>
void launch_group_mt(const GMaps& maps, const GParams& prm, int grid, cudaStream_t s) {
  prepare_group_kernel<MT, PATH>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg<MT, false>::kThreads);
  cfg.dynamicSmemBytes = Cfg<MT, false>::kSmemBytes;
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
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_group<MT, PATH>, maps, prm),
             "gemm_w4a8_group launch");
  count_launch();
}

}  // namespace

// ---------------------------------------------------------------------------- plan (host)
struct GroupPlan {
  GParams prm{};
  GMaps maps{};
  int mt = 16, path = ISB_PATH_INTEGER_SCALE, grid = 0, dev = 0;
  double makespan = 0.0;
  int* sched_dev = nullptr;   // schedule + lengths
  unsigned* sync_dev = nullptr;
  void* owned = nullptr;      // plan-owned codes / scales when the caller passes none
  ~GroupPlan() {
    if (sched_dev) cudaFree(sched_dev);
    if (sync_dev) cudaFree(sync_dev);
    if (owned) cudaFree(owned);
  }
};

namespace {

int pick_group_mt(int64_t max_m) {
  return max_m <= 16 ? 16 : 32;  // 33..64 (and beyond) as 32-token tiles (gemm_tc.cu pick_mt)
}

}  // namespace

GroupPlan* group_plan_create(const isb_group_problem* probs, int nprob, int path, int out_dtype,
                             int num_sms) {
  if (nprob < 1 || nprob > kMaxGroup)
    fail(ISB_PARAM, "grouped GEMM: 1.." + std::to_string(kMaxGroup) + " problems");
  if (path != ISB_PATH_INTEGER_SCALE && path != ISB_PATH_FLOAT_SCALE)
    fail(ISB_PARAM, "grouped GEMM: path must be integer-scale or float-scale");
  if (out_dtype != ISB_F32 && out_dtype != ISB_BF16 && out_dtype != ISB_F16 &&
      out_dtype != ISB_I32)
    fail(ISB_PARAM, "unsupported output dtype");
  if (out_dtype == ISB_I32 && path != ISB_PATH_INTEGER_SCALE)
    fail(ISB_PARAM, "raw int32 accumulator output exists only on the integer-scale path");
  int64_t max_m = 0;
  int quantize = -1;
  int64_t own_bytes = 0;
  for (int i = 0; i < nprob; ++i) {
    const isb_group_problem& q = probs[i];
    if (!q.w) fail(ISB_PARAM, "grouped GEMM: null weight handle (problem " + std::to_string(i) + ")");
    const isb_weight& w = *q.w;
    if (!w.tensor_core_ok() || w.group != kBlockK)
      fail(ISB_PARAM, "grouped GEMM needs group == 128 and K % 128 == 0");
    if (path == ISB_PATH_INTEGER_SCALE && !w.has_int_scales)
      fail(ISB_PARAM, "integer-scale path needs an IntegerScaleSet");
    if (path == ISB_PATH_INTEGER_SCALE &&
        w.static_bound > std::numeric_limits<int32_t>::max())
      fail(ISB_OVERFLOW, "static overflow bound " + std::to_string(w.static_bound) +
                             " exceeds int32 (problem " + std::to_string(i) +
                             "): the tensor-core integer-scale GEMM cannot be exact");
    if (q.m < 0 || q.m > (1 << 20)) fail(ISB_PARAM, "grouped GEMM: bad M");
    if (q.m > 0 && !q.out) fail(ISB_PARAM, "grouped GEMM: null output");
    const int qz = q.x != nullptr ? 1 : 0;
    if (quantize >= 0 && qz != quantize)
      fail(ISB_PARAM, "grouped GEMM: either every problem passes float activations or none");
    quantize = qz;
    if (qz) {
      if (q.x_dtype != ISB_F32 && q.x_dtype != ISB_BF16)
        fail(ISB_PARAM, "grouped GEMM: activations must be float32 or bf16");
      if (!q.xq) own_bytes += (q.m * w.k + 255) / 256 * 256;
      if (!q.sa) own_bytes += (q.m * 8 + 255) / 256 * 256;
    } else if (q.m > 0 && (!q.xq || !q.sa)) {
      fail(ISB_PARAM, "grouped GEMM: null activation pointer");
    }
    max_m = std::max(max_m, q.m);
  }
  auto* pl = new GroupPlan();
  try {
    cuda_check(cudaGetDevice(&pl->dev), "cudaGetDevice");
    pl->path = path;
    pl->mt = pick_group_mt(max_m);
    const int mt = pl->mt;
    const int S = mt <= 32 ? 4 : 2;
    if (own_bytes) cuda_check(cudaMalloc(&pl->owned, own_bytes), "cudaMalloc(group workspace)");
    uint8_t* own = static_cast<uint8_t*>(pl->owned);
    GParams& P = pl->prm;
    P.nprob = nprob;
    P.quantize = quantize;
    int min_groups = std::numeric_limits<int>::max();
    std::vector<int64_t> tiles(nprob);
    P.qoff[0] = 0;
    for (int i = 0; i < nprob; ++i) {
      const isb_group_problem& q = probs[i];
      const isb_weight& w = *q.w;
      GProb& g = P.prob[i];
      g.packed = w.packed;
      g.kscale = w.kscale_tiled;
      g.fscale = w.fscale_tiled;
      g.out = q.out;
      g.xf = q.x;
      g.xq = q.xq;
      g.sa_w = q.sa;
      if (quantize && q.m > 0) {
        if (!g.xq) { g.xq = reinterpret_cast<int8_t*>(own); own += (q.m * w.k + 255) / 256 * 256; }
        if (!g.sa_w) { g.sa_w = reinterpret_cast<double*>(own); own += (q.m * 8 + 255) / 256 * 256; }
      }
      g.sa = quantize ? g.sa_w : q.sa;
      g.wscale_d = nullptr;
      g.inv_amp = std::ldexp(1.0, -w.exponent);
      g.M = static_cast<int>(q.m);
      g.N = static_cast<int>(w.n);
      g.G = static_cast<int>(w.groups);
      g.K = static_cast<int>(w.k);
      g.kblocks = static_cast<int>(w.kblocks);
      g.m_tiles = static_cast<int>((q.m + mt - 1) / mt);
      g.out_dtype = out_dtype;
      g.late_shift = (path == ISB_PATH_INTEGER_SCALE && w.static_bound > 0 &&
                      w.static_bound <= (int64_t{1} << 27) - 1) ? 1 : 0;
      g.x_dtype = q.x_dtype;
      tiles[i] = static_cast<int64_t>(w.n_tiles) * g.m_tiles;
      if (q.m > 0) {
        min_groups = std::min(min_groups, g.G);
        pl->maps.m[i] = make_x_map(g.xq, q.m, w.k, mt);
      }
      P.qoff[i + 1] = P.qoff[i] + (quantize ? g.M : 0);
    }
    P.qtasks = P.qoff[nprob];
    const int64_t total_tiles = std::accumulate(tiles.begin(), tiles.end(), int64_t{0});
    if (total_tiles >= (int64_t{1} << 24)) fail(ISB_PARAM, "grouped GEMM: too many tiles");
    // Split-K width C and the schedule: longest-processing-time-first over the
    // co-resident clusters; a tile costs its steps per rank plus ~half a step of
    // hand-off (+ the cluster exchange), as in plan_gemm (gemm_tc.cu).
    static const int force_c = [] {
      const char* e = std::getenv("ISB_GROUP_C");
      return e ? std::atoi(e) : 0;
    }();
    double best = 1e30;
    std::vector<std::vector<int>> best_lists;
    int best_c = 1;
    for (int C : {1, 2, 4, 8}) {
      if (total_tiles == 0) break;
      if (C > min_groups) break;
      if (force_c && C != force_c) continue;
      int cap = group_capacity_cached(mt, path, C);
      if (cap <= 0) continue;
      cap = std::min(cap, num_sms / C);
      const int nc = static_cast<int>(std::min<int64_t>(cap, total_tiles));
      struct T { double cost; int entry; };
      std::vector<T> all;
      all.reserve(static_cast<size_t>(total_tiles));
      for (int i = 0; i < nprob; ++i) {
        const int g_cta = (P.prob[i].G + C - 1) / C;
        const double cost = std::ceil(static_cast<double>(g_cta) / S) + 0.5 + (C > 1 ? 0.25 : 0.0);
        for (int64_t t = 0; t < tiles[i]; ++t) all.push_back({cost, (i << 24) | static_cast<int>(t)});
      }
      std::stable_sort(all.begin(), all.end(), [](const T& a, const T& b) { return a.cost > b.cost; });
      using L = std::pair<double, int>;
      std::priority_queue<L, std::vector<L>, std::greater<L>> heap;
      for (int c = 0; c < nc; ++c) heap.push({0.0, c});
      std::vector<std::vector<int>> lists(nc);
      for (const T& t : all) {
        L l = heap.top();
        heap.pop();
        lists[l.second].push_back(t.entry);
        heap.push({l.first + t.cost, l.second});
      }
      double mk = 0.0;
      while (!heap.empty()) { mk = std::max(mk, heap.top().first); heap.pop(); }
      if (mk < best - 1e-9) {
        best = mk;
        best_c = C;
        best_lists = std::move(lists);
      }
    }
    if (total_tiles > 0 && best_lists.empty())
      fail(ISB_CUDA, "grouped GEMM: no cluster configuration fits the device");
    P.C = best_c;
    P.NC = static_cast<int>(best_lists.size());
    pl->makespan = best;
    size_t stride = 1;
    for (auto& l : best_lists) stride = std::max(stride, l.size());
    P.sched_stride = static_cast<int>(stride);
    std::vector<int> host(static_cast<size_t>(P.NC) * stride + P.NC + 1, 0);
    for (int c = 0; c < P.NC; ++c) {
      std::copy(best_lists[c].begin(), best_lists[c].end(), host.begin() + c * stride);
      host[static_cast<size_t>(P.NC) * stride + c] = static_cast<int>(best_lists[c].size());
    }
    cuda_check(cudaMalloc(&pl->sched_dev, host.size() * sizeof(int)), "cudaMalloc(schedule)");
    cuda_check(cudaMemcpy(pl->sched_dev, host.data(), host.size() * sizeof(int),
                          cudaMemcpyHostToDevice),
               "copy schedule");
    P.sched = pl->sched_dev;
    P.sched_len = pl->sched_dev + static_cast<size_t>(P.NC) * stride;
    cuda_check(cudaMalloc(&pl->sync_dev, kSyncWords * sizeof(unsigned)), "cudaMalloc(sync)");
    cuda_check(cudaMemset(pl->sync_dev, 0, kSyncWords * sizeof(unsigned)), "cudaMemset(sync)");
    P.sync = pl->sync_dev;
    pl->grid = P.NC * P.C;
  } catch (...) {
    delete pl;
    throw;
  }
  return pl;
}

void group_plan_run(GroupPlan* pl, cudaStream_t s) {
  if (pl->grid == 0) return;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev != pl->dev) fail(ISB_PARAM, "grouped GEMM plan used on another device");
  if (pl->mt == 16) {
    if (pl->path == ISB_PATH_INTEGER_SCALE)
      launch_group_mt<16, ISB_PATH_INTEGER_SCALE>(pl->maps, pl->prm, pl->grid, s);
    else
      launch_group_mt<16, ISB_PATH_FLOAT_SCALE>(pl->maps, pl->prm, pl->grid, s);
  } else {
    if (pl->path == ISB_PATH_INTEGER_SCALE)
      launch_group_mt<32, ISB_PATH_INTEGER_SCALE>(pl->maps, pl->prm, pl->grid, s);
    else
      launch_group_mt<32, ISB_PATH_FLOAT_SCALE>(pl->maps, pl->prm, pl->grid, s);
  }
}

void group_plan_info(const GroupPlan* pl, isb_group_info_t* info) {
  info->grid = pl->grid;
  info->cluster = pl->prm.C;
  info->tile_tokens = pl->mt;
  info->quantize = pl->prm.quantize;
  info->makespan_steps = pl->makespan;
}

void group_plan_destroy(GroupPlan* pl) { delete pl; }

int group_plan_nonfinite(GroupPlan* pl, bool clear) {
  unsigned h = 0;
  cuda_check(cudaMemcpy(&h, pl->sync_dev + kSyncBad, sizeof(unsigned), cudaMemcpyDeviceToHost),
             "read flag");
  if (clear && h) cuda_check(cudaMemset(pl->sync_dev + kSyncBad, 0, sizeof(unsigned)), "clear flag");
  return h != 0;
}

}  // namespace isb
