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
// are spread evenly over the SMs (below), so the tail is paid once per layer
// instead of once per GEMM.
//
// Per CTA the pipeline is the single-GEMM decode pipeline (gemm_tc.cu): producer
// warp (bulk copy of packed int4 weights + int32 k_g, TMA of int8 activation
// tiles), two transform warpgroups (int4 -> TMEM int8), MMA warp
// (tcgen05.mma.kind::i8, TMEM accumulators), epilogue warpgroup (per-group
// IMAD / FFMA), two reduction warps (Eq. 2 and the output stores). What differs:
//
//   schedule        one CTA per SM, no clusters. The host lays the (problem,
//                   tile) work out McNaughton-style: tiles are poured in order
//                   into per-CTA budgets of equal length, a tile that crosses a
//                   budget boundary continues on the next CTA. Every CTA gets
//                   the same number of 128-K blocks (+- one block), whatever
//                   the mix of K over the problems, and at most one tile per
//                   CTA boundary is split. A tile split into pieces is reduced
//                   through global memory in fixed piece order: each piece
//                   stores its partial (int32 or fp32) to its own slot, counts
//                   itself in with an acq_rel add, and the piece that completes
//                   the count sums the slots 0..n-1 and applies the epilogue —
//                   deterministic, and exact on the integer path;
//   quantize phase  CTA b quantizes token rows b, b + grid, ... of the
//                   concatenated problems (all its threads, exact K1 arithmetic,
//                   quant.cuh) into the problem's int8 code buffer and double
//                   scales, then publishes the row with a gpu-scope release add
//                   on the problem's readiness counter;
//   consumers       the producer (before the first TMA of a problem's codes)
//                   and the reduction warps (before reading its token scales)
//                   acquire-poll the counter until all M rows are in. The first
//                   kStages weight steps are in flight before
//                   griddepcontrol.wait;
//   replays         the readiness counters are cumulative; each CTA takes a
//                   ticket (64-bit atomic) before the launch triggers its
//                   dependents, and ticket / grid is the launch epoch the
//                   waits are relative to; every split finisher zeroes its own
//                   counter. A plan replays (CUDA graphs) with no memset node
//                   and no end-of-kernel atomic. All CTAs are co-resident
//                   (grid <= the occupancy-derived capacity), so the polls
//                   cannot deadlock.
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
constexpr int kSyncTicket = kMaxGroup;    // 64-bit CTA ticket counter (launch epoch)
constexpr int kSyncBad = kMaxGroup + 2;   // non-finite activation seen (sticky)
constexpr int kSyncWords = kMaxGroup + 4;

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
  int nprob, NC, quantize, qtasks, sched_stride;
  const int4* sched;        // [NC][sched_stride] pieces: {p << 24 | tile, g0 << 16 | g1,
                            //  piece << 16 | npieces, split id (-1: whole tile)}
  const int* sched_len;     // [NC]
  const int* split_base;    // [nsplit] first partial slot of each split tile
  uint32_t* partials;       // [slots][MT][128] int32 / fp32 piece partials
  unsigned* sync;           // [kSyncWords] + [nsplit] split-tile piece counters
  int dbg;                  // measurement knobs (isb_debug_set_flags): 1 skip TMEM st,
                            // 2 skip TMEM ld, 4 skip MMA, 8 skip the activation wait,
                            // 16 no weight prefetch before the quantize phase,
                            // 32 launch-overhead probe (no work), 64 no activation
                            // TMA, 128 no scale loads, 256 no output / reduction,
                            // 2048 pieces finalised locally (wrong sums), 4096 no Eq. 2,
                            // 8192 no output stores
                            
  int64_t* trace;           // optional per-CTA timeline [4][512] (isb_debug_set_trace)
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

// Spin (with back-off) until all `rows` rows of a problem are published in this
// launch. The counters are cumulative over launches: launch `epoch` waits for
// epoch * rows + rows (modulo 2^32).
ISB_DEVICE void wait_rows(const unsigned* ctr, unsigned epoch, unsigned rows) {
  const unsigned base = epoch * rows;
  while (ld_acquire_gpu(ctr) - base < rows) __nanosleep(32);
}

// Eq. 2 / Eq. 1 with the token scale pre-multiplied by 2^-e on the integer path:
// float((double(acc) * 2^-e) * s_a) == float(double(acc) * (s_a * 2^-e)) since both
// power-of-two scalings are exact (gemm.cpp:252).
template <int PATH>
__device__ __forceinline__ float finish_eq(int32_t iacc, float facc, double s) {
  return __double2float_rn(__dmul_rn(PATH == ISB_PATH_INTEGER_SCALE ? static_cast<double>(iacc)
                                                                    : static_cast<double>(facc),
                                     s));
}

// The CTA's walk over its pieces, one step (S 128-K blocks = S groups of one
// piece) at a time.
template <int S>
struct GCur {
  const GProb* probs;
  const int4* list;
  int it, ntiles, sj, nst, pi, nt, mt, kb0, kb1;
  __device__ void init(const GProb* probs_, const int4* list_, int ntiles_) {
    probs = probs_;
    list = list_;
    ntiles = ntiles_;
    it = 0;
    sj = 0;
    if (ntiles > 0) load();
  }
  __device__ void load() {
    const int4 e = list[it];
    pi = e.x >> 24;
    const int t = e.x & 0xFFFFFF;
    const GProb& q = probs[pi];
    nt = t / q.m_tiles;
    mt = t - nt * q.m_tiles;
    kb0 = e.y >> 16;
    kb1 = e.y & 0xFFFF;
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

// Per-CTA copies of the problem table and of the CTA's piece list (kernel
// parameters and the schedule otherwise cost a dependent L2/HBM round trip on
// every first touch, microseconds while the weight stream saturates HBM).
constexpr int kSchedSmem = 256;  // pieces per CTA held in shared memory
static_assert((kMaxGroup * sizeof(GProb)) % 16 == 0, "schedule copy alignment");
constexpr int kTableBytes = kMaxGroup * static_cast<int>(sizeof(GProb)) + kSchedSmem * 16 + 64;

// K1 on one token row by the whole CTA (kThreads threads): exact
// quantize.cpp:93-145 arithmetic (float absmax, s = double(amax) / 127, codes via
// quant_one), i.e. bit-identical to quantize_rows_* in quant.cu. Every load of a
// row of up to kThreads * 4 * V elements is issued before the first use (one
// memory round trip: the row is read while the weight stream saturates HBM, so
// each dependent round trip costs microseconds), and the codes are computed
// from the same registers.
template <int NT, typename T>
__device__ __forceinline__ void quant_row_cta(const T* __restrict__ xr, int K,
                                              int8_t* __restrict__ cr, double* s_out, float* red,
                                              uint32_t tid, unsigned* bad) {
  constexpr int V = 8;
  constexpr int kBatch = NT * V;  // 4-element groups per batch
  const int nv = K >> 2;          // K % 128 == 0
  float v[V][4];
  float mx = 0.0f;
  bool fin = true;
  for (int b0 = 0; b0 < nv; b0 += kBatch) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int e = b0 + u * NT + static_cast<int>(tid);
      if (e < nv) load4<T>(xr + 4 * e, v[u]);
    }
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int e = b0 + u * NT + static_cast<int>(tid);
      if (e < nv)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          fin = fin && isfinite(v[u][c]);
          mx = fmaxf(mx, fabsf(v[u][c]));
        }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) red[tid / 32] = mx;
  if (!fin) atomicOr(bad, 1u);
  __syncthreads();
  mx = 0.0f;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) mx = fmaxf(mx, red[w]);
  const double s = mx == 0.0f ? 1.0 : static_cast<double>(mx) / 127.0;  // quantize.cpp:120-125
  const double r = 1.0 / s;
  if (tid == 0) *s_out = s;
  const int last = (nv - 1) / kBatch * kBatch;  // the batch still in registers
  for (int b0 = 0; b0 < nv; b0 += kBatch) {
    if (b0 != last) {  // rows longer than one batch (K > NT * 4 * V): reload
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int e = b0 + u * NT + static_cast<int>(tid);
        if (e < nv) load4<T>(xr + 4 * e, v[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int e = b0 + u * NT + static_cast<int>(tid);
      if (e < nv) {
        uint32_t packed = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          packed |= (static_cast<uint32_t>(quant_one(v[u][c], s, r, -128, 127)) & 0xFFu)
                    << (8 * c);
        *reinterpret_cast<uint32_t*>(cr + 4 * e) = packed;
      }
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
  uint64_t* red_empty = pb_full + 2;        // [2] reduction warps done with a partial buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_empty + 2);
  float* qred = reinterpret_cast<float*>(bars + 64);  // quantize-phase block max [16]

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (threadIdx.x == 0 && p.trace) p.trace[4 * 512 + blockIdx.x] = globaltimer_();
  const int cta = static_cast<int>(blockIdx.x);
  uint32_t* flag_s = reinterpret_cast<uint32_t*>(bars + 80);  // split finisher flag
  uint32_t* epoch_s = flag_s + 1;                                // this launch's epoch
  GProb* probs_s = reinterpret_cast<GProb*>(reinterpret_cast<uint8_t*>(bars) + 1024);
  int4* sched_s = reinterpret_cast<int4*>(probs_s + kMaxGroup);
  const int ntiles = cta < p.NC ? p.sched_len[cta] : 0;
  const int4* list = ntiles <= kSchedSmem ? sched_s : p.sched + cta * p.sched_stride;
  if (warp == 3) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(p.prob);
    uint32_t* dst = reinterpret_cast<uint32_t*>(probs_s);
    for (int i = lane; i < p.nprob * static_cast<int>(sizeof(GProb) / 4); i += 32) dst[i] = src[i];
    if (ntiles <= kSchedSmem)
      for (int i = lane; i < ntiles; i += 32) sched_s[i] = p.sched[cta * p.sched_stride + i];
  }

  // Launch epoch: every CTA of a launch takes its ticket before the launch lets
  // its dependents start (griddepcontrol.launch_dependents below), and every
  // launch has gridDim.x CTAs, so ticket / gridDim.x numbers the launches.
  unsigned long long ticket = 0;
  if (threadIdx.x == 0 && p.quantize)
    ticket = atomicAdd(reinterpret_cast<unsigned long long*>(p.sync + kSyncTicket), 1ull);
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
      mbar_init(&red_empty[i], 2);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cf::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) {
    *epoch_s = static_cast<unsigned>(ticket / gridDim.x);  // ticket performed before the trigger
    pdl_launch_dependents();
  }
  if (threadIdx.x == 0 && p.trace) p.trace[blockIdx.x] = globaltimer_();

  // Producer lane 0: weights and scales do not depend on the preceding grid or on
  // the quantize phase, so the first kStages steps go out before
  // griddepcontrol.wait.
  auto load_static = [&](const GCur<S>& c, int stage) {
    const GProb& q = probs_s[c.pi];
    const int kb = c.kb(), nkb = c.nkb();
    const int32_t* src = PATH == ISB_PATH_INTEGER_SCALE
                             ? q.kscale : reinterpret_cast<const int32_t*>(q.fscale);
    mbar_arrive_expect_tx(&full[stage],
                          nkb * (kBlockBytes + ((p.dbg & 64) ? 0 : Cf::kXBytes) +
                                 ((p.dbg & 128) ? 0 : kTileN * 4)));
    bulk_load_evict_first(smem_w + stage * S * kBlockBytes,
                          q.packed + (static_cast<int64_t>(c.nt) * q.kblocks + kb) * kBlockBytes,
                          nkb * kBlockBytes, &full[stage]);
    if (!(p.dbg & 128))
      bulk_load(smem_sc + stage * Cf::kScBytes,
                src + (static_cast<int64_t>(c.nt) * q.G + kb) * kTileN, nkb * kTileN * 4,
                &full[stage]);
  };
  if (p.dbg & 32) {  // launch-overhead probe: setup, dependency wait, teardown only
    pdl_wait();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem_base, Cf::kTmemCols);
    return;
  }
  int pre = 0;
  if (threadIdx.x == 0 && !(p.dbg & 16)) {
    GCur<S> a;
    a.init(probs_s, list, ntiles);
    for (; pre < kStages && a.valid(); ++pre, a.next()) load_static(a, pre);
  }
  pdl_wait();  // activations / counters / outputs may belong to the preceding grid
  if (threadIdx.x == 0 && p.trace) p.trace[5 * 512 + blockIdx.x] = globaltimer_();
  if (p.quantize && static_cast<int>(blockIdx.x) < p.qtasks) {
    // ---- quantize phase (whole CTA): token rows blockIdx.x, blockIdx.x + gridDim.x, ...
    for (int t = blockIdx.x; t < p.qtasks; t += gridDim.x) {
      int pi = 0;
      while (t >= p.qoff[pi + 1]) ++pi;
      const GProb& q = probs_s[pi];
      const int row = t - p.qoff[pi];
      int8_t* cr = q.xq + static_cast<int64_t>(row) * q.K;
      if (q.x_dtype == ISB_F32)
        quant_row_cta<Cf::kThreads>(static_cast<const float*>(q.xf) + static_cast<int64_t>(row) * q.K,
                                    q.K, cr, q.sa_w + row, qred, threadIdx.x, &p.sync[kSyncBad]);
      else
        quant_row_cta<Cf::kThreads>(
            static_cast<const __nv_bfloat16*>(q.xf) + static_cast<int64_t>(row) * q.K, q.K, cr,
            q.sa_w + row, qred, threadIdx.x, &p.sync[kSyncBad]);
      fence_proxy_async_global();  // codes are read by TMA (async proxy) on other SMs
      __syncthreads();             // whole row written (and qred consumed)
      if (threadIdx.x == 0) red_release_gpu_add(&p.sync[pi], 1u);
    }
    if (threadIdx.x == 0 && p.trace) p.trace[2 * 512 + blockIdx.x] = globaltimer_();
  }

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      uint32_t seen = 0;
      GCur<S> cur;
      cur.init(probs_s, list, ntiles);
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
          if (!(p.dbg & 8))
            wait_rows(&p.sync[cur.pi], *epoch_s, static_cast<unsigned>(probs_s[cur.pi].M));
          fence_proxy_async_global();
          prefetch_tensormap(&maps.m[cur.pi]);
          if (seen == 0 && p.trace) p.trace[512 + blockIdx.x] = globaltimer_();
          seen |= 1u << cur.pi;
        }
        const int kb = cur.kb(), nkb = cur.nkb();
        for (int i = 0; i < nkb && !(p.dbg & 64); ++i)
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
    cur.init(probs_s, list, ntiles);
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
            if (!(p.dbg & 4))
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
    cur.init(probs_s, list, ntiles);
    for (int j = 0; cur.valid(); ++j, cur.next()) {
      if ((j & 1) != xw) continue;
      const int stage = j % kStages, as = j % Cf::kNA;
      const int nkb = cur.nkb();
      mbar_wait(&full[stage], (j / kStages) & 1);
      if (j == 0 && threadIdx.x == 128 && p.trace) p.trace[7 * 512 + blockIdx.x] = globaltimer_();
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
    }
  } else if (warp >= 12) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t r = (warp % 4) * 32 + lane;  // TMEM lane == output channel in tile
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t pbuf_local = smem_u32(pbuf);
    GCur<S> cur;
    cur.init(probs_s, list, ntiles);
    int j = 0;
    for (int it = 0; cur.valid(); ++it) {
      const bool late = probs_s[cur.pi].late_shift != 0;
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
              if (!(p.dbg & 2)) {
                if constexpr (kChunk == 16) tmem_ld_x16_(taddr + cc, v);
                else tmem_ld_x8(taddr + cc, *reinterpret_cast<uint32_t(*)[8]>(&v[0]));
                tmem_wait_ld();
              } else {
#pragma unroll
                for (int z = 0; z < 16; ++z) v[z] = z;
              }
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
      mbar_wait(&red_empty[buf], ((it / Cf::kPbufs) & 1) ^ 1);
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
    // Last TMEM access of the CTA (every MMA committed, every tcgen05.st waited
    // before its a_full): release TMEM now. tcgen05.dealloc completes only once
    // the CTA's outstanding global stores drain, so deallocating after the last
    // tile's output stores would hold the SM for microseconds under load.
    tc_fence_before();
    named_bar_sync(5, 128);
    if (threadIdx.x == 384 && p.trace) {
      p.trace[9 * 512 + blockIdx.x] = globaltimer_();
      p.trace[13 * 512 + blockIdx.x] = clock64_();
    }
    if (warp == 12) tmem_dealloc(tmem_base, Cf::kTmemCols);
  } else {
    // ---------------------------------------------------------------- reduction warps (2, 3)
    // Whole tiles: Eq. 2 / Eq. 1 straight from the partial buffer. Pieces of a
    // split tile: partial to the piece's global slot; the piece that completes the
    // tile's count sums the slots in piece order and finalises.
    const uint32_t u = (warp - 2) * 32 + lane;  // rows u and u + 64
    const uint32_t pbuf_local = smem_u32(pbuf);
    const int4* sched = list;
    uint32_t seen = 0;
    auto sa_prefetch = [&](int it) {
      if (it < ntiles) {
        const int4 e = sched[it];
        const int pi = e.x >> 24;
        const GProb& q = probs_s[pi];
        if (p.quantize && !((seen >> pi) & 1u)) {
          wait_rows(&p.sync[pi], *epoch_s, static_cast<unsigned>(q.M));
          seen |= 1u << pi;
        }
        if (u < static_cast<uint32_t>(MT)) {
          const int64_t m = static_cast<int64_t>((e.x & 0xFFFFFF) % q.m_tiles) * MT + u;
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
      const int4 e = sched[it];
      const GProb& q = probs_s[e.x >> 24];
      const int nt = (e.x & 0xFFFFFF) / q.m_tiles, mt = (e.x & 0xFFFFFF) % q.m_tiles;
      if (it == ntiles - 1 && u == 0 && p.trace) p.trace[12 * 512 + blockIdx.x] = globaltimer_();
      sa_prefetch(it + 1);
      cp_async_wait<1>();
      named_bar_sync(2, 64);  // sa_s[it & 1] visible to both reduction warps
      const double* sa_t = sa_s + (it & 1) * MT;
      mbar_wait(&pb_full[buf], ph);
      if (it == ntiles - 1 && u == 0 && p.trace) p.trace[10 * 512 + blockIdx.x] = globaltimer_();
      // The CTA's last tile, if whole, is finalised by all warps after their
      // roles end (below): on the critical path, 4 outputs per thread instead of
      // 32 per reduction-warp thread.
      if (it == ntiles - 1 && e.w < 0 && !(p.dbg & 256)) break;
      const uint32_t pb = pbuf_local + buf * (MT * kTileN * 4);
      if (p.dbg & 256) {  // measurement: no epilogue stores / piece reduction
        named_bar_sync(2, 64);
        if (lane == 0) mbar_arrive(&red_empty[buf]);
        continue;
      }
      // the tile's accumulators for rows u and u + 64, all MT tokens (MT = 64: loaded
      // per token chunk below — 2 x 64 accumulators do not fit next to the results)
      constexpr bool kCL = MT > 32;
      uint32_t acc[2][kCL ? 1 : MT];
      const bool whole = e.w < 0 || (p.dbg & 2048);
      const uint32_t* slots_f = nullptr;  // kCL: the finisher's slots, summed per chunk
      int npieces_f = 0;
      if (whole) {
        if constexpr (!kCL) {
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            acc[0][t] = ld_shared_u32(pb + (t * kTileN + u) * 4);
            acc[1][t] = ld_shared_u32(pb + (t * kTileN + u + 64) * 4);
          }
        }
      } else {
        // a piece of a split tile: partial to the piece's slot; the piece that
        // completes the tile's count sums the slots in piece order
        const int piece = e.z >> 16, npieces = e.z & 0xFFFF;
        uint32_t* slots = p.partials + static_cast<int64_t>(p.split_base[e.w]) * (MT * kTileN);
        uint32_t* mine = slots + static_cast<int64_t>(piece) * (MT * kTileN);
#pragma unroll 4
        for (int t = 0; t < MT; ++t) {
          mine[t * kTileN + u] = ld_shared_u32(pb + (t * kTileN + u) * 4);
          mine[t * kTileN + u + 64] = ld_shared_u32(pb + (t * kTileN + u + 64) * 4);
        }
        // Both warps' slot stores are ordered before thread 0's acq_rel add by the
        // barrier (release cumulativity), as in a serial split-K semaphore.
        named_bar_sync(2, 64);
        if (u == 0) {
          const unsigned prev = atom_add_acq_rel_gpu(&p.sync[kSyncWords + e.w], 1u);
          const bool fin = prev == static_cast<unsigned>(npieces - 1);
          if (fin) p.sync[kSyncWords + e.w] = 0u;  // re-armed for the next launch
          *flag_s = fin ? 1u : 0u;
        }
        named_bar_sync(2, 64);
        if (!*flag_s) {
          named_bar_sync(2, 64);  // flag_s and sa_s[it & 1] consumed
          if (lane == 0) mbar_arrive(&red_empty[buf]);
          continue;
        }
        slots_f = slots;
        npieces_f = npieces;
        // every slot's loads in flight together: one L2 round trip per piece
        if constexpr (!kCL) {
#pragma unroll
        for (int t = 0; t < MT; ++t) acc[0][t] = acc[1][t] = 0u;
        for (int k = 0; k < npieces; ++k) {
          const uint32_t* sl = slots + static_cast<int64_t>(k) * (MT * kTileN);
          uint32_t v[2][MT];
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            v[0][t] = __ldcg(sl + t * kTileN + u);
            v[1][t] = __ldcg(sl + t * kTileN + u + 64);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int t = 0; t < MT; ++t) {
              if (PATH == ISB_PATH_INTEGER_SCALE)
                acc[h][t] = static_cast<uint32_t>(static_cast<int32_t>(acc[h][t]) +
                                                  static_cast<int32_t>(v[h][t]));
              else
                acc[h][t] = __float_as_uint(__uint_as_float(acc[h][t]) + __uint_as_float(v[h][t]));
            }
        }
        }
      }
      // Eq. 2 / Eq. 1 in place: the outputs overwrite the partial buffer ([t][128]
      // rows of out_dtype), then leave as 16-byte vector stores along the token
      // rows — 8x fewer store instructions than one 2-byte store per output, which
      // stall for microseconds in a memory system saturated by the weight stream
      // (a bulk-copy store would queue behind the SM's pending weight loads).
      if constexpr (!kCL) named_bar_sync(2, 64);  // every source word read before any is overwritten
      const int ob = q.out_dtype == ISB_F32 || q.out_dtype == ISB_I32 ? 4 : 2;
      const int64_t n0 = static_cast<int64_t>(nt) * kTileN;
      const int nvalid = static_cast<int>(min(static_cast<int64_t>(kTileN), q.N - n0));
      const bool bulk = (q.N * ob) % 16 == 0 && (nvalid * ob) % 16 == 0;
      // All operands in registers first, then the arithmetic, then the smem
      // writes: the 32 outputs' conversion chains (I2F.F64, 2 DMUL, F2F, F2F) are
      // independent and overlap; interleaving them with volatile smem accesses
      // serialised every chain (~260 cycles per output).
      // Integer path at MT = 32: two 16-token chunks. All MT factors and results live
      // at once spilled (acc 64 + factors 64 + results 64 registers): M = 32 / 64 layer
      // 39.0 / 68.4 -> 37.0 / 62.9 us. The float path measured ~1 % faster unchunked.
      constexpr int kTC = (MT > 16 && PATH == ISB_PATH_INTEGER_SCALE) || kCL ? 16 : MT;
#pragma unroll
      for (int t0 = 0; t0 < MT; t0 += kTC) {
      uint32_t ac[2][kTC];  // this chunk's accumulators
      if constexpr (kCL) {
        if (whole) {
#pragma unroll
          for (int t = 0; t < kTC; ++t) {
            ac[0][t] = ld_shared_u32(pb + ((t0 + t) * kTileN + u) * 4);
            ac[1][t] = ld_shared_u32(pb + ((t0 + t) * kTileN + u + 64) * 4);
          }
          // the chunk's source words (its token rows, read by both warps) before any is
          // overwritten; later chunks' rows are untouched by this chunk's outputs
          named_bar_sync(2, 64);
        } else {
#pragma unroll
          for (int t = 0; t < kTC; ++t) ac[0][t] = ac[1][t] = 0u;
          for (int k = 0; k < npieces_f; ++k) {
            const uint32_t* sl = slots_f + static_cast<int64_t>(k) * (MT * kTileN) + t0 * kTileN;
            uint32_t v[2][kTC];
#pragma unroll
            for (int t = 0; t < kTC; ++t) {
              v[0][t] = __ldcg(sl + t * kTileN + u);
              v[1][t] = __ldcg(sl + t * kTileN + u + 64);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int t = 0; t < kTC; ++t) {
                if (PATH == ISB_PATH_INTEGER_SCALE)
                  ac[h][t] = static_cast<uint32_t>(static_cast<int32_t>(ac[h][t]) +
                                                   static_cast<int32_t>(v[h][t]));
                else
                  ac[h][t] = __float_as_uint(__uint_as_float(ac[h][t]) + __uint_as_float(v[h][t]));
              }
          }
        }
      } else {
#pragma unroll
        for (int t = 0; t < kTC; ++t) {
          ac[0][t] = acc[0][(t0 + t) % (kCL ? 1 : MT)];
          ac[1][t] = acc[1][(t0 + t) % (kCL ? 1 : MT)];
        }
      }
      double sav[kTC];  // integer path: s_a * 2^-e (exact), one DMUL per output left
#pragma unroll
      for (int t = 0; t < kTC; ++t)
        sav[t] = PATH == ISB_PATH_INTEGER_SCALE ? sa_t[t0 + t] * q.inv_amp : sa_t[t0 + t];
      uint32_t res[2][kTC];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < kTC; ++t) {
          const int32_t is = static_cast<int32_t>(ac[h][t]);
          const float fs = __uint_as_float(ac[h][t]);
          if ((PATH == ISB_PATH_INTEGER_SCALE && q.out_dtype == ISB_I32) || (p.dbg & 4096)) {
            res[h][t] = ac[h][t];
          } else {
            const float f = finish_eq<PATH>(is, fs, sav[t]);
            res[h][t] = ob == 4 ? __float_as_uint(f)
                        : q.out_dtype == ISB_BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(f))
                                                  : __half_as_ushort(__float2half_rn(f));
          }
        }
      if (bulk) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int t = 0; t < kTC; ++t) {
            const uint32_t dst = pb + (t0 + t) * (kTileN * 4) + (u + h * 64) * ob;
            if (ob == 4)
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(dst), "r"(res[h][t]) : "memory");
            else
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst),
                           "h"(static_cast<unsigned short>(res[h][t]))
                           : "memory");
          }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int t = 0; t < kTC; ++t) {
            const int64_t m = static_cast<int64_t>(mt) * MT + t0 + t;
            const int64_t n = n0 + u + h * 64;
            if (n < n0 + nvalid && m < q.M) {
              if (ob == 4)
                static_cast<uint32_t*>(q.out)[m * q.N + n] = res[h][t];
              else
                static_cast<unsigned short*>(q.out)[m * q.N + n] =
                    static_cast<unsigned short>(res[h][t]);
            }
          }
      }
      }
      if (bulk) {
        // 16-byte vector stores of the staged rows, consecutive threads along a row
        named_bar_sync(2, 64);
        const int cpr = nvalid * ob / 16;  // 16-byte chunks per token row
        int rows = q.M - mt * MT;
        rows = rows < MT ? rows : MT;
        for (int c = static_cast<int>(u); c < ((p.dbg & 8192) ? 0 : rows * cpr); c += 64) {
          const int t = c / cpr, cc = c - t * cpr;
          const uint4 v = ld_shared_v4(pb + t * (kTileN * 4) + cc * 16);
          const int64_t m = static_cast<int64_t>(mt) * MT + t;
          *reinterpret_cast<uint4*>(static_cast<uint8_t*>(q.out) + (m * q.N + n0) * ob + cc * 16) = v;
        }
      }
      if (it == ntiles - 1 && u == 0 && p.trace) p.trace[11 * 512 + blockIdx.x] = globaltimer_();
      named_bar_sync(2, 64);  // outputs out of the buffer; sa_s[it & 1] and flag_s consumed
      if (lane == 0) mbar_arrive(&red_empty[buf]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && p.trace) {
    p.trace[3 * 512 + blockIdx.x] = globaltimer_();
    p.trace[14 * 512 + blockIdx.x] = clock64_();
  }
  if (ntiles > 0 && list[ntiles - 1].w < 0 && !(p.dbg & 256)) {
    // The last (whole) tile: its partial is in buffer (ntiles-1) % kPbufs (pb_full
    // and the token scales were waited by the reduction warps before the barrier).
    const int it = ntiles - 1;
    const int4 e = list[it];
    const GProb& q = probs_s[e.x >> 24];
    const int nt = (e.x & 0xFFFFFF) / q.m_tiles, mt = (e.x & 0xFFFFFF) % q.m_tiles;
    const uint32_t pb = smem_u32(pbuf) + (it % Cf::kPbufs) * (MT * kTileN * 4);
    const double* sa_t = sa_s + (it & 1) * MT;
    const int64_t n0 = static_cast<int64_t>(nt) * kTileN;
    constexpr int kPer = MT * kTileN / Cf::kThreads;
    uint32_t v[kPer];
    double sc[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = static_cast<int>(threadIdx.x) + k * Cf::kThreads;  // t * 128 + r
      v[k] = ld_shared_u32(pb + idx * 4);
      sc[k] = sa_t[idx / kTileN];
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = static_cast<int>(threadIdx.x) + k * Cf::kThreads;
      const int t = idx / kTileN, r = idx % kTileN;
      const int64_t m = static_cast<int64_t>(mt) * MT + t, n = n0 + r;
      if (m < q.M && n < q.N) {
        if (PATH == ISB_PATH_INTEGER_SCALE && q.out_dtype == ISB_I32) {
          static_cast<int32_t*>(q.out)[m * q.N + n] = static_cast<int32_t>(v[k]);
        } else {
          const double s = PATH == ISB_PATH_INTEGER_SCALE ? sc[k] * q.inv_amp : sc[k];
          store_out(q.out, q.out_dtype, m * q.N + n,
                    finish_eq<PATH>(static_cast<int32_t>(v[k]), __uint_as_float(v[k]), s));
        }
      }
    }
  }
  if (threadIdx.x == 32 && p.trace) p.trace[8 * 512 + blockIdx.x] = globaltimer_();
  if (threadIdx.x == 0 && p.trace) {
    p.trace[6 * 512 + blockIdx.x] = globaltimer_();
    p.trace[15 * 512 + blockIdx.x] = clock64_();
  }
}

template <int MT, int PATH>
void prepare_group_kernel() {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemm_w4a8_group<MT, PATH>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Cfg<MT, false>::kSmemBytes + kTableBytes),
               "cudaFuncSetAttribute(smem)");
  });
}

template <int MT, int PATH>
int group_blocks_per_sm() {
  prepare_group_kernel<MT, PATH>();
  int n = 0;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gemm_w4a8_group<MT, PATH>,
                                                           Cfg<MT, false>::kThreads,
                                                           Cfg<MT, false>::kSmemBytes + kTableBytes),
             "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  return n;
}

int group_capacity(int mt, int path, int num_sms) {
  static std::mutex mu;
  static int cache[3][2] = {};
  std::lock_guard<std::mutex> lk(mu);
  int& slot = cache[mt == 16 ? 0 : mt == 32 ? 1 : 2][path == ISB_PATH_INTEGER_SCALE ? 1 : 0];
  if (!slot) {
    int n = 0;
    if (mt == 16)
      n = path == ISB_PATH_INTEGER_SCALE ? group_blocks_per_sm<16, ISB_PATH_INTEGER_SCALE>()
                                         : group_blocks_per_sm<16, ISB_PATH_FLOAT_SCALE>();
    else if (mt == 32)
      n = path == ISB_PATH_INTEGER_SCALE ? group_blocks_per_sm<32, ISB_PATH_INTEGER_SCALE>()
                                         : group_blocks_per_sm<32, ISB_PATH_FLOAT_SCALE>();
    else
      n = path == ISB_PATH_INTEGER_SCALE ? group_blocks_per_sm<64, ISB_PATH_INTEGER_SCALE>()
                                         : group_blocks_per_sm<64, ISB_PATH_FLOAT_SCALE>();
    slot = n > 0 ? n : -1;
  }
  return slot > 0 ? slot * num_sms : 0;
}

template <int MT, int PATH>
void launch_group_mt(const GMaps& maps, const GParams& prm, int grid, cudaStream_t s) {
  prepare_group_kernel<MT, PATH>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg<MT, false>::kThreads);
  cfg.dynamicSmemBytes = Cfg<MT, false>::kSmemBytes + kTableBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_w4a8_group<MT, PATH>, maps, prm),
             "gemm_w4a8_group launch");
  count_launch();
}

}  // namespace

// ---------------------------------------------------------------------------- plan (host)
struct GroupPlan {
  GParams prm{};
  GMaps maps{};
  int mt = 16, path = ISB_PATH_INTEGER_SCALE, grid = 0, dev = 0, nsplit = 0, out_dtype = 0;
  double makespan = 0.0;      // per-CTA budget in 128-K blocks (+ per-piece overhead)
  int* sched_dev = nullptr;   // schedule + lengths + split bases
  unsigned* sync_dev = nullptr;
  uint32_t* partials = nullptr;
  void* owned = nullptr;      // plan-owned codes / scales when the caller passes none
  // Prefill route (every problem M >= kSpMinM, integer scale, k_g <= 16): K1 per problem
  // (when float activations are given) + one grouped CTA-pair fold launch (gemm_sp.cu).
  SpGroupPlan* sp = nullptr;
  // Sequential route (some problem has M > kGroupMaxM but the pair kernel does not apply:
  // float scale, or k_g > 16): K1 per problem + the single-GEMM prefill kernels in turn.
  bool seq = false;
  void* seq_ws = nullptr;
  int64_t seq_ws_bytes = 0;
  isb_group_problem sp_probs[8] = {};  // resolved codes / scales pointers
  int sp_n = 0;
  int sp_x_dtype[8] = {};
  ~GroupPlan() {
    if (sp) sp_group_destroy(sp);
    if (seq_ws) cudaFree(seq_ws);
    if (sched_dev) cudaFree(sched_dev);
    if (sync_dev) cudaFree(sync_dev);
    if (partials) cudaFree(partials);
    if (owned) cudaFree(owned);
  }
};

namespace {

constexpr int64_t kGroupMaxM = 64;  // decode grouped kernel beyond this: prefill routes

int pick_group_mt(int64_t max_m) {
  // ISB_GROUP_MT=32 / 64 (A/B): the tile for 33 <= M <= 64 (default 64: one weight
  // expansion per 64 tokens instead of one per 32)
  static const int mt_big = [] {
    const char* e = std::getenv("ISB_GROUP_MT");
    return e && std::atoi(e) == 32 ? 32 : 64;
  }();
  if (max_m <= 16) return 16;
  if (max_m <= 32) return 32;
  return max_m <= 64 ? mt_big : 32;  // beyond 64: 32-token tiles (prefill M routes elsewhere)
}

// McNaughton wrap-around over `ncta` equal budgets. Tiles (cost = their 128-K
// blocks + a per-piece hand-off overhead) are poured in order; a tile crossing a
// budget boundary continues on the next CTA. Pieces shorter than one step are
// avoided by moving the boundary. Returns false if the budget is too small.
struct Piece { int entry, g0, g1, tile_id; };
bool wrap_schedule(const std::vector<std::pair<int, int>>& tiles, int ncta, int budget,
                   int overhead, int min_piece, std::vector<std::vector<Piece>>& lists) {
  lists.assign(ncta, {});
  int c = 0, room = budget;
  for (int i = 0; i < static_cast<int>(tiles.size()); ++i) {
    const int entry = tiles[i].first, g = tiles[i].second;
    int g0 = 0;
    while (g0 < g) {
      const int rem = g - g0;
      int take = std::min(rem, room - overhead);
      if (take < rem && take < min_piece) {  // too small a piece: next CTA
        if (++c == ncta) return false;
        room = budget;
        continue;
      }
      lists[c].push_back({entry, g0, g0 + take, i});
      room -= take + overhead;
      g0 += take;
      if (room <= overhead && !(i + 1 == static_cast<int>(tiles.size()) && g0 == g)) {
        if (++c == ncta) return false;
        room = budget;
      }
    }
  }
  return true;
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
    if (w.groups >= (1 << 15)) fail(ISB_PARAM, "grouped GEMM: K too large");
    if (path == ISB_PATH_INTEGER_SCALE && !w.has_int_scales)
      fail(ISB_PARAM, "integer-scale path needs an IntegerScaleSet");
    if (path == ISB_PATH_INTEGER_SCALE &&
        w.static_bound > std::numeric_limits<int32_t>::max())
      fail(ISB_OVERFLOW, "static overflow bound " + std::to_string(w.static_bound) +
                             " exceeds int32 (problem " + std::to_string(i) +
                             "): the tensor-core integer-scale GEMM cannot be exact");
    if (q.m < 0 || q.m > (1 << 20)) fail(ISB_PARAM, "grouped GEMM: bad M");
    if (q.m > 0 && !q.out) fail(ISB_PARAM, "grouped GEMM: null output");
    max_m = std::max(max_m, q.m);
    if (q.m == 0) continue;  // no work (an expert without routed tokens)
    const int qz = q.x != nullptr ? 1 : 0;
    if (quantize >= 0 && qz != quantize)
      fail(ISB_PARAM, "grouped GEMM: either every problem passes float activations or none");
    quantize = qz;
    if (qz) {
      if (q.x_dtype != ISB_F32 && q.x_dtype != ISB_BF16)
        fail(ISB_PARAM, "grouped GEMM: activations must be float32 or bf16");
      if (!q.xq) own_bytes += (q.m * w.k + 255) / 256 * 256;
      if (!q.sa) own_bytes += (q.m * 8 + 255) / 256 * 256;
    } else if (!q.xq || !q.sa) {
      fail(ISB_PARAM, "grouped GEMM: null activation pointer");
    }
  }
  if (quantize < 0) quantize = 0;
  bool prefill = path == ISB_PATH_INTEGER_SCALE;
  for (int i = 0; i < nprob && prefill; ++i)
    prefill = probs[i].m >= kSpMinM && fold_eligible(probs[i].m, *probs[i].w, path);
  auto* pl = new GroupPlan();
  try {
    cuda_check(cudaGetDevice(&pl->dev), "cudaGetDevice");
    pl->path = path;
    const bool seq = !prefill && max_m > kGroupMaxM;
    if (prefill || seq) {
      if (own_bytes) cuda_check(cudaMalloc(&pl->owned, own_bytes), "cudaMalloc(group workspace)");
      uint8_t* own = static_cast<uint8_t*>(pl->owned);
      pl->prm.quantize = quantize;
      for (int i = 0; i < nprob; ++i) {
        isb_group_problem q = probs[i];
        if (quantize) {
          if (!q.xq) { q.xq = reinterpret_cast<int8_t*>(own); own += (q.m * q.w->k + 255) / 256 * 256; }
          if (!q.sa) { q.sa = reinterpret_cast<double*>(own); own += (q.m * 8 + 255) / 256 * 256; }
          pl->sp_x_dtype[i] = q.x_dtype;
        }
        pl->sp_probs[pl->sp_n++] = q;
      }
      cuda_check(cudaMalloc(&pl->sync_dev, kSyncWords * sizeof(unsigned)), "cudaMalloc(group sync)");
      cuda_check(cudaMemset(pl->sync_dev, 0, kSyncWords * sizeof(unsigned)), "cudaMemset(group sync)");
      if (seq) {
        pl->seq = true;
        pl->out_dtype = out_dtype;
        for (int i = 0; i < nprob; ++i)
          if (probs[i].m > 0)
            pl->seq_ws_bytes = std::max(pl->seq_ws_bytes, gemm_workspace_size(probs[i].m, *probs[i].w));
        pl->seq_ws_bytes = std::max<int64_t>(pl->seq_ws_bytes, 256);
        cuda_check(cudaMalloc(&pl->seq_ws, pl->seq_ws_bytes), "cudaMalloc(group gemm workspace)");
        cuda_check(cudaMemset(pl->seq_ws, 0, pl->seq_ws_bytes), "cudaMemset(group gemm workspace)");
        pl->grid = 1;
        pl->mt = 0;
        return pl;
      }
      pl->sp = sp_group_create(pl->sp_probs, nprob, out_dtype, num_sms);
      pl->grid = 2 * (num_sms / 2);
      pl->mt = kSpTileTokens;
      pl->makespan = 1.0 / std::max(1e-9, sp_group_balance(pl->sp));
      return pl;
    }
    pl->mt = pick_group_mt(max_m);
    const int mt = pl->mt;
    const int S = mt == 64 ? Cfg<64, false>::S : Cfg<32, false>::S;
    if (own_bytes) cuda_check(cudaMalloc(&pl->owned, own_bytes), "cudaMalloc(group workspace)");
    uint8_t* own = static_cast<uint8_t*>(pl->owned);
    GParams& P = pl->prm;
    P.nprob = nprob;
    P.quantize = quantize;
    P.dbg = g_dbg;
    P.trace = g_trace;
    std::vector<std::pair<int, int>> tiles;  // (entry, groups) in problem order
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
      const int64_t nt = static_cast<int64_t>(w.n_tiles) * g.m_tiles;
      if (static_cast<int64_t>(tiles.size()) + nt >= (int64_t{1} << 24))
        fail(ISB_PARAM, "grouped GEMM: too many tiles");
      for (int64_t t = 0; t < nt; ++t) tiles.push_back({(i << 24) | static_cast<int>(t), g.G});
      if (q.m > 0) pl->maps.m[i] = make_x_map(g.xq, q.m, w.k, mt);
      P.qoff[i + 1] = P.qoff[i] + (quantize ? g.M : 0);
    }
    P.qtasks = P.qoff[nprob];
    // Budgets in 128-K blocks: every CTA gets total / ncta (+ a hand-off overhead
    // of half a step per piece); ISB_GROUP_CTAS overrides the CTA count (A/B).
    static const int force_ctas = [] {
      const char* e = std::getenv("ISB_GROUP_CTAS");
      return e ? std::atoi(e) : 0;
    }();
    int ncta = group_capacity(mt, path, num_sms);
    if (ncta <= 0) fail(ISB_CUDA, "grouped GEMM: kernel does not fit the device");
    if (force_ctas > 0) ncta = std::min(ncta, force_ctas);
    // Longest tiles first: a tile about as long as a budget (e.g. LLaMA down_proj,
    // K = 11008) then lands whole on its own CTA instead of being cut at every
    // budget boundary, so lists rarely end with a split piece (whose global
    // hand-off would trail the CTA's last step).
    std::stable_sort(tiles.begin(), tiles.end(),
                     [](const std::pair<int, int>& a, const std::pair<int, int>& b) {
                       return a.second > b.second;
                     });
    int64_t total = 0;
    for (auto& t : tiles) total += t.second;
    const int overhead = S / 2;
    std::vector<std::vector<Piece>> lists;
    if (!tiles.empty()) {
      ncta = static_cast<int>(std::min<int64_t>(ncta, total / S + 1));  // >= ~one step each
      int budget = static_cast<int>((total + overhead * static_cast<int64_t>(tiles.size()) +
                                     ncta - 1) / ncta) + overhead;
      while (!wrap_schedule(tiles, ncta, budget, overhead, S, lists)) ++budget;
      pl->makespan = budget / static_cast<double>(S);
    } else {
      ncta = 0;
    }
    // split tiles: ids, partial slots, counters
    std::vector<int> pieces_of(tiles.size(), 0);
    for (auto& l : lists)
      for (auto& pc : l) ++pieces_of[pc.tile_id];
    std::vector<int> split_id(tiles.size(), -1), split_base;
    int slots = 0;
    for (size_t i = 0; i < tiles.size(); ++i)
      if (pieces_of[i] > 1) {
        if (pieces_of[i] >= (1 << 15)) fail(ISB_PARAM, "grouped GEMM: tile split too finely");
        split_id[i] = static_cast<int>(split_base.size());
        split_base.push_back(slots);
        slots += pieces_of[i];
      }
    pl->nsplit = static_cast<int>(split_base.size());
    // Pieces of split tiles first in every CTA's list: their global hand-off
    // (slot stores, counter, the finisher's slot reads) then overlaps the whole
    // tiles' weight stream instead of trailing the CTA's last step.
    for (auto& l : lists)
      std::stable_partition(l.begin(), l.end(),
                            [&](const Piece& pc) { return pieces_of[pc.tile_id] > 1; });
    std::vector<int> seen(tiles.size(), 0);
    size_t stride = 1;
    for (auto& l : lists) stride = std::max(stride, l.size());
    const size_t n_sched = static_cast<size_t>(ncta) * stride;
    std::vector<int4> sched(n_sched, int4{0, 0, 0, -1});
    std::vector<int> lens(ncta, 0);
    for (int c = 0; c < ncta; ++c) {
      lens[c] = static_cast<int>(lists[c].size());
      for (size_t k = 0; k < lists[c].size(); ++k) {
        const Piece& pc = lists[c][k];
        const int piece = seen[pc.tile_id]++;
        sched[c * stride + k] = int4{pc.entry, (pc.g0 << 16) | pc.g1,
                                     (piece << 16) | pieces_of[pc.tile_id], split_id[pc.tile_id]};
      }
    }
    // one device buffer: schedule (int4), lengths, split bases
    const size_t bytes = n_sched * sizeof(int4) + (lens.size() + split_base.size() + 1) * 4;
    cuda_check(cudaMalloc(&pl->sched_dev, bytes), "cudaMalloc(schedule)");
    auto* base = reinterpret_cast<uint8_t*>(pl->sched_dev);
    cuda_check(cudaMemcpy(base, sched.data(), n_sched * sizeof(int4), cudaMemcpyHostToDevice),
               "copy schedule");
    int* lens_d = reinterpret_cast<int*>(base + n_sched * sizeof(int4));
    if (!lens.empty())
      cuda_check(cudaMemcpy(lens_d, lens.data(), lens.size() * 4, cudaMemcpyHostToDevice),
                 "copy lengths");
    int* split_d = lens_d + lens.size();
    if (!split_base.empty())
      cuda_check(cudaMemcpy(split_d, split_base.data(), split_base.size() * 4,
                            cudaMemcpyHostToDevice),
                 "copy split bases");
    P.NC = ncta;
    P.sched = reinterpret_cast<const int4*>(base);
    P.sched_stride = static_cast<int>(stride);
    P.sched_len = lens_d;
    P.split_base = split_d;
    if (slots)
      cuda_check(cudaMalloc(&pl->partials, static_cast<size_t>(slots) * mt * kTileN * 4),
                 "cudaMalloc(partials)");
    P.partials = pl->partials;
    const size_t sync_words = kSyncWords + split_base.size();
    cuda_check(cudaMalloc(&pl->sync_dev, sync_words * sizeof(unsigned)), "cudaMalloc(sync)");
    cuda_check(cudaMemset(pl->sync_dev, 0, sync_words * sizeof(unsigned)), "cudaMemset(sync)");
    P.sync = pl->sync_dev;
    pl->grid = ncta;
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
  if (pl->seq) {  // K1 per problem, then the single-GEMM kernels in turn
    for (int i = 0; i < pl->sp_n; ++i) {
      const isb_group_problem& q = pl->sp_probs[i];
      if (q.m == 0) continue;
      if (pl->prm.quantize)
        launch_quantize_per_token(q.x, pl->sp_x_dtype[i], q.m, q.w->k, q.xq, q.sa,
                                  reinterpret_cast<int*>(pl->sync_dev + kSyncBad), s);
      gemm_dispatch(pl->path, q.xq, q.sa, q.m, *q.w, q.out, pl->out_dtype, pl->seq_ws,
                    pl->seq_ws_bytes, s);
    }
    return;
  }
  if (pl->sp) {
    if (pl->prm.quantize)
      for (int i = 0; i < pl->sp_n; ++i) {
        const isb_group_problem& q = pl->sp_probs[i];
        launch_quantize_per_token(q.x, pl->sp_x_dtype[i], q.m, q.w->k, q.xq, q.sa,
                                  reinterpret_cast<int*>(pl->sync_dev + kSyncBad), s);
      }
    sp_group_run(pl->sp, s);
    return;
  }
  if (pl->mt == 16) {
    if (pl->path == ISB_PATH_INTEGER_SCALE)
      launch_group_mt<16, ISB_PATH_INTEGER_SCALE>(pl->maps, pl->prm, pl->grid, s);
    else
      launch_group_mt<16, ISB_PATH_FLOAT_SCALE>(pl->maps, pl->prm, pl->grid, s);
  } else if (pl->mt == 32) {
    if (pl->path == ISB_PATH_INTEGER_SCALE)
      launch_group_mt<32, ISB_PATH_INTEGER_SCALE>(pl->maps, pl->prm, pl->grid, s);
    else
      launch_group_mt<32, ISB_PATH_FLOAT_SCALE>(pl->maps, pl->prm, pl->grid, s);
  } else {
    if (pl->path == ISB_PATH_INTEGER_SCALE)
      launch_group_mt<64, ISB_PATH_INTEGER_SCALE>(pl->maps, pl->prm, pl->grid, s);
    else
      launch_group_mt<64, ISB_PATH_FLOAT_SCALE>(pl->maps, pl->prm, pl->grid, s);
  }
}

void group_plan_info(const GroupPlan* pl, isb_group_info_t* info) {
  info->grid = pl->grid;
  info->cluster = 1;
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
