// Dense fp16 / bf16 baseline GEMM on tcgen05 (kind::f16, fp32 accumulate), no cuBLAS.
//
// North star (BASELINE.json): "an fp16 cuBLAS-free dense baseline kernel and the
// float-scale W4A8 variant are reported for the paper's speedup claims" — the
// paper's FP16 comparison (Table 5 / Fig. 1). out[M][N] = x[M][K] * w[N][K]^T
// (nn.Linear layout: w is [out][in], K contiguous).
//
// Same swap-AB shape as K3: output channels are UMMA M (128 per tile), tokens are
// UMMA N (MT = 16..256). Both operands arrive by TMA (SWIZZLE_128B, 64-element K
// blocks) and feed tcgen05.mma directly from shared memory (SS form).
//   warp 0   producer : TMA of the 128 x 64 weight block + MT x 64 activation block
//   warp 1   MMA      : 4 x kind::f16 (K = 16) per block into a TMEM accumulator
//                       (double-buffered: the epilogue of tile t overlaps tile t+1)
//   warp 2   TMEM allocator
//   warps 4-7 epilogue: tcgen05.ld -> fp16/bf16/fp32 stores; with split-K (decode)
//                       each rank publishes its fp32 partial in shared memory and
//                       finalises MT/C tokens over all ranks' partials (DSMEM, fixed
//                       rank order -> deterministic).
// Persistent: clusters of C CTAs (split-K ways) own tiles cid, cid + #clusters, ...
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

constexpr int kDK = 64;  // K elements per block (128 B rows: one SWIZZLE_128B atom wide)

template <int MT>
struct DCfg {
  static constexpr int kABytes = 128 * kDK * 2;
  static constexpr int kBBytes = MT * kDK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * MT <= 32 ? 32 : 2 * MT <= 64 ? 64 : 2 * MT <= 128 ? 128
                                   : 2 * MT <= 256 ? 256 : 512;
  static constexpr int kPbufBytes = MT <= 64 ? MT * 128 * 4 : 0;  // split-K partial (fp32)
  static constexpr int kFixed = 1024 + kPbufBytes + 1024;
  static constexpr int kStagesRaw = (227 * 1024 - kFixed) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmemBytes = kFixed + kStages * kStageBytes;
  static constexpr int kThreads = 256;
  static_assert(kStages >= 2, "smem");
};

struct DParams {
  void* out;
  int M, N, KB, m_tiles, tiles, out_dtype, C, NC;
  uint32_t idesc;
};

ISB_DEVICE void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void store_d(void* out, int dtype, int64_t idx, float f) {
  if (dtype == ISB_F32)
    static_cast<float*>(out)[idx] = f;
  else if (dtype == ISB_BF16)
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
  else
    static_cast<__half*>(out)[idx] = __float2half_rn(f);
}

// I8 = true: the same pipeline on kind::i8 (int8 x int8 -> int32, 128-element K
// blocks) — the upper bound of an SS-form int8 kernel (debug / measurement only).
template <int MT, bool I8 = false>
__global__ void __launch_bounds__(DCfg<MT>::kThreads, 1)
    gemm_f16_tc(const __grid_constant__ CUtensorMap w_map, const __grid_constant__ CUtensorMap x_map,
                const DParams p) {
  using Cf = DCfg<MT>;
  constexpr int kStages = Cf::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;                                   // [stage][128 x 64 fp16]
  uint8_t* smem_b = smem_a + kStages * Cf::kABytes;         // [stage][MT x 64 fp16]
  float* pbuf = reinterpret_cast<float*>(smem_b + kStages * Cf::kBBytes);  // [MT][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(pbuf) + Cf::kPbufBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* d_full = empty + kStages;   // [2]
  uint64_t* d_empty = d_full + 2;       // [2]
  uint64_t* red_full = d_empty + 2;     // all ranks' partials published (cluster)
  uint64_t* red_empty = red_full + 1;   // all ranks done reading ours (cluster)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_empty + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int cid = blockIdx.x / p.C, rank = blockIdx.x % p.C;
  const int kb0 = rank * p.KB / p.C, kb1 = (rank + 1) * p.KB / p.C;
  const int ntiles = cid < p.tiles ? (p.tiles - cid + p.NC - 1) / p.NC : 0;

  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&w_map);
    prefetch_tensormap(&x_map);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4);
    }
    mbar_init(red_full, 4 * p.C);
    mbar_init(red_empty, 4 * p.C);
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
      pdl_wait();
      int j = 0;
      for (int it = 0; it < ntiles; ++it) {
        const int tile = cid + it * p.NC;
        const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
        for (int kb = kb0; kb < kb1; ++kb, ++j) {
          const int s = j % kStages;
          mbar_wait(&empty[s], ((j / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], Cf::kStageBytes);
          tma_load_2d(smem_a + s * Cf::kABytes, &w_map, &full[s], kb * kDK, nt * 128);
          tma_load_2d(smem_b + s * Cf::kBBytes, &x_map, &full[s], kb * kDK, mt * MT);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      int j = 0;
      for (int it = 0; it < ntiles; ++it) {
        const int buf = it & 1;
        mbar_wait(&d_empty[buf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * MT;
        for (int kb = kb0; kb < kb1; ++kb, ++j) {
          const int s = j % kStages;
          mbar_wait(&full[s], (j / kStages) & 1);
          tc_fence_after();
          const uint64_t adesc = make_sw128_kmajor_desc(smem_u32(smem_a + s * Cf::kABytes));
          const uint64_t bdesc = make_sw128_kmajor_desc(smem_u32(smem_b + s * Cf::kBBytes));
#pragma unroll
          for (int c = 0; c < 4; ++c)  // K = 16 per MMA = 32 B = 2 descriptor units
            if constexpr (I8)
              mma_i8_ss(d_tmem, adesc + static_cast<uint64_t>(c * 2),
                        bdesc + static_cast<uint64_t>(c * 2), p.idesc, (kb > kb0 || c > 0) ? 1u : 0u);
            else
              mma_f16_ss(d_tmem, adesc + static_cast<uint64_t>(c * 2),
                         bdesc + static_cast<uint64_t>(c * 2), p.idesc, (kb > kb0 || c > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&d_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const uint32_t ew = warp - 4;
    const uint32_t r = ew * 32 + lane;  // TMEM lane == output channel within the tile
    const uint32_t lane_base = (ew * 32) << 16;
    pdl_wait();  // the output may be read by the preceding grid
    for (int it = 0; it < ntiles; ++it) {
      const int tile = cid + it * p.NC;
      const int nt = tile / p.m_tiles, mt = tile % p.m_tiles;
      const int buf = it & 1;
      const int64_t n = static_cast<int64_t>(nt) * 128 + r;
      mbar_wait(&d_full[buf], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + lane_base + buf * MT;
      if (p.C == 1) {
#pragma unroll 1
        for (int c = 0; c < MT; c += 16) {
          uint32_t v[16];
          tmem_ld_x16_(taddr + c, v);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int64_t m = static_cast<int64_t>(mt) * MT + c + t;
            const float f = I8 ? static_cast<float>(static_cast<int32_t>(v[t])) : __uint_as_float(v[t]);
            if (m < p.M && n < p.N) store_d(p.out, p.out_dtype, m * p.N + n, f);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[buf]);
      } else {
        if constexpr (Cf::kPbufBytes > 0) {
        // split-K: publish the fp32 partial, finalise tokens [rank*MT/C, (rank+1)*MT/C)
        if (it > 0) mbar_wait_cluster(red_empty, (it - 1) & 1);
#pragma unroll 1
        for (int c = 0; c < MT; c += 16) {
          uint32_t v[16];
          tmem_ld_x16_(taddr + c, v);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 16; ++t)
            pbuf[(c + t) * 128 + r] = I8 ? static_cast<float>(static_cast<int32_t>(v[t])) : __uint_as_float(v[t]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[buf]);
        if (lane < static_cast<uint32_t>(p.C)) mbar_arrive_remote_release(mapa_shared(smem_u32(red_full), lane));
        mbar_wait_cluster(red_full, it & 1);
        const int lo = rank * MT / p.C, hi = (rank + 1) * MT / p.C;
        for (int t = lo; t < hi; ++t) {
          float acc = 0.0f;
          const uint32_t off = smem_u32(pbuf + t * 128 + r);
          for (int q = 0; q < p.C; ++q) acc += __uint_as_float(ld_shared_cluster_u32(mapa_shared(off, q)));
          const int64_t m = static_cast<int64_t>(mt) * MT + t;
          if (m < p.M && n < p.N) store_d(p.out, p.out_dtype, m * p.N + n, acc);
        }
        __syncwarp();
        if (lane < static_cast<uint32_t>(p.C)) mbar_arrive_remote(mapa_shared(smem_u32(red_empty), lane));
        }
      }
    }
    // peers may still read this CTA's partial: wait until every rank is done with it
    if (p.C > 1 && ntiles > 0) mbar_wait_cluster(red_empty, (ntiles - 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, Cf::kTmemCols);
}

CUtensorMap make_map_f16(const void* base, int64_t rows, int64_t k, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  if (!fn) fail(ISB_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kDK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult rc = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) fail(ISB_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(rc) + ")");
  return map;
}

template <int MT, bool I8 = false>
void prepare_dense() {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemm_f16_tc<MT, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    DCfg<MT>::kSmemBytes),
               "cudaFuncSetAttribute(smem)");
    cuda_check(cudaFuncSetAttribute(gemm_f16_tc<MT, I8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
               "cudaFuncSetAttribute(cluster)");
  });
}

template <int MT>
int dense_capacity(int C) {
  static std::mutex mu;
  static int cache[9] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (!cache[C]) {
    prepare_dense<MT>();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C * 64);
    cfg.blockDim = dim3(DCfg<MT>::kThreads);
    cfg.dynamicSmemBytes = DCfg<MT>::kSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_f16_tc<MT>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cache[C] = n > 0 ? n : -1;
  }
  return cache[C];
}

template <int MT, bool I8 = false>
void launch_dense_mt(const void* x, const void* w, int64_t m, int64_t n, int64_t k, void* out,
                     int out_dtype, bool bf16, int sms, cudaStream_t s) {
  DParams p{};
  p.out = out;
  p.M = static_cast<int>(m);
  p.N = static_cast<int>(n);
  p.KB = static_cast<int>(k / (I8 ? 2 * kDK : kDK));
  p.m_tiles = static_cast<int>((m + MT - 1) / MT);
  const int n_tiles = static_cast<int>((n + 127) / 128);
  p.tiles = n_tiles * p.m_tiles;
  p.out_dtype = out_dtype;
  const uint32_t fmt = bf16 ? 1u : 0u;
  p.idesc = I8 ? make_idesc_i8(128, MT)
               : (1u << 4) | (fmt << 7) | (fmt << 10) | ((static_cast<uint32_t>(MT) >> 3) << 17) |
                     ((128u >> 4) << 24);
  // split-K width: same cost model as K3 (rounds * (k-blocks per CTA + per-tile cost))
  static const int force_c = [] {
    const char* e = std::getenv("ISB_DENSE_C");
    return e ? std::atoi(e) : 0;
  }();
  double best = 1e30;
  p.C = 1;
  int nc_best = 1;
  for (int C : {1, 2, 4, 8}) {
    if (C > 1 && DCfg<MT>::kPbufBytes == 0) break;
    if (C > p.KB) break;
    if (force_c && C != force_c) continue;
    int cap = dense_capacity<MT>(C);
    if (cap <= 0) continue;
    cap = std::min(cap, sms / C);
    const int nc = std::min(cap, p.tiles);
    const int rounds = (p.tiles + nc - 1) / nc;
    const double steps = std::ceil(static_cast<double>(p.KB) / C);
    const double cost = rounds * (steps + 2.0 + (C > 1 ? 1.0 : 0.0));
    if (cost < best - 1e-9) {
      best = cost;
      p.C = C;
      nc_best = nc;
    }
  }
  p.NC = nc_best;
  // int8: same 128-byte rows, viewed as k/2 16-bit elements per row
  const CUtensorMap wmap = make_map_f16(w, n, I8 ? k / 2 : k, 128);
  const CUtensorMap xmap = make_map_f16(x, m, I8 ? k / 2 : k, MT);
  prepare_dense<MT, I8>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nc_best * p.C);
  cfg.blockDim = dim3(DCfg<MT>::kThreads);
  cfg.dynamicSmemBytes = DCfg<MT>::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = p.C;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cuda_check(cudaLaunchKernelEx(&cfg, gemm_f16_tc<MT, I8>, wmap, xmap, p), "gemm_f16_tc launch");
  count_launch();
}

}  // namespace

void launch_gemm_dense(const void* x, const void* w, int64_t m, int64_t n, int64_t k, void* out,
                       int out_dtype, bool bf16, int sms, cudaStream_t s) {
  if (m <= 16) launch_dense_mt<16>(x, w, m, n, k, out, out_dtype, bf16, sms, s);
  else if (m <= 32) launch_dense_mt<32>(x, w, m, n, k, out, out_dtype, bf16, sms, s);
  else if (m <= 64) launch_dense_mt<64>(x, w, m, n, k, out, out_dtype, bf16, sms, s);
  else if (m <= 128) launch_dense_mt<128>(x, w, m, n, k, out, out_dtype, bf16, sms, s);
  else launch_dense_mt<256>(x, w, m, n, k, out, out_dtype, bf16, sms, s);
}

void launch_gemm_dense_i8(const void* x, const void* w, int64_t m, int64_t n, int64_t k, void* out,
                          int sms, cudaStream_t s) {
  if (m <= 16) launch_dense_mt<16, true>(x, w, m, n, k, out, ISB_F32, false, sms, s);
  else if (m <= 128) launch_dense_mt<128, true>(x, w, m, n, k, out, ISB_F32, false, sms, s);
  else launch_dense_mt<256, true>(x, w, m, n, k, out, ISB_F32, false, sms, s);
}

}  // namespace isb
