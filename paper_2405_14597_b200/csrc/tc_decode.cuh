// Decode-family tile configuration and epilogue pieces shared by the single-GEMM
// kernel (gemm_tc.cu) and the grouped layer kernel (gemm_group.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

// XQ: per-token activation quantization fused into the GEMM (config C3). The CTA
// quantizes the float activation slice of its K range (its cluster rank's
// groups) straight into a resident SWIZZLE_128B smem region; the full-row absmax
// the per-token scale needs (quantize.cpp:120-125) is combined across the
// cluster's ranks over DSMEM (the ranks of a cluster cover all of K).
template <int MT, bool XQ = false>
struct Cfg {
  static constexpr int S = MT <= 32 ? 4 : (MT == 64 ? 2 : 1);    // 128-K blocks per step
  static constexpr int kXformWG = MT >= 128 ? 1 : 2;             // transform warpgroups
  static constexpr int kEpiWG = MT >= 128 ? 4 : 1;               // epilogue warpgroups
  static constexpr int kCols = MT / kEpiWG;                      // tokens per epilogue thread
  static constexpr int kThreads = 128 + 128 * kXformWG + 128 * kEpiWG;
  static constexpr int kNA = MT <= 32 ? 2 : (MT == 64 ? 3 : 4);  // TMEM A stages (S*32 cols)
  static constexpr int kND = MT <= 16 ? 3 : (MT <= 64 ? 2 : 3);  // TMEM D slots (S*MT cols)
  static constexpr int kACols = S * 32;
  static constexpr int kDCols = S * MT;
  static constexpr int kTmemUsed = kNA * kACols + kND * kDCols;
  static constexpr int kTmemCols = kTmemUsed <= 32 ? 32 : kTmemUsed <= 64 ? 64
                                   : kTmemUsed <= 128 ? 128 : kTmemUsed <= 256 ? 256 : 512;
  static_assert(kTmemUsed <= 512, "TMEM overflow");
  static constexpr int kXBytes = MT * 128;
  static constexpr int kXTile = kXBytes < 1024 ? 1024 : kXBytes;  // SW128 tile stride
  static constexpr int kXSlot = XQ ? 0 : kXTile;                  // per-step activation slots
  static constexpr int kXRes = XQ ? 64 * 1024 : 0;                // resident quantized slice
  static constexpr int kXResBlocks = XQ ? kXRes / kXTile : 0;
  static constexpr int kAmaxBytes = XQ ? 8 * MT * 4 + MT * 4 + MT * 8 : 0;  // peers, local, s_a
  static constexpr int kScBytes = S * kTileN * 4;     // group scales riding with the step
  static constexpr int kStageBytes = S * (kBlockBytes + kXSlot) + kScBytes;
  // Tile partials handed from the epilogue to the reduction warps (2/3), which do
  // the cluster split-K exchange + finalise off the epilogue's critical path.
  // MT = 128 (prefill) finalises straight from the epilogue's registers.
  static constexpr int kPbufs = MT <= 64 ? 2 : 0;
  static constexpr int kPbufBytes = kPbufs * MT * kTileN * 4;
  static constexpr int kSaBytes = 2 * MT * 8;  // token scales, prefetched a tile ahead
  static constexpr int kFixed = 1024 + kXRes + kPbufBytes + kSaBytes + kAmaxBytes + 1024;
  static_assert(!XQ || kPbufs > 0, "fused activation quantization: decode tiles only");
  static constexpr int kStagesRaw = (227 * 1024 - kFixed) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmemBytes = kFixed + kStages * kStageBytes;
  static_assert(kStages >= 2, "smem");
  static_assert(kSmemBytes <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ void store_out(void* out, int dtype, int64_t idx, float f) {
  if (dtype == ISB_F32)
    static_cast<float*>(out)[idx] = f;
  else if (dtype == ISB_BF16)
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
  else
    static_cast<__half*>(out)[idx] = __float2half_rn(f);
}

// Eq. 2 epilogue (integer) / Eq. 1 (float): one double conversion per output.
template <int PATH>
__device__ __forceinline__ float finish(int32_t iacc, float facc, double s_a, double inv_amp,
                                        double s_w = 0.0) {
  double o;
  if (PATH == ISB_PATH_INTEGER_SCALE)
    o = __dmul_rn(static_cast<double>(iacc) * inv_amp, s_a);  // (acc / 2^e) * s_a, /2^e exact
  else if (PATH == ISB_PATH_COARSE)  // gemm_coarse (gemm.cpp:293): (double(acc) * s_w[j]) * s_a
    o = __dmul_rn(__dmul_rn(static_cast<double>(iacc), s_w), s_a);
  else
    o = __dmul_rn(static_cast<double>(facc), s_a);
  return __double2float_rn(o);
}

// Reduction-warp finalise of one tile: rank `rank` of a CC-CTA cluster owns tokens
// [rank*MT/CC, (rank+1)*MT/CC); thread u handles rows u and u+64. All partial
// loads (DSMEM when CC > 1) and token scales of a chunk are issued before first
// use so the chunk costs one round trip, not one per element.
template <int MT, int CC, int PATH, class P>
__device__ __forceinline__ void reduce_tile(const P& p, uint32_t pb, const double* sa_t,
                                            int rank, int nt, int mt, uint32_t u) {
  // Rank `rank` finalises tokens [rank*MT/CC, (rank+1)*MT/CC) (uneven when CC = 3).
  constexpr int SLM = (MT + CC - 1) / CC;
  constexpr int CH = SLM < 8 ? SLM : 8;
  const int lo = rank * MT / CC;
  const int sl = (MT % CC == 0) ? MT / CC : (rank + 1) * MT / CC - lo;
#pragma unroll 1
  for (int c0 = 0; c0 < sl; c0 += CH) {
    double sav[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) sav[i] = (c0 + i < sl) ? sa_t[lo + c0 + i] : 0.0;
    // both row halves' partial loads in flight before first use: one DSMEM round trip
    uint32_t vv[2][CH][CC];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < CH; ++i)
#pragma unroll
        for (int q = 0; q < CC; ++q) {
          const uint32_t off = pb + ((lo + min(c0 + i, sl - 1)) * kTileN + u + h * 64) * 4;
          vv[h][i][q] = CC > 1 ? ld_shared_cluster_u32(mapa_shared(off, q)) : ld_shared_u32(off);
        }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t rr = u + h * 64;
      const uint32_t (&v)[CH][CC] = vv[h];
      const int64_t n = static_cast<int64_t>(nt) * kTileN + rr;
      const double s_w = (PATH == ISB_PATH_COARSE && n < p.N) ? p.wscale_d[n] : 0.0;
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        int32_t is = 0;
        float fs = 0.0f;
#pragma unroll
        for (int q = 0; q < CC; ++q) {
          if (PATH != ISB_PATH_FLOAT_SCALE) is += static_cast<int32_t>(v[i][q]);
          else fs += __uint_as_float(v[i][q]);
        }
        const int64_t m = static_cast<int64_t>(mt) * MT + lo + c0 + i;
        if (c0 + i < sl && n < p.N && m < p.M) {
          if (PATH == ISB_PATH_INTEGER_SCALE && p.out_dtype == ISB_I32)
            static_cast<int32_t*>(p.out)[m * p.N + n] = is;  // raw acc (row-parallel TP)
          else
            store_out(p.out, p.out_dtype, m * p.N + n,
                      finish<PATH>(is, fs, sav[i], p.inv_amp, s_w));
        }
      }
    }
  }
}

}  // namespace
}  // namespace isb
