// K1 — per-token symmetric int8 activation quantizer, and the offline group
// weight quantizer that feeds the packer.
//
// Reference semantics: quantize(x, 8, symmetric, per_token) and
// quantize(w, 4, symmetric, group_of(g)), quantize.cpp:93-145:
//   s = max(|min|, |max|) / qmax over the unit (s = 1 when the unit is all 0),
//   q = clamp(llround(double(x) / s), qmin, qmax)   (round half away from zero)
// Both are reproduced bit-exactly.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"
#include "quant.cuh"

#include <algorithm>
#include <cstdlib>

namespace isb {
namespace {

constexpr int kQuantThreads = 256;

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < kQuantThreads / 32 ? red[l] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const float r = red[0];
  __syncthreads();
  return r;
}

// One CTA per token row; the row stays in registers (V x 4 elements per
// thread), so HBM is read exactly once: M*K*sizeof(T) in, M*K + 8M out.
template <int V, typename T>
__global__ void __launch_bounds__(kQuantThreads)
    quantize_rows_cached(const T* __restrict__ x, int64_t k, int8_t* __restrict__ codes,
                         double* __restrict__ scales, int* __restrict__ bad) {
  __shared__ float red[kQuantThreads / 32];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * k;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // x may be produced by the preceding grid
  float v[V][4];
  float amax = 0.0f;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t e = (static_cast<int64_t>(i) * kQuantThreads + threadIdx.x) * 4;
    if (e < k) {
      load4<T>(xr + e, v[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        finite = finite && isfinite(v[i][j]);
        amax = fmaxf(amax, fabsf(v[i][j]));
      }
    }
  }
  if (!finite) atomicExch(bad, 1);
  amax = block_max(amax, red);
  const double s = amax == 0.0f ? 1.0 : static_cast<double>(amax) / 127.0;
  const double r = 1.0 / s;
  if (threadIdx.x == 0) scales[row] = s;
  int8_t* cr = codes + row * k;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t e = (static_cast<int64_t>(i) * kQuantThreads + threadIdx.x) * 4;
    if (e < k) {
      uint32_t packed = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        packed |= (static_cast<uint32_t>(quant_one(v[i][j], s, r, -128, 127)) & 0xFFu) << (8 * j);
      *reinterpret_cast<uint32_t*>(cr + e) = packed;
    }
  }
}

// Decode-sized M: a cluster of CPR CTAs shares one token row (each CTA owns a
// contiguous K slice held in registers); the row max is combined over DSMEM, so a
// 16-token activation is quantised by 16*CPR CTAs instead of 16.
template <int V, typename T>
__global__ void __launch_bounds__(kQuantThreads)
    quantize_rows_cluster(const T* __restrict__ x, int64_t k, int64_t chunk,
                          int8_t* __restrict__ codes, double* __restrict__ scales,
                          int* __restrict__ bad) {
  __shared__ float red[kQuantThreads / 32];
  __shared__ float cta_max;
  const uint32_t cpr = gridDim.y;                      // cluster spans blockIdx.y
  const uint32_t rank = cluster_ctarank();
  const int64_t row = blockIdx.x;
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * chunk;
  const int64_t k1 = min(k, k0 + chunk);
  const T* xr = x + row * k;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  float v[V][4];
  float amax = 0.0f;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t e = k0 + (static_cast<int64_t>(i) * kQuantThreads + threadIdx.x) * 4;
    if (e < k1) {
      load4<T>(xr + e, v[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        finite = finite && isfinite(v[i][j]);
        amax = fmaxf(amax, fabsf(v[i][j]));
      }
    }
  }
  if (!finite) atomicExch(bad, 1);
  amax = block_max(amax, red);
  if (threadIdx.x == 0) cta_max = amax;
  cluster_sync_all();
  if (threadIdx.x < 32) {
    float mx = 0.0f;
    for (uint32_t q = threadIdx.x; q < cpr; q += 32)
      mx = fmaxf(mx, __uint_as_float(ld_shared_cluster_u32(mapa_shared(smem_u32(&cta_max), q))));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) red[0] = mx;
  }
  cluster_sync_all();  // peers finished reading cta_max; red[0] visible CTA-wide
  amax = red[0];
  const double s = amax == 0.0f ? 1.0 : static_cast<double>(amax) / 127.0;
  const double r = 1.0 / s;
  if (threadIdx.x == 0 && rank == 0) scales[row] = s;
  int8_t* cr = codes + row * k;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t e = k0 + (static_cast<int64_t>(i) * kQuantThreads + threadIdx.x) * 4;
    if (e < k1) {
      uint32_t packed = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        packed |= (static_cast<uint32_t>(quant_one(v[i][j], s, r, -128, 127)) & 0xFFu) << (8 * j);
      *reinterpret_cast<uint32_t*>(cr + e) = packed;
    }
  }
}

// Decode-sized M, K <= 1024 * 4 * V: one 1024-thread CTA per token row, every
// thread holds V float4 of the row, so all loads of the row are in flight at once
// and a single block reduction gives the row max (no cluster barriers).
template <int V, typename T>
__global__ void __launch_bounds__(1024)
    quantize_rows_wide(const T* __restrict__ x, int64_t k, int8_t* __restrict__ codes,
                       double* __restrict__ scales, int* __restrict__ bad) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * k;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // x may be produced by the preceding grid
  float v[V][4];
  float amax = 0.0f;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t e = (static_cast<int64_t>(i) * 1024 + threadIdx.x) * 4;
    if (e < k) {
      load4<T>(xr + e, v[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        finite = finite && isfinite(v[i][j]);
        amax = fmaxf(amax, fabsf(v[i][j]));
      }
    }
  }
  if (!finite) atomicExch(bad, 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = amax;
  __syncthreads();
  amax = red[threadIdx.x & 31];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const double s = amax == 0.0f ? 1.0 : static_cast<double>(amax) / 127.0;
  const double r = 1.0 / s;
  if (threadIdx.x == 0) scales[row] = s;
  int8_t* cr = codes + row * k;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t e = (static_cast<int64_t>(i) * 1024 + threadIdx.x) * 4;
    if (e < k) {
      uint32_t packed = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        packed |= (static_cast<uint32_t>(quant_one(v[i][j], s, r, -128, 127)) & 0xFFu) << (8 * j);
      *reinterpret_cast<uint32_t*>(cr + e) = packed;
    }
  }
}

// Any K / alignment: two passes over the row (the second hits L2).
template <typename T>
__global__ void __launch_bounds__(kQuantThreads)
    quantize_rows_generic(const T* __restrict__ x, int64_t k, int8_t* __restrict__ codes,
                          double* __restrict__ scales, int* __restrict__ bad) {
  __shared__ float red[kQuantThreads / 32];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * k;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  float amax = 0.0f;
  bool finite = true;
  for (int64_t e = threadIdx.x; e < k; e += kQuantThreads) {
    const float f = load1<T>(xr + e);
    finite = finite && isfinite(f);
    amax = fmaxf(amax, fabsf(f));
  }
  if (!finite) atomicExch(bad, 1);
  amax = block_max(amax, red);
  const double s = amax == 0.0f ? 1.0 : static_cast<double>(amax) / 127.0;
  const double r = 1.0 / s;
  if (threadIdx.x == 0) scales[row] = s;
  for (int64_t e = threadIdx.x; e < k; e += kQuantThreads)
    codes[row * k + e] = static_cast<int8_t>(quant_one(load1<T>(xr + e), s, r, -128, 127));
}

// Offline group quantizer: one thread per (column n, group t); consecutive
// threads take consecutive columns so every row read is coalesced.
__global__ void quantize_weight_groups_kernel(const float* __restrict__ w, int64_t k, int64_t n,
                                              int64_t g, int bits, int16_t* __restrict__ codes,
                                              double* __restrict__ scales, int* __restrict__ bad) {
  const int64_t groups = k / g;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * groups) return;
  const int64_t c = idx % n, t = idx / n;
  const int qmax = (1 << (bits - 1)) - 1, qmin = -(1 << (bits - 1));
  double amax = 0.0;
  bool finite = true;
  for (int64_t r = t * g; r < (t + 1) * g; ++r) {
    const float v = w[r * n + c];
    finite = finite && isfinite(v);
    amax = fmax(amax, fabs(static_cast<double>(v)));
  }
  if (!finite) atomicExch(bad, 1);
  const double s = amax == 0.0 ? 1.0 : amax / static_cast<double>(qmax);
  scales[c * groups + t] = s;  // unit = c * (K/g) + r/g   (quantize.cpp:51)
  for (int64_t r = t * g; r < (t + 1) * g; ++r) {
    double q = round(static_cast<double>(w[r * n + c]) / s);
    q = fmin(fmax(q, static_cast<double>(qmin)), static_cast<double>(qmax));
    codes[r * n + c] = static_cast<int16_t>(q);
  }
}

template <typename T>
void launch_rows(const T* x, int64_t m, int64_t k, int8_t* codes, double* scales, int* bad,
                 cudaStream_t s) {
  const bool vec_ok = (k % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % (4 * sizeof(T)) == 0) &&
                      (reinterpret_cast<uintptr_t>(codes) % 4 == 0);
  const int64_t per_pass = static_cast<int64_t>(kQuantThreads) * 4;
  const int64_t v = (k + per_pass - 1) / per_pass;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(m));
  cfg.blockDim = dim3(kQuantThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  // Decode-sized M: one 1024-thread CTA per row holds the whole row (K <= 16384).
  static const int k1_mode = [] {  // ISB_K1=cluster keeps the cluster variant (A/B)
    const char* e = std::getenv("ISB_K1");
    return (e && e[0] == 'c') ? 1 : 0;
  }();
  if (vec_ok && m < 148 && k1_mode == 0 && k <= 4096 * 4) {
    cfg.blockDim = dim3(1024);
    const int64_t vw = (k + 4095) / 4096;
    if (vw <= 1)
      e = cudaLaunchKernelEx(&cfg, quantize_rows_wide<1, T>, x, k, codes, scales, bad);
    else if (vw <= 2)
      e = cudaLaunchKernelEx(&cfg, quantize_rows_wide<2, T>, x, k, codes, scales, bad);
    else
      e = cudaLaunchKernelEx(&cfg, quantize_rows_wide<4, T>, x, k, codes, scales, bad);
    cuda_check(e, "quantize_per_token launch");
    count_launch();
    return;
  }
  // Decode-sized M: spread each row over a cluster of CTAs (<= 1024 elements each).
  const int64_t cpr = std::min<int64_t>(8, (k + 1023) / 1024);
  if (vec_ok && m < 148 && cpr > 1 && round_up((k + cpr - 1) / cpr, 4) <= 4096) {
    const int64_t chunk = round_up((k + cpr - 1) / cpr, 4);
    cfg.gridDim = dim3(static_cast<unsigned>(m), static_cast<unsigned>(cpr));
    cudaLaunchAttribute cattr[2];
    cattr[0] = attr[0];
    cattr[1].id = cudaLaunchAttributeClusterDimension;
    cattr[1].val.clusterDim.x = 1;
    cattr[1].val.clusterDim.y = static_cast<unsigned>(cpr);
    cattr[1].val.clusterDim.z = 1;
    cfg.attrs = cattr;
    cfg.numAttrs = 2;
    if (chunk <= 1024)
      e = cudaLaunchKernelEx(&cfg, quantize_rows_cluster<1, T>, x, k, chunk, codes, scales, bad);
    else if (chunk <= 2048)
      e = cudaLaunchKernelEx(&cfg, quantize_rows_cluster<2, T>, x, k, chunk, codes, scales, bad);
    else
      e = cudaLaunchKernelEx(&cfg, quantize_rows_cluster<4, T>, x, k, chunk, codes, scales, bad);
    cuda_check(e, "quantize_per_token launch");
    count_launch();
    return;
  }
  if (vec_ok && v <= 1)
    e = cudaLaunchKernelEx(&cfg, quantize_rows_cached<1, T>, x, k, codes, scales, bad);
  else if (vec_ok && v <= 2)
    e = cudaLaunchKernelEx(&cfg, quantize_rows_cached<2, T>, x, k, codes, scales, bad);
  else if (vec_ok && v <= 4)
    e = cudaLaunchKernelEx(&cfg, quantize_rows_cached<4, T>, x, k, codes, scales, bad);
  else if (vec_ok && v <= 8)
    e = cudaLaunchKernelEx(&cfg, quantize_rows_cached<8, T>, x, k, codes, scales, bad);
  else if (vec_ok && v <= 14)
    e = cudaLaunchKernelEx(&cfg, quantize_rows_cached<14, T>, x, k, codes, scales, bad);
  else
    e = cudaLaunchKernelEx(&cfg, quantize_rows_generic<T>, x, k, codes, scales, bad);
  cuda_check(e, "quantize_per_token launch");
  cuda_check(cudaGetLastError(), "quantize_per_token launch");
  count_launch();
}

}  // namespace

void launch_quantize_per_token(const void* x, int x_dtype, int64_t m, int64_t k, int8_t* codes,
                               double* scales, int* bad, cudaStream_t s) {
  if (x_dtype == ISB_F32)
    launch_rows(static_cast<const float*>(x), m, k, codes, scales, bad, s);
  else if (x_dtype == ISB_BF16)
    launch_rows(static_cast<const __nv_bfloat16*>(x), m, k, codes, scales, bad, s);
  else
    fail(ISB_PARAM, "activation dtype must be float32 or bfloat16");
}

void launch_quantize_weight_groups(const float* w, int64_t k, int64_t n, int64_t group,
                                        int bits, int16_t* codes, double* scales, int* bad,
                                        cudaStream_t s) {
  const int64_t total = n * (k / group);
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  quantize_weight_groups_kernel<<<static_cast<unsigned>(blocks), threads, 0, s>>>(
      w, k, n, group, bits, codes, scales, bad);
  cuda_check(cudaGetLastError(), "quantize_weight_groups launch");
  count_launch();
}

}  // namespace isb
