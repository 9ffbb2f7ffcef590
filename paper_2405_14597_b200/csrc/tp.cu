// Tensor-parallel helpers: row absmax + quantize-with-global-max
// for K-sharded activations, and the Eq. 2 epilogue of an all-reduced int32
// accumulator. HBM-bound elementwise kernels; no reference analogue (the
// reference is single-process), semantics from quantize.cpp:93-145 and
// gemm.cpp:252.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "quant.cuh"

namespace isb {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float block_max256(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < kThreads / 32 ? red[l] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// Rows are split into kChunk-element chunks, one CTA per (chunk, row): decode-sized M
// (16 rows of a 28672-wide slice) still spreads over ~100 SMs instead of 16.
constexpr int kChunk = kThreads * 16;

// max |x| over the (local slice of the) row: per-CTA max, then an atomic max on the
// float bits into amax (zeroed by the launcher; non-negative floats order as integers).
// NaNs are ignored (fmaxf), as in the one-CTA form.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    row_absmax_kernel(const T* __restrict__ x, int64_t k, float* __restrict__ amax, bool vec) {
  __shared__ float red[kThreads / 32];
  const int64_t row = blockIdx.y;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kChunk;
  const T* xr = x + row * k;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  float m = 0.0f;
  if (vec) {
    for (int64_t e = c0 + threadIdx.x * 4; e < min(k, c0 + kChunk); e += kThreads * 4) {
      float v[4];
      load4<T>(xr + e, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) m = fmaxf(m, fabsf(v[i]));
    }
  } else {
    for (int64_t e = c0 + threadIdx.x; e < min(k, c0 + kChunk); e += kThreads)
      m = fmaxf(m, fabsf(load1<T>(xr + e)));
  }
  m = block_max256(m, red);
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<int*>(amax) + row, __float_as_int(m));
}

// K1 with the row max supplied (the all-reduced global max), one CTA per (chunk, row).
template <typename T>
__global__ void __launch_bounds__(kThreads)
    quantize_amax_kernel(const T* __restrict__ x, int64_t k, const float* __restrict__ amax,
                         int8_t* __restrict__ codes, double* __restrict__ scales, bool vec) {
  const int64_t row = blockIdx.y;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kChunk;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  const float a = amax[row];
  const double s = a == 0.0f ? 1.0 : static_cast<double>(a) / 127.0;  // quantize.cpp:120-125
  const double r = 1.0 / s;
  if (threadIdx.x == 0 && blockIdx.x == 0) scales[row] = s;
  const T* xr = x + row * k;
  int8_t* cr = codes + row * k;
  if (vec) {
    for (int64_t e = c0 + threadIdx.x * 4; e < min(k, c0 + kChunk); e += kThreads * 4) {
      float v[4];
      load4<T>(xr + e, v);
      char4 q;
      q.x = static_cast<signed char>(quant_one(v[0], s, r, -128, 127));
      q.y = static_cast<signed char>(quant_one(v[1], s, r, -128, 127));
      q.z = static_cast<signed char>(quant_one(v[2], s, r, -128, 127));
      q.w = static_cast<signed char>(quant_one(v[3], s, r, -128, 127));
      *reinterpret_cast<char4*>(cr + e) = q;
    }
  } else {
    for (int64_t e = c0 + threadIdx.x; e < min(k, c0 + kChunk); e += kThreads)
      cr[e] = static_cast<int8_t>(quant_one(load1<T>(xr + e), s, r, -128, 127));
  }
}

// out[i, j] = float((double(acc[i, j]) * 2^-e) * s_a[i])  (gemm.cpp:252, /2^e exact).
__global__ void __launch_bounds__(kThreads)
    finalize_acc_kernel(const int32_t* __restrict__ acc, const double* __restrict__ sa, int64_t m,
                        int64_t n, double inv_amp, void* __restrict__ out, int dtype) {
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  const int64_t total = m * n;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * kThreads) {
    const int64_t i = idx / n;
    const double o = __dmul_rn(static_cast<double>(acc[idx]) * inv_amp, sa[i]);
    const float f = __double2float_rn(o);
    if (dtype == ISB_F32) static_cast<float*>(out)[idx] = f;
    else if (dtype == ISB_BF16) static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
    else static_cast<__half*>(out)[idx] = __float2half_rn(f);
  }
}

// Unsafe layers (static bound > int32): the GEMM runs as C K-chunks whose own bounds
// fit int32 (raw accumulators in acc[c][m][n]); the exact int64 sum of the chunks is the
// reference's acc (gemm.cpp:205-262 accumulates in int64), then Eq. 2 as above
// (double(acc) is exact below 2^53).
__global__ void __launch_bounds__(kThreads)
    finalize_chunks_kernel(int32_t* __restrict__ acc, int chunks, const double* __restrict__ sa,
                           int64_t m, int64_t n, double inv_amp, void* __restrict__ out, int dtype) {
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  const int64_t total = m * n;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * kThreads) {
    int64_t a = 0;
    for (int c = 0; c < chunks; ++c) {
      int32_t* pc = acc + c * total + idx;
      a += *pc;
      *pc = 0;  // the GEMM workspace is handed back zeroed (isb_gemm_workspace_size contract)
    }
    const int64_t i = idx / n;
    const double o = __dmul_rn(static_cast<double>(a) * inv_amp, sa[i]);
    const float f = __double2float_rn(o);
    if (dtype == ISB_F32) static_cast<float*>(out)[idx] = f;
    else if (dtype == ISB_BF16) static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
    else static_cast<__half*>(out)[idx] = __float2half_rn(f);
  }
}

template <typename K, typename... Args>
void launch_opt(bool pdl, K kern, dim3 grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl && pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, args...), "tensor-parallel kernel launch");
  count_launch();
}

template <typename K, typename... Args>
void launch_pdl(K kern, dim3 grid, cudaStream_t s, Args... args) {
  launch_opt(true, kern, grid, s, args...);
}


}  // namespace

namespace {
dim3 chunk_grid(int64_t m, int64_t k) {
  return dim3(static_cast<unsigned>(std::max<int64_t>(1, (k + kChunk - 1) / kChunk)),
              static_cast<unsigned>(m));
}
bool vec_ok(const void* x, const void* codes, int64_t k, int elt) {
  return k % 4 == 0 && reinterpret_cast<uintptr_t>(x) % (4 * elt) == 0 &&
         (codes == nullptr || reinterpret_cast<uintptr_t>(codes) % 4 == 0);
}
}  // namespace

void launch_row_absmax(const void* x, int x_dtype, int64_t m, int64_t k, float* amax,
                       cudaStream_t s) {
  if (m <= 0) return;
  cuda_check(cudaMemsetAsync(amax, 0, static_cast<size_t>(m) * sizeof(float), s), "memset(amax)");
  const dim3 grid = chunk_grid(m, k);
  // no programmatic overlap: the kernel's atomics must follow the memset
  if (x_dtype == ISB_F32)
    launch_opt(false, row_absmax_kernel<float>, grid, s, static_cast<const float*>(x), k, amax,
               vec_ok(x, nullptr, k, 4));
  else if (x_dtype == ISB_BF16)
    launch_opt(false, row_absmax_kernel<__nv_bfloat16>, grid, s,
               static_cast<const __nv_bfloat16*>(x), k, amax, vec_ok(x, nullptr, k, 2));
  else
    fail(ISB_PARAM, "activation dtype must be float32 or bfloat16");
}

void launch_quantize_amax(const void* x, int x_dtype, int64_t m, int64_t k, const float* amax,
                          int8_t* codes, double* scales, cudaStream_t s) {
  if (m <= 0) return;
  const dim3 grid = chunk_grid(m, k);
  if (x_dtype == ISB_F32)
    launch_pdl(quantize_amax_kernel<float>, grid, s, static_cast<const float*>(x), k, amax,
               codes, scales, vec_ok(x, codes, k, 4));
  else if (x_dtype == ISB_BF16)
    launch_pdl(quantize_amax_kernel<__nv_bfloat16>, grid, s,
               static_cast<const __nv_bfloat16*>(x), k, amax, codes, scales,
               vec_ok(x, codes, k, 2));
  else
    fail(ISB_PARAM, "activation dtype must be float32 or bfloat16");
}

void launch_finalize_acc(const int32_t* acc, const double* sa, int64_t m, int64_t n,
                         double inv_amp, void* out, int out_dtype, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((m * n + kThreads - 1) / kThreads, 148 * 16);
  launch_pdl(finalize_acc_kernel, dim3(static_cast<unsigned>(std::max<int64_t>(blocks, 1))), s,
             acc, sa, m, n, inv_amp, out, out_dtype);
}

void launch_finalize_chunks(int32_t* acc, int chunks, const double* sa, int64_t m, int64_t n,
                            double inv_amp, void* out, int out_dtype, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((m * n + kThreads - 1) / kThreads, 148 * 16);
  launch_pdl(finalize_chunks_kernel, dim3(static_cast<unsigned>(std::max<int64_t>(blocks, 1))), s,
             acc, chunks, sa, m, n, inv_amp, out, out_dtype);
}

}  // namespace isb
