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

// One CTA per row: max |x| over the (local slice of the) row. Exact (max).
template <typename T>
__global__ void __launch_bounds__(kThreads)
    row_absmax_kernel(const T* __restrict__ x, int64_t k, float* __restrict__ amax) {
  __shared__ float red[kThreads / 32];
  const T* xr = x + static_cast<int64_t>(blockIdx.x) * k;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  float m = 0.0f;
  for (int64_t e = threadIdx.x; e < k; e += kThreads) m = fmaxf(m, fabsf(load1<T>(xr + e)));
  m = block_max256(m, red);
  if (threadIdx.x == 0) amax[blockIdx.x] = m;
}

// One CTA per row: K1 with the row max supplied (the all-reduced global max).
template <typename T>
__global__ void __launch_bounds__(kThreads)
    quantize_amax_kernel(const T* __restrict__ x, int64_t k, const float* __restrict__ amax,
                         int8_t* __restrict__ codes, double* __restrict__ scales) {
  const int64_t row = blockIdx.x;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  const float a = amax[row];
  const double s = a == 0.0f ? 1.0 : static_cast<double>(a) / 127.0;  // quantize.cpp:120-125
  const double r = 1.0 / s;
  if (threadIdx.x == 0) scales[row] = s;
  const T* xr = x + row * k;
  for (int64_t e = threadIdx.x; e < k; e += kThreads)
    codes[row * k + e] = static_cast<int8_t>(quant_one(load1<T>(xr + e), s, r, -128, 127));
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

template <typename K, typename... Args>
void launch_pdl(K kern, dim3 grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, args...), "tensor-parallel kernel launch");
  count_launch();
}

}  // namespace

void launch_row_absmax(const void* x, int x_dtype, int64_t m, int64_t k, float* amax,
                       cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>(m));
  if (x_dtype == ISB_F32)
    launch_pdl(row_absmax_kernel<float>, grid, s, static_cast<const float*>(x), k, amax);
  else if (x_dtype == ISB_BF16)
    launch_pdl(row_absmax_kernel<__nv_bfloat16>, grid, s,
               static_cast<const __nv_bfloat16*>(x), k, amax);
  else
    fail(ISB_PARAM, "activation dtype must be float32 or bfloat16");
}

void launch_quantize_amax(const void* x, int x_dtype, int64_t m, int64_t k, const float* amax,
                          int8_t* codes, double* scales, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>(m));
  if (x_dtype == ISB_F32)
    launch_pdl(quantize_amax_kernel<float>, grid, s, static_cast<const float*>(x), k, amax,
               codes, scales);
  else if (x_dtype == ISB_BF16)
    launch_pdl(quantize_amax_kernel<__nv_bfloat16>, grid, s,
               static_cast<const __nv_bfloat16*>(x), k, amax, codes, scales);
  else
    fail(ISB_PARAM, "activation dtype must be float32 or bfloat16");
}

void launch_finalize_acc(const int32_t* acc, const double* sa, int64_t m, int64_t n,
                         double inv_amp, void* out, int out_dtype, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((m * n + kThreads - 1) / kThreads, 148 * 16);
  launch_pdl(finalize_acc_kernel, dim3(static_cast<unsigned>(std::max<int64_t>(blocks, 1))), s,
             acc, sa, m, n, inv_amp, out, out_dtype);
}

}  // namespace isb
