// QServe-style dual quantization (the paper's QServe comparison):
// an 8-bit per-channel symmetric weight whose integer codes are re-quantized to
// asymmetric 4-bit groups, GEMM'd by reconstructing (w - z) * s_i in double.
//
// Reference: dual_inner_quantize (gemm.cpp:311-345) and gemm_dual_quant
// (gemm.cpp:347-412). The reference accumulates every product sequentially in
// double, so the result depends on the order of K; these CUDA-core kernels keep that
// order per output (one thread per (i, j), IEEE __dmul_rn / __dadd_rn, no FMA
// contraction) and are bit-identical to it. This is the comparison path the paper
// measures against (its real-domain reconstruction is the cost the integer scale
// avoids), not a tensor-core kernel.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace isb {
namespace {

__device__ __forceinline__ int64_t llround_(double v) {  // half away from zero
  return static_cast<int64_t>(round(v));
}

__device__ __forceinline__ int64_t clamp15(int64_t v) { return v < 0 ? 0 : (v > 15 ? 15 : v); }

__global__ void dual_inner_quantize_kernel(const int16_t* __restrict__ w8, int64_t k, int64_t n,
                                           int64_t group, int16_t* __restrict__ codes,
                                           double* __restrict__ scales, int32_t* __restrict__ zps) {
  const int64_t groups = k / group;
  const int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // j*G + t
  if (u >= n * groups) return;
  const int64_t j = u / groups, t = u % groups;
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t r = t * group; r < (t + 1) * group; ++r) {
    const double v = static_cast<double>(w8[r * n + j]);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  const double s = hi == lo ? 1.0 : __ddiv_rn(hi - lo, 15.0);
  const int32_t z = static_cast<int32_t>(clamp15(llround_(__ddiv_rn(-lo, s))));
  scales[u] = s;
  zps[u] = z;
  for (int64_t r = t * group; r < (t + 1) * group; ++r) {
    const int64_t q = llround_(__ddiv_rn(static_cast<double>(w8[r * n + j]), s)) + z;
    codes[r * n + j] = static_cast<int16_t>(clamp15(q));
  }
}

// Error flags: [0] activation code -128, [1] inner code outside [0, 15],
// [2] zero point outside [0, 15], [3] scale not positive / finite.
__global__ void dual_validate_kernel(const int8_t* __restrict__ xq, int64_t mk,
                                     const int16_t* __restrict__ codes, int64_t kn,
                                     const int32_t* __restrict__ zps,
                                     const double* __restrict__ scales, int64_t units,
                                     int* __restrict__ flags) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < mk; i += stride)
    if (xq[i] == -128) flags[0] = 1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < kn; i += stride)
    if (codes[i] < 0 || codes[i] > 15) flags[1] = 1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < units; i += stride) {
    if (zps[i] < 0 || zps[i] > 15) flags[2] = 1;
    if (!(scales[i] > 0.0) || !isfinite(scales[i])) flags[3] = 1;
  }
}

__global__ void __launch_bounds__(128)
    gemm_dual_quant_kernel(const int8_t* __restrict__ xq, const double* __restrict__ sa,
                           int64_t m, int64_t k, const int16_t* __restrict__ codes,
                           const double* __restrict__ scales, const int32_t* __restrict__ zps,
                           int64_t group, const double* __restrict__ s_outer, int64_t n,
                           float* __restrict__ out, double* __restrict__ out_f64) {
  const int64_t j = blockIdx.x * 128ll + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= n || i >= m) return;
  const int64_t groups = k / group;
  const int8_t* xr = xq + i * k;
  double cd = 0.0;
  for (int64_t gi = 0; gi < groups; ++gi) {
    const double si = scales[j * groups + gi];
    const int32_t z = zps[j * groups + gi];
    for (int64_t kk = gi * group; kk < (gi + 1) * group; ++kk) {
      const double wrec = __dmul_rn(static_cast<double>(static_cast<int32_t>(codes[kk * n + j]) - z), si);
      cd = __dadd_rn(cd, __dmul_rn(static_cast<double>(xr[kk]), wrec));
    }
  }
  const double o = __dmul_rn(__dmul_rn(cd, s_outer[j]), sa[i]);
  out[i * n + j] = __double2float_rn(o);
  if (out_f64) out_f64[i * n + j] = o;
}

}  // namespace

void launch_dual_inner_quantize(const int16_t* w8, int64_t k, int64_t n, int64_t group,
                                int16_t* codes, double* scales, int32_t* zps, cudaStream_t s) {
  const int64_t units = n * (k / group);
  dual_inner_quantize_kernel<<<static_cast<unsigned>((units + 127) / 128), 128, 0, s>>>(
      w8, k, n, group, codes, scales, zps);
  cuda_check(cudaGetLastError(), "dual_inner_quantize launch");
  count_launch();
}

void validate_dual(const int8_t* xq, int64_t m, int64_t k, const int16_t* codes, int64_t n,
                   const int32_t* zps, const double* scales, int64_t group, cudaStream_t s) {
  int* flags = nullptr;
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&flags), 4 * sizeof(int), s), "cudaMallocAsync");
  cuda_check(cudaMemsetAsync(flags, 0, 4 * sizeof(int), s), "memset");
  dual_validate_kernel<<<148, 256, 0, s>>>(xq, m * k, codes, k * n, zps, scales, n * (k / group),
                                          flags);
  cuda_check(cudaGetLastError(), "dual validate launch");
  count_launch();
  int h[4] = {0, 0, 0, 0};
  cuda_check(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s), "copy flags");
  cuda_check(cudaStreamSynchronize(s), "sync");
  cudaFreeAsync(flags, s);
  // validate_activation (gemm.cpp:114), then the inner checks (gemm.cpp:366-372)
  if (h[0]) fail(ISB_VALUE, "activation code -128 outside the symmetric range");
  if (h[1]) fail(ISB_VALUE, "inner codes outside [0, 15]");
  if (h[2]) fail(ISB_VALUE, "inner zero point outside [0, 15]");
  if (h[3]) fail(ISB_VALUE, "inner scale must be positive and finite");
}

void launch_gemm_dual_quant(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                            const int16_t* codes, const double* scales, const int32_t* zps,
                            int64_t group, const double* s_outer, int64_t n, float* out,
                            double* out_f64, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>(m));
  gemm_dual_quant_kernel<<<grid, 128, 0, s>>>(xq, sa, m, k, codes, scales, zps, group, s_outer, n,
                                             out, out_f64);
  cuda_check(cudaGetLastError(), "gemm_dual_quant launch");
  count_launch();
}

}  // namespace isb
