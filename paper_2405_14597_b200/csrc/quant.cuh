// Per-element pieces of the bit-exact per-token quantizer (K1), shared by
// quant.cu and the tensor-parallel kernels in tp.cu. Semantics:
// quantize.cpp:93-145 (q = clamp(llround(double(x) / s), qmin, qmax)).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace isb {

// llround(double(x) / s) (quantize.cpp:136-142), computed as an fp32 product
// x * fl32(1/s) except within 1e-3 of a rounding tie, where the exact IEEE
// double quotient decides. The fp32 product is within ~2.3e-5 of the real
// quotient for |x/s| <= 127 (two roundings of 2^-24 relative), so outside the
// window both round to the same integer; ties are never decided in fp32.
// The exact path (IEEE double quotient, round half away from zero), out of line:
// taken for ~0.2% of elements, it would otherwise bloat every unrolled call site.
static __device__ __noinline__ float quant_exact(float xf, double s) {
  return static_cast<float>(round(static_cast<double>(xf) / s));
}

__device__ __forceinline__ int quant_one(float xf, double s, double r, int qmin, int qmax) {
  const float rf = static_cast<float>(r);
  const float y = xf * rf;
  const float ay = fabsf(y);
  float q = rintf(y);  // not near a tie: nearest integer == round half away from zero
  // Rows with absmax below ~127/FLT_MAX make fl32(1/s) infinite: the exact path
  // decides every element of such a row (the comparison is false for inf/NaN).
  if (!(fabsf((ay - floorf(ay)) - 0.5f) > 1e-3f) || !(rf <= 3.4e38f)) q = quant_exact(xf, s);
  q = fminf(fmaxf(q, static_cast<float>(qmin)), static_cast<float>(qmax));
  return static_cast<int>(q);
}

template <typename T>
__device__ __forceinline__ void load4(const T* p, float (&v)[4]);

template <>
__device__ __forceinline__ void load4<float>(const float* p, float (&v)[4]) {
  const float4 f = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
}

template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* p, float (&v)[4]) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  v[0] = __uint_as_float(u.x << 16);
  v[1] = __uint_as_float(u.x & 0xFFFF0000u);
  v[2] = __uint_as_float(u.y << 16);
  v[3] = __uint_as_float(u.y & 0xFFFF0000u);
}

template <typename T>
__device__ __forceinline__ float load1(const T* p);
template <>
__device__ __forceinline__ float load1<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float load1<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

}  // namespace isb
