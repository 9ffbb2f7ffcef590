// int4 -> (k_g * w) int8 expansion shared by the folded K3 kernels (gemm_fold.cu,
// gemm_tc.cu FD): the integer scale k_g <= 16 is folded into the weight operand so
// the tensor core accumulates sum_g k_g * P_g directly (exact).
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

namespace isb {
namespace {

// ((w ^ x) & m) | o as one LOP3 (x subset of m, o disjoint from m):
// f(w, b = m, c = x | o) = b ? (w ^ c) : c  -> LUT 0x6A.
__device__ __forceinline__ uint32_t lop_extract(uint32_t w, uint32_t m, uint32_t xo) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(w), "r"(m), "r"(xo));
  return d;
}

__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint32_t half2_bits(float v) {
  const __half h = __float2half_rn(v);
  const uint32_t u = __half_as_ushort(h);
  return u | (u << 16);
}

// One packed word (8 two's-complement nibbles; byte b = code(k0+b) | code(k0+4+b) << 4)
// -> k*code for k0..k0+3 (lo) and k0+4..k0+7 (hi), int8 lanes.
// Nibble n at bit 0 of a 16-bit lane, biased (XOR 8 -> c + 8) and OR'ed into an fp16
// with exponent field 0x64 is exactly 1024 + (c + 8); at bit 4 it is 1024 + 16 (c + 8).
// HFMA2 (exact: the result is an integer in [1408, 1648], representable) gives
// 1536 + k*c, whose low mantissa byte is (512 + k*c) mod 256 = k*c mod 256.
__device__ __forceinline__ void fold_word(uint32_t w, uint32_t k1, uint32_t k16, uint32_t cA,
                                          uint32_t cB, uint32_t& lo, uint32_t& hi) {
  const uint32_t w8 = w >> 8;
  const uint32_t hA = lop_extract(w, 0x000F000Fu, 0x64086408u);   // codes k0, k0+2
  const uint32_t hB = lop_extract(w, 0x00F000F0u, 0x64806480u);   // k0+4, k0+6
  const uint32_t hC = lop_extract(w8, 0x000F000Fu, 0x64086408u);  // k0+1, k0+3
  const uint32_t hD = lop_extract(w8, 0x00F000F0u, 0x64806480u);  // k0+5, k0+7
  const uint32_t rA = hfma2(hA, k1, cA);
  const uint32_t rB = hfma2(hB, k16, cB);
  const uint32_t rC = hfma2(hC, k1, cA);
  const uint32_t rD = hfma2(hD, k16, cB);
  lo = __byte_perm(rA, rC, 0x6240);
  hi = __byte_perm(rB, rD, 0x6240);
}


// fp16 constants of fold_word for one k_g.
struct FoldK {
  uint32_t k1, k16, cA, cB;
};
__device__ __forceinline__ FoldK fold_constants(int32_t k) {
  const float kf = static_cast<float>(k);
  return {half2_bits(kf), half2_bits(kf * 0.0625f), half2_bits(1536.0f - 1032.0f * kf),
          half2_bits(1536.0f - 72.0f * kf)};
}

}  // namespace
}  // namespace isb
