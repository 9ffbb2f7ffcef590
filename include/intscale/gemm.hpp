// B200 drop-in for proj/include/intscale/gemm.hpp (fine-grained paths, gemm.hpp:34-126).
//
// gemm_integer_scale: output from the tcgen05 K3 kernel when the layer is eligible
// (K % 128 == 0, group % 128 == 0, 4-bit weights, static bound safe); the
// reference's accumulator statistics (max_abs_accumulator, overflow flag / first
// (i, j), strict mode, record_partials) come from the exact int64 checked kernel.
// gemm_float_scale: the checked kernel's double accumulation (bit-identical to
// gemm.cpp:156-203). The fp32 tcgen05 float-scale kernel (K4) is exposed through the
// C ABI for the speed comparison.
#pragma once

#include <string>

#include "intscale/integer_scale.hpp"
#include "intscale/quantize.hpp"

namespace intscale {

enum class PathKind { float_scale, integer_scale, coarse, dual_quant };
std::string to_string(PathKind k);
PathKind path_from_string(const std::string& s);

enum class OverflowMode { strict, permissive };
enum class FallbackPolicy { none, float_scale_on_overflow_risk };

struct GemmOptions {
  OverflowMode overflow = OverflowMode::permissive;
  int workers = 1;  // accepted for API compatibility; the GPU path has no host workers
  bool record_partials = false;
  // B200 extension: compute the reference's accumulator statistics (needs a second,
  // CUDA-core pass). false => output only, stats.max_abs_accumulator = -1.
  bool track_accumulator = true;
};

struct KernelStats {
  std::int64_t int_to_float_conversions = 0;
  std::int64_t integer_multiply_adds = 0;
  std::int64_t elementwise_multiplies = 0;
  std::int64_t elementwise_subtractions = 0;
  std::int64_t max_abs_accumulator = 0;
  bool overflow_detected = false;
  bool fallback_applied = false;
  double wall_ms = 0.0;
  bool tensor_core = false;  // B200: output came from the tcgen05 kernel
};

struct GemmResult {
  MatF output;
  KernelStats stats;
  MatI64 abs_group_partials;
  MatD output_f64;
};

GemmResult gemm_float_scale(const QuantizedTensor& x, const QuantizedTensor& w,
                            const GemmOptions& opt = {});
GemmResult gemm_integer_scale(const QuantizedTensor& x, const QuantizedTensor& w,
                              const IntegerScaleSet& int_scales, const GemmOptions& opt = {});

/// Coarse-grained (per-channel) W4A8, gemm.hpp:97 / gemm.cpp:264-309.
GemmResult gemm_coarse(const QuantizedTensor& x, const QuantizedTensor& w,
                       const GemmOptions& opt = {});

/// Inner stage of the dual-quantization path (gemm.hpp:18-27): asymmetric 4-bit
/// group codes of an 8-bit per-channel weight's integer codes.
struct DualInnerQuant {
  MatQ values;
  VecD scales;
  VecI zero_points;
  Index group_size = 128;
};

/// dual_inner_quantize (gemm.hpp:31, gemm.cpp:311-345) — on the device, bit-exact.
DualInnerQuant dual_inner_quantize(const QuantizedTensor& w_outer, Index group_size);

/// gemm_dual_quant (gemm.hpp:105, gemm.cpp:347-412): the QServe-style comparison path,
/// sequential double accumulation on CUDA cores, bit-exact.
GemmResult gemm_dual_quant(const QuantizedTensor& x, const QuantizedTensor& w_outer,
                           const DualInnerQuant& inner, const GemmOptions& opt = {});

struct PathConfig {
  PathKind kind = PathKind::integer_scale;
  const IntegerScaleSet* int_scales = nullptr;
  const DualInnerQuant* inner = nullptr;
};

GemmResult run_layer(const QuantizedTensor& x, const QuantizedTensor& w, const PathConfig& path,
                     FallbackPolicy fallback, const GemmOptions& opt = {});

}  // namespace intscale
