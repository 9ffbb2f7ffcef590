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
#include "intscale_b200.h"

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
  // B200 extension, opt-in: compute the reference's accumulator statistics
  // (max_abs_accumulator / overflow flag) with a second, exact int64 CUDA-core pass.
  // false (default) => tcgen05 output only, stats.max_abs_accumulator = -1. Strict mode,
  // record_partials and layers outside the tensor-core envelope always run that pass.
  bool track_accumulator = false;
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

/// B200 performance entry points (SURVEY §8b "packed-weight handle + device X"): the
/// host-matrix functions above upload and pack on every call, as the reference
/// signatures require; these keep the packed weight and the activations in HBM and
/// only enqueue kernels on `stream` (no host copies, no allocation, no synchronization).
/// Results are bit-identical to the host-matrix calls on the same inputs.
namespace device {

enum class OutType { f32 = 0, bf16 = 1, f16 = 2, i32 = 3 };  // = ISB_F32 .. ISB_I32

/// The reference's K x N 4-bit group-quantized weight (quantize.cpp:93-145 output),
/// packed once into the device layout (the reference's gemm.hpp:92 weight argument).
/// With `int_scales` (integerize_scales of the same weight) the integer-scale path is
/// available; without, only the float-scale path.
class PackedWeight {
 public:
  explicit PackedWeight(const QuantizedTensor& w, const IntegerScaleSet* int_scales = nullptr,
                        void* stream = nullptr);
  ~PackedWeight();
  PackedWeight(PackedWeight&& o) noexcept;
  PackedWeight& operator=(PackedWeight&& o) noexcept;
  PackedWeight(const PackedWeight&) = delete;
  PackedWeight& operator=(const PackedWeight&) = delete;
  const isb_weight* handle() const { return h_; }
  Index k() const { return k_; }
  Index n() const { return n_; }

 private:
  isb_weight* h_ = nullptr;
  Index k_ = 0, n_ = 0;
};

/// Per-token int8 codes [m][k] and their double scales [m], device pointers (caller-owned).
struct Activations {
  std::int8_t* codes = nullptr;
  double* scales = nullptr;
  Index m = 0, k = 0;
};

/// quantize(x, 8, symmetric, per_token) (quantize.cpp:93-145) of a device float32 [m][k]
/// into `out` (its codes / scales must hold m*k bytes / m doubles). Non-finite inputs are
/// not checked here (the check needs a host read-back); use the host-matrix quantize.
void quantize_per_token(const float* x, Activations& out, void* stream = nullptr);

/// Device workspace bytes for an [m x k] activation against `w` (zero-filled once by the
/// caller before first use; the kernels leave it zeroed).
std::size_t workspace_bytes(Index m, const PackedWeight& w);

/// out[m][n] (device, `type`) = gemm_integer_scale(x, w) (gemm.cpp:205-262). Throws
/// OverflowError if the weight's overflow_analyzer bound exceeds int32 (run the host-matrix
/// call, or gemm_float_scale, as run_layer's fallback does).
void gemm_integer_scale(const Activations& x, const PackedWeight& w, void* out, OutType type,
                        void* workspace, std::size_t workspace_bytes, void* stream = nullptr);
/// out[m][n] = gemm_float_scale(x, w) (gemm.cpp:156-203) on the tensor core (fp32 group
/// accumulation: within float rounding of the reference's double accumulation).
void gemm_float_scale(const Activations& x, const PackedWeight& w, void* out, OutType type,
                      void* workspace, std::size_t workspace_bytes, void* stream = nullptr);

}  // namespace device

}  // namespace intscale
