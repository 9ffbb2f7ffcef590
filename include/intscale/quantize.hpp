// B200 drop-in for proj/include/intscale/quantize.hpp (quantize.hpp:12-93).
// quantize() runs on the GPU: symmetric per-token 8-bit uses K1, symmetric
// group / per-channel weights use the group quantizer; both bit-exact with
// quantize.cpp:93-145. Other schemes/granularities are outside the B200 path
// (ParamError).
#pragma once

#include <filesystem>
#include <string>

#include "intscale/types.hpp"

namespace intscale {

enum class Scheme { symmetric, asymmetric };
enum class GranKind { per_tensor, per_token, per_channel, group };

struct Granularity {
  GranKind kind = GranKind::group;
  Index group_size = 128;

  static Granularity per_tensor() { return {GranKind::per_tensor, 0}; }
  static Granularity per_token() { return {GranKind::per_token, 0}; }
  static Granularity per_channel() { return {GranKind::per_channel, 0}; }
  static Granularity group_of(Index g = 128) { return {GranKind::group, g}; }

  void validate(Index rows, Index cols) const;   // quantize.cpp:26-34
  Index unit_count(Index rows, Index cols) const;  // quantize.cpp:36-44
  Index unit_of(Index rows, Index r, Index c) const;  // quantize.cpp:46-54
};

struct QuantParams {
  int bit_width = 4;
  Scheme scheme = Scheme::symmetric;
  Granularity granularity;
  VecD scales;
  VecI zero_points;

  std::int64_t qmin() const;  // quantize.cpp:84-86
  std::int64_t qmax() const;  // quantize.cpp:88-91
};

struct QuantizedTensor {
  MatQ values;
  QuantParams params;
  Index rows() const { return values.rows(); }
  Index cols() const { return values.cols(); }
};

QuantizedTensor quantize(const MatF& x, int bit_width, Scheme scheme, const Granularity& g);

// Names and sidecar persistence (quantize.hpp:40-43, :91-93; quantize.cpp:56-82,
// :175-270). The values go to a QTNS file, the parameters to `<path>.json`.
std::string to_string(Scheme s);
std::string to_string(GranKind k);
Scheme scheme_from_string(const std::string& s);
GranKind gran_kind_from_string(const std::string& s);
void write_quantized(const QuantizedTensor& q, const std::filesystem::path& values_path);
QuantizedTensor read_quantized(const std::filesystem::path& values_path);

}  // namespace intscale
