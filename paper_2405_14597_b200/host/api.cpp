// C++ drop-in layer: the reference operator API (namespace intscale,
// proj/include/intscale/*.hpp) implemented on top of the C ABI
// (include/intscale_b200.h). Host code validates arguments exactly as the
// reference does (gemm.cpp:106-134, :212-216; quantize.cpp:93-96) and moves data;
// every compute step is a CUDA kernel of this library.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/intscale/analysis.hpp"
#include "../../include/intscale/gemm.hpp"
#include "../../include/intscale/integer_scale.hpp"
#include "../../include/intscale/quantize.hpp"
#include "../../include/intscale/tensor_io.hpp"
#include "../../include/intscale_b200.h"

namespace intscale {
namespace {

[[noreturn]] void throw_status(int rc, const std::string& msg) {
  switch (rc) {
    case ISB_PARAM: throw ParamError(msg);
    case ISB_DIMENSION: throw DimensionError(msg);
    case ISB_VALUE: throw ValueError(msg);
    case ISB_OVERFLOW: throw OverflowError(msg);
    case ISB_LENGTH: throw LengthError(msg);
    case ISB_FORMAT: throw FormatError(msg);
    default: throw Error(msg);
  }
}

void check(int rc) {
  if (rc != ISB_OK) throw_status(rc, isb_last_error());
}

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device buffer.
struct Dev {
  void* p = nullptr;
  explicit Dev(std::size_t bytes) {
    if (bytes) cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

template <class T>
void up(Dev& d, const T* h, std::size_t n) {
  cuda(cudaMemcpy(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
}
template <class T>
void down(T* h, const Dev& d, std::size_t n) {
  cuda(cudaMemcpy(h, d.p, n * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
}

struct Weight {
  isb_weight* h = nullptr;
  ~Weight() { isb_weight_destroy(h); }
};

bool all_finite(const MatF& x) {
  for (Index i = 0; i < x.size(); ++i)
    if (!std::isfinite(x.data()[i])) return false;
  return true;
}


// gemm.cpp:106-116
void validate_activation(const QuantizedTensor& x) {
  if (x.params.scheme != Scheme::symmetric || x.params.granularity.kind != GranKind::per_token)
    throw ParamError("activations must be symmetric per-token quantized");
  if (x.params.bit_width != 8) throw ParamError("activations must be 8-bit");
  if (x.params.scales.size() != x.rows()) throw ParamError("activation scale count != rows");
  if (x.values.minCoeff() < -x.params.qmax() || x.values.maxCoeff() > x.params.qmax())
    throw ValueError("activation codes outside max-based symmetric range");
}

// gemm.cpp:119-134 (the weight part)
Index validate_weight(const QuantizedTensor& w) {
  if (w.params.scheme != Scheme::symmetric) throw ParamError("weights must be symmetric");
  const GranKind kind = w.params.granularity.kind;
  if (kind != GranKind::group && kind != GranKind::per_channel)
    throw ParamError("weights must be group or per-channel quantized");
  if (w.values.minCoeff() < w.params.qmin() || w.values.maxCoeff() > w.params.qmax())
    throw ValueError("weight codes outside quantized range");
  const Index g = kind == GranKind::group ? w.params.granularity.group_size : w.rows();
  w.params.granularity.validate(w.rows(), w.cols());
  if (w.params.scales.size() != (w.rows() / g) * w.cols())
    throw ParamError("weight scale count does not match grouping");
  if (w.params.bit_width != 4)
    throw ParamError("the B200 path packs 4-bit weights (W4A8); got " +
                     std::to_string(w.params.bit_width) + "-bit");
  return g;
}

// gemm.cpp:119-134
Index validate_grouped_weight(const QuantizedTensor& x, const QuantizedTensor& w) {
  if (x.cols() != w.rows())
    throw DimensionError("activation K=" + std::to_string(x.cols()) + " vs weight rows " +
                         std::to_string(w.rows()));
  return validate_weight(w);
}

// Device operands of one GEMM call.
struct Operands {
  Index m, k, n, g, groups;
  Dev xq, sa, codes, scales, ks;
  Weight w;
  Operands(const QuantizedTensor& x, const QuantizedTensor& wq, Index g_, const VecI* int_scales,
           std::int64_t amp)
      : m(x.rows()), k(x.cols()), n(wq.cols()), g(g_), groups(wq.rows() / g_),
        xq(static_cast<std::size_t>(m * k)), sa(static_cast<std::size_t>(m) * 8),
        codes(static_cast<std::size_t>(k * n) * 2),
        scales(static_cast<std::size_t>(n * groups) * 8),
        ks(int_scales ? static_cast<std::size_t>(n * groups) * 4 : 0) {
    std::vector<std::int8_t> x8(static_cast<std::size_t>(m * k));
    for (Index i = 0; i < m * k; ++i) x8[i] = static_cast<std::int8_t>(x.values.data()[i]);
    up(xq, x8.data(), x8.size());
    up(sa, x.params.scales.data(), static_cast<std::size_t>(m));
    up(codes, wq.values.data(), static_cast<std::size_t>(k * n));
    up(scales, wq.params.scales.data(), static_cast<std::size_t>(n * groups));
    if (int_scales) up(ks, int_scales->data(), static_cast<std::size_t>(n * groups));
    check(isb_weight_pack_codes(codes.as<std::int16_t>(), k, n, g, scales.as<double>(),
                                int_scales ? ks.as<std::int32_t>() : nullptr, amp, nullptr, &w.h));
  }
};

// Exact int64 pass: output, doubles, partials and the reference statistics.
void run_checked(int path, Operands& o, bool strict, bool record, GemmResult& res) {
  Dev out(static_cast<std::size_t>(o.m * o.n) * 4), of(static_cast<std::size_t>(o.m * o.n) * 8);
  Dev part(record ? static_cast<std::size_t>(o.m * o.n * o.groups) * 8 : 0);
  isb_gemm_stats st{};
  check(isb_gemm_checked(path, o.xq.as<std::int8_t>(), o.sa.as<double>(), o.m, o.k, o.w.h,
                         strict ? 1 : 0, out.as<float>(), of.as<double>(), nullptr,
                         record ? part.as<std::int64_t>() : nullptr, &st, nullptr));
  res.output.resize(o.m, o.n);
  down(res.output.data(), out, static_cast<std::size_t>(o.m * o.n));
  if (record) {
    res.output_f64.resize(o.m, o.n);
    down(res.output_f64.data(), of, static_cast<std::size_t>(o.m * o.n));
    res.abs_group_partials.resize(o.m, o.n * o.groups);
    down(res.abs_group_partials.data(), part, static_cast<std::size_t>(o.m * o.n * o.groups));
    for (Index i = 0; i < res.abs_group_partials.size(); ++i)
      res.abs_group_partials.data()[i] = std::abs(res.abs_group_partials.data()[i]);
  }
  res.stats.max_abs_accumulator = st.max_abs_accumulator;
  res.stats.overflow_detected = st.overflow_detected != 0;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

// ---------------------------------------------------------------------------- quantize.hpp
void Granularity::validate(Index rows, Index cols) const {  // quantize.cpp:26-34
  if (rows < 1 || cols < 1) throw ParamError("shape must be at least 1x1");
  if (kind == GranKind::group) {
    if (group_size < 1) throw ParamError("group size must be >= 1");
    if (rows % group_size != 0)
      throw ParamError("group size " + std::to_string(group_size) +
                       " does not divide the reduction dimension " + std::to_string(rows));
  }
}

Index Granularity::unit_count(Index rows, Index cols) const {
  switch (kind) {
    case GranKind::per_tensor: return 1;
    case GranKind::per_token: return rows;
    case GranKind::per_channel: return cols;
    case GranKind::group: return cols * (rows / group_size);
  }
  throw ParamError("unknown granularity");
}

Index Granularity::unit_of(Index rows, Index r, Index c) const {
  switch (kind) {
    case GranKind::per_tensor: return 0;
    case GranKind::per_token: return r;
    case GranKind::per_channel: return c;
    case GranKind::group: return c * (rows / group_size) + r / group_size;
  }
  throw ParamError("unknown granularity");
}

std::int64_t QuantParams::qmin() const {
  return scheme == Scheme::symmetric ? -(std::int64_t{1} << (bit_width - 1)) : 0;
}
std::int64_t QuantParams::qmax() const {
  return scheme == Scheme::symmetric ? (std::int64_t{1} << (bit_width - 1)) - 1
                                     : (std::int64_t{1} << bit_width) - 1;
}

QuantizedTensor quantize(const MatF& x, int bit_width, Scheme scheme, const Granularity& g) {
  if (bit_width != 4 && bit_width != 8)
    throw ParamError("bit width must be 4 or 8, got " + std::to_string(bit_width));
  g.validate(x.rows(), x.cols());
  if (!all_finite(x)) throw ValueError("input has non-finite values");
  if (scheme != Scheme::symmetric)
    throw ParamError("the B200 path quantizes symmetric tensors only");
  const Index rows = x.rows(), cols = x.cols();
  QuantizedTensor q;
  q.params.bit_width = bit_width;
  q.params.scheme = scheme;
  q.params.granularity = g;
  q.values.resize(rows, cols);
  Dev dx(static_cast<std::size_t>(rows * cols) * 4);
  up(dx, x.data(), static_cast<std::size_t>(rows * cols));
  if (g.kind == GranKind::per_token && bit_width == 8) {  // K1
    Dev codes(static_cast<std::size_t>(rows * cols)), sc(static_cast<std::size_t>(rows) * 8);
    check(isb_quantize_per_token(dx.p, ISB_F32, rows, cols, codes.as<std::int8_t>(),
                                 sc.as<double>(), 1, nullptr));
    std::vector<std::int8_t> c8(static_cast<std::size_t>(rows * cols));
    down(c8.data(), codes, c8.size());
    for (Index i = 0; i < rows * cols; ++i) q.values.data()[i] = c8[i];
    q.params.scales.resize(rows);
    down(q.params.scales.data(), sc, static_cast<std::size_t>(rows));
    return q;
  }
  if (g.kind == GranKind::group || g.kind == GranKind::per_channel) {  // weights
    const Index gs = g.kind == GranKind::group ? g.group_size : rows;
    const Index units = cols * (rows / gs);
    Dev codes(static_cast<std::size_t>(rows * cols) * 2), sc(static_cast<std::size_t>(units) * 8);
    check(isb_quantize_weight_groups(dx.as<float>(), rows, cols, gs, bit_width,
                                     codes.as<std::int16_t>(), sc.as<double>(), nullptr));
    down(q.values.data(), codes, static_cast<std::size_t>(rows * cols));
    q.params.scales.resize(units);
    down(q.params.scales.data(), sc, static_cast<std::size_t>(units));
    return q;
  }
  throw ParamError("the B200 path quantizes per-token activations and group/per-channel weights");
}

// ---------------------------------------------------------------------------- integer_scale.hpp
int search_amplifier_exponent(const VecD& scales) {
  std::int32_t e = 0;
  check(isb_search_amplifier_exponent(scales.data(), scales.size(), &e));
  return e;
}

std::int64_t search_amplifier(const VecD& scales) {
  return std::int64_t{1} << search_amplifier_exponent(scales);
}

IntegerScaleSet integerize_scales(const VecD& scales, std::int64_t amplifier) {
  IntegerScaleSet s;
  s.int_scales.resize(scales.size());
  std::int32_t e = 0;
  check(isb_integerize_scales(scales.data(), scales.size(), amplifier, s.int_scales.data(), &e));
  s.amplifier = amplifier;
  s.exponent = e;
  return s;
}

// ---------------------------------------------------------------------------- tensor_io.hpp
std::vector<std::uint8_t> pack_signed4(const MatQ& values) {
  const Index rows = values.rows(), cols = values.cols();
  const Index n = rows * cols;
  std::vector<std::uint8_t> out(static_cast<std::size_t>((n + 1) / 2), 0);
  if (n == 0) return out;
  Dev codes(static_cast<std::size_t>(n) * 2), sc(static_cast<std::size_t>(cols) * 8);
  up(codes, values.data(), static_cast<std::size_t>(n));
  const std::vector<double> ones(static_cast<std::size_t>(cols), 1.0);
  up(sc, ones.data(), ones.size());
  Weight w;
  check(isb_weight_pack_codes(codes.as<std::int16_t>(), rows, cols, rows, sc.as<double>(), nullptr,
                              1, nullptr, &w.h));
  Dev bytes(out.size());
  check(isb_weight_repack_signed4(w.h, bytes.as<std::uint8_t>(), nullptr));
  down(out.data(), bytes, out.size());
  return out;
}

MatQ unpack_signed4(const std::vector<std::uint8_t>& bytes, Index rows, Index cols) {
  const Index n = rows * cols;
  if (static_cast<Index>(bytes.size()) != (n + 1) / 2)
    throw LengthError("packed payload is " + std::to_string(bytes.size()) + " bytes, expected " +
                      std::to_string((n + 1) / 2));
  MatQ v(rows, cols);
  Dev d(bytes.size()), sc(static_cast<std::size_t>(cols) * 8), codes(static_cast<std::size_t>(n) * 2);
  up(d, bytes.data(), bytes.size());
  const std::vector<double> ones(static_cast<std::size_t>(cols), 1.0);
  up(sc, ones.data(), ones.size());
  Weight w;
  check(isb_weight_pack_signed4(d.as<std::uint8_t>(), static_cast<std::int64_t>(bytes.size()), rows,
                                cols, rows, sc.as<double>(), nullptr, 1, nullptr, &w.h));
  check(isb_weight_unpack_codes(w.h, codes.as<std::int16_t>(), nullptr));
  down(v.data(), codes, static_cast<std::size_t>(n));
  return v;
}

// ---------------------------------------------------------------------------- analysis.hpp
OverflowReport overflow_analyzer(Index k, Index group_size, int act_bits, int weight_bits,
                                 const IntegerScaleSet& s) {
  OverflowReport r;
  std::int32_t safe = 0;
  check(isb_overflow_analyzer(k, group_size, act_bits, weight_bits, s.int_scales.data(),
                              s.int_scales.size(), &r.static_bound, &r.headroom_bits, &safe));
  r.safe = safe != 0;
  return r;
}

KernelStats expected_counters(PathKind path, Index m, Index n, Index k, Index group) {
  KernelStats s;  // analysis.cpp:129-153
  const Index groups = k / group;
  switch (path) {
    case PathKind::float_scale:
      s.int_to_float_conversions = m * n * groups;
      s.integer_multiply_adds = m * n * k;
      break;
    case PathKind::integer_scale:
      s.int_to_float_conversions = m * n;
      s.integer_multiply_adds = m * n * (k + groups);
      break;
    case PathKind::coarse:
      s.int_to_float_conversions = m * n;
      s.integer_multiply_adds = m * n * k;
      break;
    case PathKind::dual_quant:
      s.int_to_float_conversions = m * n * k;
      s.elementwise_multiplies = m * n * k;
      s.elementwise_subtractions = m * n * k;
      break;
  }
  return s;
}

// ---------------------------------------------------------------------------- gemm.hpp
std::string to_string(PathKind k) {
  switch (k) {
    case PathKind::float_scale: return "float-scale";
    case PathKind::integer_scale: return "integer-scale";
    case PathKind::coarse: return "coarse";
    case PathKind::dual_quant: return "dual-quant";
  }
  return "?";
}

PathKind path_from_string(const std::string& s) {
  if (s == "float-scale" || s == "float_scale") return PathKind::float_scale;
  if (s == "integer-scale" || s == "integer_scale") return PathKind::integer_scale;
  if (s == "coarse") return PathKind::coarse;
  if (s == "dual-quant" || s == "dual_quant") return PathKind::dual_quant;
  throw ParamError("unknown path '" + s + "'");
}

GemmResult gemm_float_scale(const QuantizedTensor& x, const QuantizedTensor& w,
                            const GemmOptions& opt) {
  validate_activation(x);
  const Index g = validate_grouped_weight(x, w);
  const double t0 = now_ms();
  Operands o(x, w, g, nullptr, 1);
  GemmResult res;
  run_checked(ISB_PATH_FLOAT_SCALE, o, opt.overflow == OverflowMode::strict, opt.record_partials,
              res);
  res.stats.int_to_float_conversions = o.m * o.n * o.groups;  // gemm.cpp:196
  res.stats.integer_multiply_adds = o.m * o.n * o.k;          // gemm.cpp:197
  res.stats.wall_ms = now_ms() - t0;
  return res;
}

GemmResult gemm_integer_scale(const QuantizedTensor& x, const QuantizedTensor& w,
                              const IntegerScaleSet& int_scales, const GemmOptions& opt) {
  validate_activation(x);
  const Index g = validate_grouped_weight(x, w);
  // gemm.cpp:212-216: the set must be exactly integerize_scales(w.scales, amplifier)
  const IntegerScaleSet expect = integerize_scales(w.params.scales, int_scales.amplifier);
  if (int_scales.exponent != expect.exponent ||
      int_scales.int_scales.size() != expect.int_scales.size() ||
      !std::equal(expect.int_scales.data(), expect.int_scales.data() + expect.int_scales.size(),
                  int_scales.int_scales.data()))
    throw ParamError("integer scales are not integerize_scales(weight scales, amplifier)");

  const double t0 = now_ms();
  Operands o(x, w, g, &int_scales.int_scales, int_scales.amplifier);
  const OverflowReport rep = overflow_analyzer(o.k, g, 8, 4, int_scales);
  const bool tc = g % 128 == 0 && o.k % 128 == 0 && rep.safe;
  const bool strict = opt.overflow == OverflowMode::strict;
  GemmResult res;
  res.stats.max_abs_accumulator = -1;
  if (opt.track_accumulator || strict || opt.record_partials || !tc)
    run_checked(ISB_PATH_INTEGER_SCALE, o, strict, opt.record_partials, res);
  if (tc) {  // tcgen05 K3 produces the output
    std::int64_t wsb = 0;
    check(isb_gemm_workspace_size(o.m, o.w.h, &wsb));
    Dev ws(static_cast<std::size_t>(std::max<std::int64_t>(wsb, 256)));
    cuda(cudaMemset(ws.p, 0, static_cast<std::size_t>(std::max<std::int64_t>(wsb, 256))), "memset");
    Dev out(static_cast<std::size_t>(o.m * o.n) * 4);
    check(isb_gemm_integer_scale(o.xq.as<std::int8_t>(), o.sa.as<double>(), o.m, o.k, o.w.h, out.p,
                                 ISB_F32, ws.p, std::max<std::int64_t>(wsb, 256), nullptr));
    MatF y(o.m, o.n);
    down(y.data(), out, static_cast<std::size_t>(o.m * o.n));
    if (res.output.size() && !(res.output == y))
      throw Error("tcgen05 integer-scale output disagrees with the exact int64 pass");
    res.output = std::move(y);
    res.stats.tensor_core = true;
  }
  res.stats.int_to_float_conversions = o.m * o.n;               // gemm.cpp:255
  res.stats.integer_multiply_adds = o.m * o.n * (o.k + o.groups);  // gemm.cpp:256
  res.stats.wall_ms = now_ms() - t0;
  return res;
}

GemmResult gemm_coarse(const QuantizedTensor& x, const QuantizedTensor& w,
                       const GemmOptions& opt) {  // gemm.cpp:264-309
  validate_activation(x);
  if (w.params.granularity.kind != GranKind::per_channel)
    throw ParamError("coarse path requires per-channel weights");  // gemm.cpp:267-268
  const Index g = validate_grouped_weight(x, w);
  const double t0 = now_ms();
  Operands o(x, w, g, nullptr, 1);
  GemmResult res;
  const bool strict = opt.overflow == OverflowMode::strict;
  const bool tc = o.k % 128 == 0;
  // One group per channel: the checked float path computes the same
  // double(acc) * s_w[j] * s_a[i] (gemm.cpp:190-194 with a single group).
  if (strict || opt.record_partials || opt.track_accumulator || !tc)
    run_checked(ISB_PATH_FLOAT_SCALE, o, strict, opt.record_partials, res);
  if (tc) {  // tcgen05: exact int32 sum over K, the reference's double epilogue
    Dev out(static_cast<std::size_t>(o.m * o.n) * 4);
    Dev ws(256);
    check(isb_gemm_coarse(o.xq.as<std::int8_t>(), o.sa.as<double>(), o.m, o.k, o.w.h, out.p,
                          ISB_F32, ws.p, 256, nullptr));
    MatF y(o.m, o.n);
    down(y.data(), out, static_cast<std::size_t>(o.m * o.n));
    if (res.output.size() && !(res.output == y))
      throw Error("tcgen05 coarse output disagrees with the exact int64 pass");
    res.output = std::move(y);
    res.stats.tensor_core = true;
  }
  res.stats.int_to_float_conversions = o.m * o.n;      // gemm.cpp:303
  res.stats.integer_multiply_adds = o.m * o.n * o.k;   // gemm.cpp:304
  res.stats.wall_ms = now_ms() - t0;
  return res;
}

DualInnerQuant dual_inner_quantize(const QuantizedTensor& w_outer, Index group_size) {
  if (w_outer.params.bit_width != 8 || w_outer.params.scheme != Scheme::symmetric ||
      w_outer.params.granularity.kind != GranKind::per_channel)
    throw ParamError("dual quantization layers over an 8-bit per-channel symmetric weight");
  if (group_size < 1 || w_outer.rows() % group_size != 0)
    throw ParamError("group size must divide the reduction dimension");
  const Index k = w_outer.rows(), n = w_outer.cols(), units = n * (k / group_size);
  Dev w8(static_cast<std::size_t>(k * n) * 2), codes(static_cast<std::size_t>(k * n) * 2),
      sc(static_cast<std::size_t>(units) * 8), zp(static_cast<std::size_t>(units) * 4);
  up(w8, w_outer.values.data(), static_cast<std::size_t>(k * n));
  check(isb_dual_inner_quantize(w8.as<std::int16_t>(), k, n, group_size, codes.as<std::int16_t>(),
                                sc.as<double>(), zp.as<std::int32_t>(), nullptr));
  DualInnerQuant inner;
  inner.group_size = group_size;
  inner.values.resize(k, n);
  inner.scales.resize(units);
  inner.zero_points.resize(units);
  down(inner.values.data(), codes, static_cast<std::size_t>(k * n));
  down(inner.scales.data(), sc, static_cast<std::size_t>(units));
  down(inner.zero_points.data(), zp, static_cast<std::size_t>(units));
  return inner;
}

GemmResult gemm_dual_quant(const QuantizedTensor& x, const QuantizedTensor& w_outer,
                           const DualInnerQuant& inner, const GemmOptions& opt) {
  validate_activation(x);  // gemm.cpp:349
  if (w_outer.params.bit_width != 8 || w_outer.params.scheme != Scheme::symmetric ||
      w_outer.params.granularity.kind != GranKind::per_channel)
    throw ParamError("dual-quant outer weight must be 8-bit per-channel symmetric");
  if (x.cols() != w_outer.rows())
    throw DimensionError("activation K=" + std::to_string(x.cols()) + " vs weight rows " +
                         std::to_string(w_outer.rows()));
  const Index m = x.rows(), k = x.cols(), n = w_outer.cols(), g = inner.group_size;
  if (g < 1 || k % g != 0) throw ParamError("inner group size must divide K");
  const Index units = n * (k / g);
  if (inner.values.rows() != k || inner.values.cols() != n)
    throw DimensionError("inner values shape does not match the outer weight");
  if (inner.scales.size() != units || inner.zero_points.size() != units)
    throw ParamError("inner parameter count does not match the grouping");
  if (w_outer.params.scales.size() != n) throw ParamError("outer scale count != channels");
  const double t0 = now_ms();
  std::vector<std::int8_t> x8(static_cast<std::size_t>(m * k));
  for (Index i = 0; i < m * k; ++i) x8[static_cast<std::size_t>(i)] = static_cast<std::int8_t>(x.values.data()[i]);
  Dev xq(x8.size()), sa(static_cast<std::size_t>(m) * 8), codes(static_cast<std::size_t>(k * n) * 2),
      sc(static_cast<std::size_t>(units) * 8), zp(static_cast<std::size_t>(units) * 4),
      so(static_cast<std::size_t>(n) * 8), out(static_cast<std::size_t>(m * n) * 4),
      of(opt.record_partials ? static_cast<std::size_t>(m * n) * 8 : 0);
  up(xq, x8.data(), x8.size());
  up(sa, x.params.scales.data(), static_cast<std::size_t>(m));
  up(codes, inner.values.data(), static_cast<std::size_t>(k * n));
  up(sc, inner.scales.data(), static_cast<std::size_t>(units));
  up(zp, inner.zero_points.data(), static_cast<std::size_t>(units));
  up(so, w_outer.params.scales.data(), static_cast<std::size_t>(n));
  check(isb_gemm_dual_quant(xq.as<std::int8_t>(), sa.as<double>(), m, k, codes.as<std::int16_t>(),
                            sc.as<double>(), zp.as<std::int32_t>(), g, so.as<double>(), n,
                            out.as<float>(), opt.record_partials ? of.as<double>() : nullptr, nullptr));
  GemmResult res;
  res.output.resize(m, n);
  down(res.output.data(), out, static_cast<std::size_t>(m * n));
  if (opt.record_partials) {
    res.output_f64.resize(m, n);
    down(res.output_f64.data(), of, static_cast<std::size_t>(m * n));
  }
  res.stats.int_to_float_conversions = m * n * k;  // gemm.cpp:405-407
  res.stats.elementwise_multiplies = m * n * k;
  res.stats.elementwise_subtractions = m * n * k;
  res.stats.max_abs_accumulator = 0;
  res.stats.wall_ms = now_ms() - t0;
  return res;
}

GemmResult run_layer(const QuantizedTensor& x, const QuantizedTensor& w, const PathConfig& path,
                     FallbackPolicy fallback, const GemmOptions& opt) {  // gemm.cpp:489-516
  switch (path.kind) {
    case PathKind::float_scale: return gemm_float_scale(x, w, opt);
    case PathKind::integer_scale: {
      if (!path.int_scales) throw ParamError("integer-scale path needs an IntegerScaleSet");
      if (fallback == FallbackPolicy::float_scale_on_overflow_risk) {
        const Index g = w.params.granularity.kind == GranKind::group
                            ? w.params.granularity.group_size
                            : w.rows();
        const OverflowReport report = overflow_analyzer(x.cols(), g, x.params.bit_width,
                                                        w.params.bit_width, *path.int_scales);
        if (!report.safe) {
          GemmResult res = gemm_float_scale(x, w, opt);
          res.stats.fallback_applied = true;
          return res;
        }
      }
      return gemm_integer_scale(x, w, *path.int_scales, opt);
    }
    case PathKind::coarse: return gemm_coarse(x, w, opt);
    case PathKind::dual_quant:
      if (!path.inner) throw ParamError("dual-quant path needs inner parameters");
      return gemm_dual_quant(x, w, *path.inner, opt);
    default:
      throw ParamError("path '" + to_string(path.kind) + "' is outside the B200 integer-scale path");
  }
}

// ---------------------------------------------------------------------------
// Device-resident entry points (include/intscale/gemm.hpp, namespace device).
namespace device {

PackedWeight::PackedWeight(const QuantizedTensor& w, const IntegerScaleSet* int_scales, void* stream) {
  const Index g = validate_weight(w);
  const Index k = w.rows(), n = w.cols(), groups = k / g;
  Dev codes(static_cast<std::size_t>(k * n) * 2), scales(static_cast<std::size_t>(n * groups) * 8),
      ks(int_scales ? static_cast<std::size_t>(n * groups) * 4 : 0);
  up(codes, w.values.data(), static_cast<std::size_t>(k * n));
  up(scales, w.params.scales.data(), static_cast<std::size_t>(n * groups));
  if (int_scales) {
    if (int_scales->int_scales.size() != n * groups)
      throw ParamError("integer scale count does not match the weight's groups");
    up(ks, int_scales->int_scales.data(), static_cast<std::size_t>(n * groups));
  }
  check(isb_weight_pack_codes(codes.as<std::int16_t>(), k, n, g, scales.as<double>(),
                              int_scales ? ks.as<std::int32_t>() : nullptr,
                              int_scales ? int_scales->amplifier : 1, stream, &h_));
  // the packer reads its inputs asynchronously: keep them alive until it has run
  cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "pack");
  k_ = k;
  n_ = n;
}

PackedWeight::~PackedWeight() { isb_weight_destroy(h_); }

PackedWeight::PackedWeight(PackedWeight&& o) noexcept : h_(o.h_), k_(o.k_), n_(o.n_) {
  o.h_ = nullptr;
}

PackedWeight& PackedWeight::operator=(PackedWeight&& o) noexcept {
  if (this != &o) {
    isb_weight_destroy(h_);
    h_ = o.h_;
    k_ = o.k_;
    n_ = o.n_;
    o.h_ = nullptr;
  }
  return *this;
}

void quantize_per_token(const float* x, Activations& out, void* stream) {
  check(isb_quantize_per_token(x, ISB_F32, out.m, out.k, out.codes, out.scales, 0, stream));
}

std::size_t workspace_bytes(Index m, const PackedWeight& w) {
  std::int64_t b = 0;
  check(isb_gemm_workspace_size(m, w.handle(), &b));
  return static_cast<std::size_t>(b);
}

void gemm_integer_scale(const Activations& x, const PackedWeight& w, void* out, OutType type,
                        void* workspace, std::size_t ws_bytes, void* stream) {
  check(isb_gemm_integer_scale(x.codes, x.scales, x.m, x.k, w.handle(), out,
                               static_cast<int>(type), workspace,
                               static_cast<std::int64_t>(ws_bytes), stream));
}

void gemm_float_scale(const Activations& x, const PackedWeight& w, void* out, OutType type,
                      void* workspace, std::size_t ws_bytes, void* stream) {
  check(isb_gemm_float_scale(x.codes, x.scales, x.m, x.k, w.handle(), out, static_cast<int>(type),
                             workspace, static_cast<std::int64_t>(ws_bytes), stream));
}

}  // namespace device

}  // namespace intscale
