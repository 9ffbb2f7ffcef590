// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference integer-scale W4A8 path
// (/root/reference/proj, arXiv 2405.14597 "Integer Scale"). It exists to
// CHECK the B200 product path; only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it. The product
// library (paper_2405_14597_b200/) never links, imports or calls this file.
//
// Parity pin: the reference cannot be compiled in this image (it needs Eigen3
// and its vendor/ headers, both absent — see DESIGN.md), so this restatement is
// pinned against every golden vector / known-answer test the reference's own
// tests hold for the path (tests/test_oracle_golden.py transcribes them with
// file:line citations).
//
// Every function cites the reference lines it restates. Build flags follow the
// reference (-O3 -DNDEBUG) plus -ffp-contract=off so `od += double(p)*s`
// (gemm.cpp:190) is not fused into an FMA.

#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

// Error taxonomy, types.hpp:29-67. Status codes are the ones the product C ABI
// uses (include/intscale_b200.h) so tests can compare error behaviour 1:1.
enum Status : int {
  OK = 0,
  PARAM = 1,
  DIMENSION = 2,
  VALUE = 3,
  OVERFLOW_ = 4,
  LENGTH = 5,
  FORMAT = 6,
  ERROR = 7,
};

struct OracleError : std::runtime_error {
  int code;
  OracleError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_last_error;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_last_error.clear();
    return OK;
  } catch (const OracleError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ERROR;
  }
}

[[noreturn]] void fail(int code, const std::string& msg) { throw OracleError(code, msg); }

using Index = std::int64_t;

// ---------------------------------------------------------------------------
// Generators, tensor_io.cpp:64-122 and :305-321. Draw order matters.

double u01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
double u01_open0(std::mt19937_64& rng) {
  return static_cast<double>((rng() >> 11) + 1) * 0x1.0p-53;
}
// Box-Muller, cosine branch only (tensor_io.cpp:70-76).
double gauss(std::mt19937_64& rng) {
  const double r = std::sqrt(-2.0 * std::log(u01_open0(rng)));
  return r * std::cos(2.0 * std::numbers::pi * u01(rng));
}

// ---------------------------------------------------------------------------
// Quantizer, quantize.cpp:26-145.

enum GranKind : int { PER_TENSOR = 0, PER_TOKEN = 1, PER_CHANNEL = 2, GROUP = 3 };
enum Scheme : int { SYMMETRIC = 0, ASYMMETRIC = 1 };

struct QParams {
  int bit_width;
  int scheme;
  int kind;
  Index group;
};

std::int64_t qmin(const QParams& p) {  // quantize.cpp:84-86
  return p.scheme == SYMMETRIC ? -(std::int64_t{1} << (p.bit_width - 1)) : 0;
}
std::int64_t qmax(const QParams& p) {  // quantize.cpp:88-91
  return p.scheme == SYMMETRIC ? (std::int64_t{1} << (p.bit_width - 1)) - 1
                               : (std::int64_t{1} << p.bit_width) - 1;
}

void gran_validate(const QParams& p, Index rows, Index cols) {  // quantize.cpp:26-34
  if (rows < 1 || cols < 1) fail(PARAM, "shape must be at least 1x1");
  if (p.kind == GROUP) {
    if (p.group < 1) fail(PARAM, "group size must be >= 1");
    if (rows % p.group != 0)
      fail(PARAM, "group size " + std::to_string(p.group) +
                      " does not divide the reduction dimension " + std::to_string(rows));
  }
}

Index unit_count(const QParams& p, Index rows, Index cols) {  // quantize.cpp:36-44
  switch (p.kind) {
    case PER_TENSOR: return 1;
    case PER_TOKEN: return rows;
    case PER_CHANNEL: return cols;
    case GROUP: return cols * (rows / p.group);
  }
  fail(PARAM, "unknown granularity");
}

Index unit_of(const QParams& p, Index rows, Index r, Index c) {  // quantize.cpp:46-54
  switch (p.kind) {
    case PER_TENSOR: return 0;
    case PER_TOKEN: return r;
    case PER_CHANNEL: return c;
    case GROUP: return c * (rows / p.group) + r / p.group;
  }
  fail(PARAM, "unknown granularity");
}

// quantize.cpp:93-145. Round half away from zero via llround; zero unit => s=1.
void quantize_impl(const float* x, Index rows, Index cols, const QParams& p, std::int16_t* codes,
                   double* scales, std::int32_t* zps) {
  if (p.bit_width != 4 && p.bit_width != 8)
    fail(PARAM, "bit width must be 4 or 8, got " + std::to_string(p.bit_width));
  gran_validate(p, rows, cols);
  for (Index i = 0; i < rows * cols; ++i)
    if (!std::isfinite(x[i])) fail(VALUE, "input has non-finite values");
  const Index units = unit_count(p, rows, cols);
  std::vector<double> umin(units, std::numeric_limits<double>::infinity());
  std::vector<double> umax(units, -std::numeric_limits<double>::infinity());
  for (Index r = 0; r < rows; ++r)
    for (Index c = 0; c < cols; ++c) {
      const Index u = unit_of(p, rows, r, c);
      const double v = x[r * cols + c];
      umin[u] = std::min(umin[u], v);
      umax[u] = std::max(umax[u], v);
    }
  const std::int64_t lo = qmin(p), hi = qmax(p);
  for (Index u = 0; u < units; ++u) {
    if (p.scheme == SYMMETRIC) {
      const double amax = std::max(std::abs(umin[u]), std::abs(umax[u]));
      scales[u] = amax == 0.0 ? 1.0 : amax / static_cast<double>(hi);
    } else {
      const double range = umax[u] - umin[u];
      const double s = range == 0.0 ? 1.0 : range / static_cast<double>(hi);
      scales[u] = s;
      zps[u] = static_cast<std::int32_t>(
          std::min(std::max<std::int64_t>(std::llround(-umin[u] / s), 0), hi));
    }
  }
  for (Index r = 0; r < rows; ++r)
    for (Index c = 0; c < cols; ++c) {
      const Index u = unit_of(p, rows, r, c);
      std::int64_t level = std::llround(static_cast<double>(x[r * cols + c]) / scales[u]);
      if (p.scheme == ASYMMETRIC) level += zps[u];
      codes[r * cols + c] = static_cast<std::int16_t>(std::min(std::max(level, lo), hi));
    }
}

// ---------------------------------------------------------------------------
// Integer scale, integer_scale.cpp:21-59.

void require_positive_scales(const double* s, Index n) {  // integer_scale.cpp:13-18
  if (n == 0) fail(PARAM, "scale list is empty");
  for (Index i = 0; i < n; ++i)
    if (!std::isfinite(s[i]) || s[i] <= 0.0)
      fail(PARAM, "scale " + std::to_string(i) + " is not a positive finite number");
}

int search_exponent(const double* s, Index n) {  // integer_scale.cpp:21-34
  require_positive_scales(s, n);
  const double smin = *std::min_element(s, s + n);
  int e = 0;
  double a = smin;
  while (a < 1.0) {
    if (e >= 62) fail(PARAM, "smallest scale is too small to amplify");
    a *= 2.0;
    ++e;
  }
  return e;
}

int integerize_impl(const double* s, Index n, std::int64_t amp, std::int32_t* out) {
  // integer_scale.cpp:40-59
  require_positive_scales(s, n);
  if (amp < 1 || (amp & (amp - 1)) != 0)
    fail(PARAM, "amplifier must be a power of two >= 1, got " + std::to_string(amp));
  for (Index i = 0; i < n; ++i) {
    const std::int64_t k = std::llround(s[i] * static_cast<double>(amp));
    if (k > std::numeric_limits<std::int32_t>::max())
      fail(OVERFLOW_, "amplified scale " + std::to_string(i) +
                          " exceeds int32; amplifier too large for this scale set");
    out[i] = static_cast<std::int32_t>(std::max<std::int64_t>(k, 1));
  }
  return std::countr_zero(static_cast<std::uint64_t>(amp));
}

// ---------------------------------------------------------------------------
// GEMM engine, gemm.cpp:17-134 (semantics) and :156-262 (paths).

constexpr std::int64_t kWindowLo = std::numeric_limits<std::int32_t>::min();
constexpr std::int64_t kWindowHi = std::numeric_limits<std::int32_t>::max();
constexpr std::int64_t kHardLimit = std::int64_t{1} << 62;

struct WorkerState {  // gemm.cpp:33-53
  std::int64_t max_abs = 0;
  bool overflow = false;
  Index ov_i = -1, ov_j = -1;
  void track(std::int64_t acc, Index i, Index j) {
    max_abs = std::max(max_abs, acc < 0 ? -acc : acc);
    if ((acc < kWindowLo || acc > kWindowHi) && !overflow) {
      overflow = true;
      ov_i = i;
      ov_j = j;
    }
    if (acc < -kHardLimit || acc > kHardLimit)
      fail(ERROR, "accumulator exceeded the 64-bit safety margin at output (" +
                      std::to_string(i) + ", " + std::to_string(j) + ")");
  }
};

}  // namespace

extern "C" {

// Mirrors KernelStats (gemm.hpp:44-61) plus the first overflow coordinate the
// reference only exposes through the strict-mode message (gemm.cpp:96-98).
struct OrStats {
  std::int64_t int_to_float_conversions;
  std::int64_t integer_multiply_adds;
  std::int64_t max_abs_accumulator;
  std::int32_t overflow_detected;
  std::int32_t fallback_applied;
  std::int64_t overflow_i;
  std::int64_t overflow_j;
  double wall_ms;
};

struct OrReport {  // analysis.hpp:25-30
  std::int64_t static_bound;
  std::int64_t observed_max;
  double headroom_bits;
  std::int32_t safe;
};

}  // extern "C"

namespace {

template <class Fn>
OrStats run_partitioned(Index m, int workers_in, int strict, const Fn& rows_fn) {
  // gemm.cpp:55-100: contiguous row blocks per std::thread, deterministic merge.
  const int workers = std::max(1, workers_in);
  std::vector<WorkerState> states(static_cast<std::size_t>(workers));
  if (workers == 1) {
    rows_fn(Index{0}, m, states[0]);
  } else {
    const Index chunk = (m + workers - 1) / workers;
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errors(static_cast<std::size_t>(workers));
    for (int w = 0; w < workers; ++w) {
      const Index lo = std::min<Index>(m, chunk * w);
      const Index hi = std::min<Index>(m, chunk * (w + 1));
      threads.emplace_back([&, w, lo, hi] {
        try {
          rows_fn(lo, hi, states[static_cast<std::size_t>(w)]);
        } catch (...) {
          errors[static_cast<std::size_t>(w)] = std::current_exception();
        }
      });
    }
    for (auto& t : threads) t.join();
    for (const auto& e : errors)
      if (e) std::rethrow_exception(e);
  }
  OrStats st{};
  Index ov_i = -1, ov_j = -1;
  for (const WorkerState& s : states) {
    st.max_abs_accumulator = std::max(st.max_abs_accumulator, s.max_abs);
    if (s.overflow && (ov_i < 0 || s.ov_i < ov_i || (s.ov_i == ov_i && s.ov_j < ov_j))) {
      ov_i = s.ov_i;
      ov_j = s.ov_j;
    }
    st.overflow_detected = st.overflow_detected || s.overflow;
  }
  st.overflow_i = ov_i;
  st.overflow_j = ov_j;
  if (st.overflow_detected && strict)
    fail(OVERFLOW_, "integer accumulation left the 32-bit window at output (" +
                        std::to_string(ov_i) + ", " + std::to_string(ov_j) + ")");
  return st;
}

std::int64_t abs_bound(const QParams& p) { return std::max(std::abs(qmin(p)), qmax(p)); }

void validate_activation(const std::int16_t* xv, Index m, Index k, const QParams& xp,
                         Index n_scales) {  // gemm.cpp:106-116
  if (xp.scheme != SYMMETRIC || xp.kind != PER_TOKEN)
    fail(PARAM, "activations must be symmetric per-token quantized");
  if (xp.bit_width != 8) fail(PARAM, "activations must be 8-bit");
  if (n_scales != m) fail(PARAM, "activation scale count != rows");
  const auto [mn, mx] = std::minmax_element(xv, xv + m * k);
  if (*mn < -qmax(xp) || *mx > qmax(xp))
    fail(VALUE, "activation codes outside max-based symmetric range");
}

Index validate_grouped_weight(Index kx, const std::int16_t* wv, Index k, Index n,
                              const QParams& wp, Index n_scales) {  // gemm.cpp:119-134
  if (kx != k)
    fail(DIMENSION,
         "activation K=" + std::to_string(kx) + " vs weight rows " + std::to_string(k));
  if (wp.scheme != SYMMETRIC) fail(PARAM, "weights must be symmetric");
  if (wp.kind != GROUP && wp.kind != PER_CHANNEL)
    fail(PARAM, "weights must be group or per-channel quantized");
  const auto [mn, mx] = std::minmax_element(wv, wv + k * n);
  if (*mn < qmin(wp) || *mx > qmax(wp)) fail(VALUE, "weight codes outside quantized range");
  const Index g = wp.kind == GROUP ? wp.group : k;
  gran_validate(wp, k, n);
  if (n_scales != (k / g) * n) fail(PARAM, "weight scale count does not match grouping");
  return g;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

extern "C" {

const char* or_last_error() { return g_last_error.c_str(); }

// Raw std::mt19937_64 stream, so Python tests can replay the reference tests'
// own draw sequences (test_gemm.cpp:76-90, acceptance.cpp:34-39).
void* or_rng_new(std::uint64_t seed) { return new std::mt19937_64(seed); }
void or_rng_next(void* h, std::int64_t n, std::uint64_t* out) {
  auto* r = static_cast<std::mt19937_64*>(h);
  for (std::int64_t i = 0; i < n; ++i) out[i] = (*r)();
}
void or_rng_free(void* h) { delete static_cast<std::mt19937_64*>(h); }
// glibc exp2, so test-side fixtures reproduce std::exp2 bit for bit.
double or_exp2(double x) { return std::exp2(x); }

int or_generate(int dist, std::int64_t rows, std::int64_t cols, double p0, double p1,
                std::uint64_t seed, float* out) {
  // generate_synthetic, tensor_io.cpp:305-321; dist 0 gaussian{p0}, 1 uniform{p0,p1}, 2 llama_like.
  return guarded([&] {
    if (rows < 1 || cols < 1) fail(PARAM, "shape must be at least 1x1");
    std::mt19937_64 rng(seed);
    if (dist == 0) {
      if (!(p0 > 0.0) || p0 > 1e30) fail(PARAM, "gaussian sigma must be in (0, 1e30]");
      for (Index i = 0; i < rows * cols; ++i) out[i] = static_cast<float>(p0 * gauss(rng));
    } else if (dist == 1) {
      if (!std::isfinite(p0) || !std::isfinite(p1) || p0 > p1)
        fail(PARAM, "uniform bounds must be finite with lo <= hi");
      if (std::abs(p0) > 1e30 || std::abs(p1) > 1e30) fail(PARAM, "uniform bounds out of range");
      if (p0 == p1) {  // tensor_io.cpp:86
        for (Index i = 0; i < rows * cols; ++i) out[i] = static_cast<float>(p0);
      } else {
        for (Index i = 0; i < rows * cols; ++i)
          out[i] = static_cast<float>(p0 + (p1 - p0) * u01(rng));
      }
    } else {
      // gen_llama_like, tensor_io.cpp:101-122 (column-major fill order).
      constexpr Index kGroup = 128;
      if (rows % kGroup != 0)
        fail(PARAM, "llama_like needs rows divisible by 128, got " + std::to_string(rows));
      const Index groups = rows / kGroup;
      for (Index c = 0; c < cols; ++c)
        for (Index t = 0; t < groups; ++t) {
          const bool floor_group = (c == 0 && t == 0);
          const double ulo = -9.99;
          const double uhi = floor_group ? -9.05 : -6.05;
          const double u = ulo + (uhi - ulo) * u01(rng);
          const float vmax = static_cast<float>(7.0 * std::exp2(u));
          const Index anchor = t * kGroup + static_cast<Index>(rng() % kGroup);
          const float sign = (rng() & 1) ? 1.0f : -1.0f;
          for (Index r = t * kGroup; r < (t + 1) * kGroup; ++r)
            out[r * cols + c] = static_cast<float>((2.0 * u01(rng) - 1.0) * 0.97 * vmax);
          out[anchor * cols + c] = sign * vmax;
        }
    }
  });
}

int or_quantize(const float* x, std::int64_t rows, std::int64_t cols, int bits, int scheme,
                int kind, std::int64_t group, std::int16_t* codes, double* scales,
                std::int32_t* zps) {
  return guarded([&] {
    QParams p{bits, scheme, kind, group};
    quantize_impl(x, rows, cols, p, codes, scales, zps);
  });
}

int or_unit_count(int kind, std::int64_t group, std::int64_t rows, std::int64_t cols,
                  std::int64_t* out) {
  return guarded([&] {
    QParams p{8, SYMMETRIC, kind, group};
    gran_validate(p, rows, cols);
    *out = unit_count(p, rows, cols);
  });
}

int or_search_amplifier_exponent(const double* s, std::int64_t n, int* exponent) {
  return guarded([&] { *exponent = search_exponent(s, n); });
}

int or_integerize_scales(const double* s, std::int64_t n, std::int64_t amp, std::int32_t* out,
                         int* exponent) {
  return guarded([&] { *exponent = integerize_impl(s, n, amp, out); });
}

// tensor_io.cpp:179-193
int or_pack_signed4(const std::int16_t* v, std::int64_t n, std::uint8_t* out) {
  return guarded([&] {
    std::memset(out, 0, static_cast<std::size_t>((n + 1) / 2));
    for (Index i = 0; i < n; ++i) {
      const int x = v[i];
      if (x < -8 || x > 7)
        fail(VALUE, "value " + std::to_string(x) + " outside signed 4-bit range");
      const auto nib = static_cast<std::uint8_t>(x & 0xf);
      if (i % 2 == 0)
        out[i / 2] = nib;
      else
        out[i / 2] |= static_cast<std::uint8_t>(nib << 4);
    }
  });
}

// tensor_io.cpp:195-208
int or_unpack_signed4(const std::uint8_t* bytes, std::int64_t nbytes, std::int64_t rows,
                      std::int64_t cols, std::int16_t* out) {
  return guarded([&] {
    const Index n = rows * cols;
    if (nbytes != (n + 1) / 2)
      fail(LENGTH, "packed payload is " + std::to_string(nbytes) + " bytes, expected " +
                       std::to_string((n + 1) / 2));
    for (Index i = 0; i < n; ++i) {
      const std::uint8_t b = bytes[i / 2];
      int x = (i % 2 == 0) ? (b & 0xf) : (b >> 4);
      if (x >= 8) x -= 16;
      out[i] = static_cast<std::int16_t>(x);
    }
  });
}

// gemm_integer_scale, gemm.cpp:205-262. x: m x k int16 codes + sa[m];
// w: k x n int16 codes (w_bits, w_kind, w_group) + w_scales ((k/g)*n) doubles;
// ks: int_scales ((k/g)*n) with amplifier amp. Outputs (nullable):
//   out f32 m x n, out_f64 m x n, acc int64 m x n (the scaled accumulator the
//   reference API cannot return), partials int64 m x (n*G) SIGNED P_g.
int or_gemm_integer_scale(int x_bits, int x_scheme, int x_kind, int w_scheme, const std::int16_t* xv, const double* sa, std::int64_t m,
                          std::int64_t kx, std::int64_t n_sa, const std::int16_t* wv,
                          std::int64_t k, std::int64_t n, int w_bits, int w_kind,
                          std::int64_t w_group, const double* w_scales, std::int64_t n_wscales,
                          const std::int32_t* ks, std::int64_t n_ks, std::int64_t amp,
                          int exponent, int strict, int workers, float* out, double* out_f64,
                          std::int64_t* acc_out, std::int64_t* partials, OrStats* stats) {
  return guarded([&] {
    const QParams xp{x_bits, x_scheme, x_kind, 0};
    const QParams wp{w_bits, w_scheme, w_kind, w_group};
    validate_activation(xv, m, kx, xp, n_sa);
    const Index g = validate_grouped_weight(kx, wv, k, n, wp, n_wscales);
    const Index groups = k / g;
    // Re-check int_scales == integerize_scales(w.scales, amp) (gemm.cpp:212-216).
    std::vector<std::int32_t> expect(static_cast<std::size_t>(n_wscales));
    const int e = integerize_impl(w_scales, n_wscales, amp, expect.data());
    if (exponent != e || n_ks != n_wscales || !std::equal(expect.begin(), expect.end(), ks))
      fail(PARAM, "integer scales are not integerize_scales(weight scales, amplifier)");

    const double t0 = now_ms();
    // W transpose inside the timer (gemm.cpp:226).
    std::vector<std::int16_t> wt(static_cast<std::size_t>(k * n));
    for (Index r = 0; r < k; ++r)
      for (Index c = 0; c < n; ++c) wt[c * k + r] = wv[r * n + c];
    const double ampd = static_cast<double>(amp);
    const std::int64_t p_worst = g * abs_bound(xp) * abs_bound(wp);
    const bool check_macs = p_worst > kWindowHi;

    OrStats st = run_partitioned(m, workers, strict, [&](Index lo, Index hi, WorkerState& ws) {
      for (Index i = lo; i < hi; ++i) {
        const std::int16_t* xr = xv + i * k;
        const double s_a = sa[i];
        for (Index j = 0; j < n; ++j) {
          const std::int16_t* wr = wt.data() + j * k;
          const std::int32_t* kk_s = ks + j * groups;
          std::int64_t acc = 0;
          for (Index gi = 0; gi < groups; ++gi) {
            std::int64_t p = 0;
            for (Index kk = gi * g; kk < (gi + 1) * g; ++kk) {
              p += std::int32_t{xr[kk]} * std::int32_t{wr[kk]};
              if (check_macs) ws.track(p, i, j);
            }
            ws.track(p, i, j);
            acc += p * std::int64_t{kk_s[gi]};
            ws.track(acc, i, j);
            if (partials) partials[i * (n * groups) + j * groups + gi] = p;
          }
          const double o = (static_cast<double>(acc) / ampd) * s_a;
          if (out) out[i * n + j] = static_cast<float>(o);
          if (out_f64) out_f64[i * n + j] = o;
          if (acc_out) acc_out[i * n + j] = acc;
        }
      }
    });
    st.wall_ms = now_ms() - t0;
    st.int_to_float_conversions = m * n;          // gemm.cpp:255
    st.integer_multiply_adds = m * n * (k + groups);  // gemm.cpp:256
    if (stats) *stats = st;
  });
}

// gemm_float_scale, gemm.cpp:156-203.
int or_gemm_float_scale(int x_bits, int x_scheme, int x_kind, int w_scheme, const std::int16_t* xv, const double* sa, std::int64_t m,
                        std::int64_t kx, std::int64_t n_sa, const std::int16_t* wv,
                        std::int64_t k, std::int64_t n, int w_bits, int w_kind,
                        std::int64_t w_group, const double* w_scales, std::int64_t n_wscales,
                        int strict, int workers, float* out, double* out_f64,
                        std::int64_t* partials, OrStats* stats) {
  return guarded([&] {
    const QParams xp{x_bits, x_scheme, x_kind, 0};
    const QParams wp{w_bits, w_scheme, w_kind, w_group};
    validate_activation(xv, m, kx, xp, n_sa);
    const Index g = validate_grouped_weight(kx, wv, k, n, wp, n_wscales);
    const Index groups = k / g;
    const double t0 = now_ms();
    std::vector<std::int16_t> wt(static_cast<std::size_t>(k * n));
    for (Index r = 0; r < k; ++r)
      for (Index c = 0; c < n; ++c) wt[c * k + r] = wv[r * n + c];
    const std::int64_t p_worst = g * abs_bound(xp) * abs_bound(wp);
    const bool check_macs = p_worst > kWindowHi;
    OrStats st = run_partitioned(m, workers, strict, [&](Index lo, Index hi, WorkerState& ws) {
      for (Index i = lo; i < hi; ++i) {
        const std::int16_t* xr = xv + i * k;
        const double s_a = sa[i];
        for (Index j = 0; j < n; ++j) {
          const std::int16_t* wr = wt.data() + j * k;
          const double* sw = w_scales + j * groups;
          double od = 0.0;
          for (Index gi = 0; gi < groups; ++gi) {
            std::int64_t p = 0;
            for (Index kk = gi * g; kk < (gi + 1) * g; ++kk) {
              p += std::int32_t{xr[kk]} * std::int32_t{wr[kk]};
              if (check_macs) ws.track(p, i, j);
            }
            ws.track(p, i, j);
            od += static_cast<double>(p) * sw[gi];
            if (partials) partials[i * (n * groups) + j * groups + gi] = p;
          }
          const double o = od * s_a;
          if (out) out[i * n + j] = static_cast<float>(o);
          if (out_f64) out_f64[i * n + j] = o;
        }
      }
    });
    st.wall_ms = now_ms() - t0;
    st.int_to_float_conversions = m * n * groups;  // gemm.cpp:196
    st.integer_multiply_adds = m * n * k;          // gemm.cpp:197
    if (stats) *stats = st;
  });
}

// gemm_oracle for the two fine-grained paths, gemm.cpp:414-449. path 0 float, 1 integer.
int or_gemm_oracle(int path, int x_bits, int x_scheme, int x_kind, int w_scheme, const std::int16_t* xv, const double* sa, std::int64_t m,
                   std::int64_t kx, std::int64_t n_sa, const std::int16_t* wv, std::int64_t k,
                   std::int64_t n, int w_bits, int w_kind, std::int64_t w_group,
                   const double* w_scales, std::int64_t n_wscales, std::int64_t amp, float* out) {
  return guarded([&] {
    const QParams xp{x_bits, x_scheme, x_kind, 0};
    const QParams wp{w_bits, w_scheme, w_kind, w_group};
    validate_activation(xv, m, kx, xp, n_sa);
    const Index g = validate_grouped_weight(kx, wv, k, n, wp, n_wscales);
    const Index groups = k / g;
    std::vector<std::int32_t> own;
    if (path == 1) {
      own.resize(static_cast<std::size_t>(n_wscales));
      integerize_impl(w_scales, n_wscales, amp, own.data());
    }
    for (Index i = 0; i < m; ++i)
      for (Index j = 0; j < n; ++j) {
        double od = 0.0;
        std::int64_t acc = 0;
        for (Index gi = 0; gi < groups; ++gi) {
          std::int64_t p = 0;
          for (Index kk = gi * g; kk < (gi + 1) * g; ++kk)
            p += std::int64_t{xv[i * k + kk]} * std::int64_t{wv[kk * n + j]};
          if (path == 1)
            acc += p * std::int64_t{own[static_cast<std::size_t>(j * groups + gi)]};
          else
            od += static_cast<double>(p) * w_scales[j * groups + gi];
        }
        if (path == 1) od = static_cast<double>(acc) / static_cast<double>(amp);
        out[i * n + j] = static_cast<float>(od * sa[i]);
      }
  });
}

// overflow_analyzer, analysis.cpp:24-59 (128-bit, saturated to int64).
int or_overflow_analyzer(std::int64_t k, std::int64_t g, int act_bits, int w_bits,
                         const std::int32_t* ks, std::int64_t n_ks, OrReport* r) {
  return guarded([&] {
    if (act_bits != 4 && act_bits != 8) fail(PARAM, "activation bits must be 4 or 8");
    if (w_bits != 4 && w_bits != 8) fail(PARAM, "weight bits must be 4 or 8");
    if (k < 1 || g < 1 || k % g != 0) fail(PARAM, "group size must divide K");
    const Index groups = k / g;
    if (n_ks < groups || n_ks % groups != 0)
      fail(PARAM, "integer scale count incompatible with the grouping");
    for (Index i = 0; i < n_ks; ++i)
      if (ks[i] < 1) fail(PARAM, "integer scales must be >= 1");
    const std::int64_t a_max = (std::int64_t{1} << (act_bits - 1)) - 1;
    const std::int64_t w_max = std::int64_t{1} << (w_bits - 1);
    const auto per_mac = static_cast<unsigned __int128>(g) * static_cast<unsigned __int128>(a_max) *
                         static_cast<unsigned __int128>(w_max);
    const Index columns = n_ks / groups;
    unsigned __int128 worst = 0;
    for (Index c = 0; c < columns; ++c) {
      unsigned __int128 col = 0;
      for (Index gi = 0; gi < groups; ++gi)
        col += per_mac * static_cast<unsigned __int128>(ks[c * groups + gi]);
      worst = std::max(worst, col);
    }
    const auto cap = static_cast<unsigned __int128>(std::numeric_limits<std::int64_t>::max());
    r->static_bound = worst > cap ? std::numeric_limits<std::int64_t>::max()
                                  : static_cast<std::int64_t>(worst);
    r->observed_max = 0;
    r->safe = r->static_bound <= kWindowHi;
    r->headroom_bits = std::log2(static_cast<double>(kWindowHi)) -
                       std::log2(static_cast<double>(r->static_bound));
  });
}

// expected_counters, analysis.cpp:129-153. path 0 float, 1 integer, 2 coarse, 3 dual.
void or_expected_counters(int path, std::int64_t m, std::int64_t n, std::int64_t k,
                          std::int64_t g, std::int64_t* conversions, std::int64_t* imads) {
  const Index groups = k / g;
  switch (path) {
    case 0: *conversions = m * n * groups; *imads = m * n * k; break;
    case 1: *conversions = m * n; *imads = m * n * (k + groups); break;
    case 2: *conversions = m * n; *imads = m * n * k; break;
    default: *conversions = m * n * k; *imads = 0; break;
  }
}

// dual_inner_quantize, gemm.cpp:311-345: asymmetric 4-bit group quantization of an
// 8-bit per-channel weight's integer codes. w8 K x N row-major; unit u = j*G + t.
int or_dual_inner_quantize(const std::int16_t* w8, std::int64_t k, std::int64_t n,
                           std::int64_t group, std::int16_t* codes, double* scales,
                           std::int32_t* zps) {
  return guarded([&] {
    if (group < 1 || k % group != 0) fail(PARAM, "group size must divide the reduction dimension");
    const Index groups = k / group;
    for (Index j = 0; j < n; ++j)
      for (Index t = 0; t < groups; ++t) {
        double lo = std::numeric_limits<double>::infinity(), hi = -lo;
        for (Index r = t * group; r < (t + 1) * group; ++r) {
          lo = std::min(lo, static_cast<double>(w8[r * n + j]));
          hi = std::max(hi, static_cast<double>(w8[r * n + j]));
        }
        const double sc = hi == lo ? 1.0 : (hi - lo) / 15.0;
        const auto z = static_cast<std::int32_t>(std::clamp<std::int64_t>(std::llround(-lo / sc), 0, 15));
        scales[j * groups + t] = sc;
        zps[j * groups + t] = z;
        for (Index r = t * group; r < (t + 1) * group; ++r) {
          const std::int64_t q = std::llround(static_cast<double>(w8[r * n + j]) / sc) + z;
          codes[r * n + j] = static_cast<std::int16_t>(std::clamp<std::int64_t>(q, 0, 15));
        }
      }
  });
}

// gemm_dual_quant, gemm.cpp:347-412 (after validation): per output a sequential
// double accumulation cd += double(x) * ((double)(w - z) * s_i) over k in order,
// then out = float(cd * s_outer[j] * s_a[i]) (-ffp-contract=off: no FMA).
int or_gemm_dual_quant(const std::int16_t* x, const double* sa, std::int64_t m, std::int64_t k,
                       const std::int16_t* codes, const double* scales, const std::int32_t* zps,
                       std::int64_t group, const double* s_outer, std::int64_t n, float* out,
                       double* out_f64) {
  return guarded([&] {
    if (group < 1 || k % group != 0) fail(PARAM, "inner group size must divide K");
    const Index groups = k / group;
    for (Index i = 0; i < m; ++i)
      for (Index j = 0; j < n; ++j) {
        double cd = 0.0;
        for (Index gi = 0; gi < groups; ++gi) {
          const double si = scales[j * groups + gi];
          const std::int32_t z = zps[j * groups + gi];
          for (Index kk = gi * group; kk < (gi + 1) * group; ++kk) {
            const double wrec = static_cast<double>(std::int32_t{codes[kk * n + j]} - z) * si;
            cd += static_cast<double>(x[i * k + kk]) * wrec;
          }
        }
        const double o = cd * s_outer[j] * sa[i];
        out[i * n + j] = static_cast<float>(o);
        if (out_f64) out_f64[i * n + j] = o;
      }
  });
}

}  // extern "C"
