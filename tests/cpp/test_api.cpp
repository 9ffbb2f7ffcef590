// C++ drop-in tests: the reference's own hot-path test cases (proj/tests/*.cpp)
// run against the B200 library through the reference-signature C++ API
// (include/intscale/*.hpp). Cases cite the reference test they mirror. Needs a GPU.
#include <intscale/analysis.hpp>
#include <intscale/gemm.hpp>
#include <intscale/integer_scale.hpp>
#include <intscale/quantize.hpp>
#include <intscale/tensor_io.hpp>

#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>

#include <bit>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <random>
#include <string>
#include <vector>

using namespace intscale;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(c)) {                                                               \
      ++g_fail;                                                               \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);       \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    bool ok = false;                                                          \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const T&) {                                                      \
      ok = true;                                                              \
    } catch (...) {                                                           \
    }                                                                         \
    if (!ok) {                                                                \
      ++g_fail;                                                               \
      std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                         \
  } while (0)

static std::int64_t ulp_distance(float a, float b) {  // test_gemm.cpp:22-29
  if (a == b) return 0;
  auto key = [](float x) {
    auto u = std::bit_cast<std::int32_t>(x);
    return std::int64_t{u < 0 ? std::numeric_limits<std::int32_t>::min() - std::int64_t{u} : u};
  };
  return std::abs(key(a) - key(b));
}

static QuantizedTensor make_activation(std::initializer_list<std::initializer_list<int>> rows,
                                       std::initializer_list<double> scales) {
  QuantizedTensor t;
  t.values.resize(static_cast<Index>(rows.size()), static_cast<Index>(rows.begin()->size()));
  Index i = 0;
  for (auto& r : rows) {
    Index j = 0;
    for (int v : r) t.values(i, j++) = static_cast<std::int16_t>(v);
    ++i;
  }
  t.params.bit_width = 8;
  t.params.scheme = Scheme::symmetric;
  t.params.granularity = Granularity::per_token();
  t.params.scales.resize(static_cast<Index>(scales.size()));
  Index u = 0;
  for (double s : scales) t.params.scales[u++] = s;
  return t;
}

static QuantizedTensor make_weight(std::initializer_list<std::initializer_list<int>> rows,
                                   std::initializer_list<double> scales, int bits, Granularity g) {
  QuantizedTensor t = make_activation(rows, scales);
  t.params.bit_width = bits;
  t.params.granularity = g;
  return t;
}

static void test_scalar_hand_example() {  // test_gemm.cpp:94-118
  auto x = make_activation({{2, 3}}, {0.5});
  auto w = make_weight({{4}, {5}}, {0.25, 0.125}, 4, Granularity::group_of(1));
  auto rf = gemm_float_scale(x, w);
  CHECK(rf.output(0, 0) == 1.9375f);
  CHECK(rf.stats.int_to_float_conversions == 2);
  CHECK(rf.stats.integer_multiply_adds == 2);
  CHECK(rf.stats.max_abs_accumulator == 15);
  CHECK(!rf.stats.overflow_detected);
  auto set = integerize_scales(w.params.scales, 8);
  CHECK(set.int_scales[0] == 2);
  CHECK(set.int_scales[1] == 1);
  auto ri = gemm_integer_scale(x, w, set);
  CHECK(ri.output(0, 0) == 1.9375f);
  CHECK(ri.stats.int_to_float_conversions == 1);
  CHECK(ri.stats.integer_multiply_adds == 4);
  CHECK(ri.stats.max_abs_accumulator == 31);
}

static void test_unit_scales() {  // test_gemm.cpp:120-135
  auto x = make_activation({{1, 2, 3, 4}, {-1, 0, 1, 0}}, {1.0, 1.0});
  auto w = make_weight({{1, -1}, {2, 0}, {0, 3}, {-2, 1}}, {1.0, 1.0}, 4, Granularity::per_channel());
  auto rf = gemm_float_scale(x, w);
  CHECK(rf.output(0, 0) == -3.0f);
  CHECK(rf.output(0, 1) == 12.0f);
  CHECK(rf.output(1, 0) == -1.0f);
  CHECK(rf.output(1, 1) == 4.0f);
}

static void test_validation() {  // test_gemm.cpp:303-339
  auto x = make_activation({{1, 2}}, {1.0});
  auto w = make_weight({{1}, {1}}, {1.0}, 4, Granularity::group_of(1));
  CHECK_THROWS_AS(gemm_float_scale(x, w), ParamError);
  auto w3 = make_weight({{1}, {1}, {1}}, {1.0, 1.0, 1.0}, 4, Granularity::group_of(1));
  CHECK_THROWS_AS(gemm_float_scale(x, w3), DimensionError);
  auto wok = make_weight({{1}, {1}}, {1.0, 1.0}, 4, Granularity::group_of(1));
  auto xs = x;
  xs.params.granularity = Granularity::per_tensor();
  CHECK_THROWS_AS(gemm_float_scale(xs, wok), ParamError);
  auto x4 = x;
  x4.params.bit_width = 4;
  CHECK_THROWS_AS(gemm_float_scale(x4, wok), ParamError);
  auto xneg = make_activation({{-128, 0}}, {1.0});
  CHECK_THROWS_AS(gemm_float_scale(xneg, wok), ValueError);
  auto wbig = make_weight({{9}, {1}}, {1.0, 1.0}, 4, Granularity::group_of(1));
  CHECK_THROWS_AS(gemm_float_scale(x, wbig), ValueError);
  auto set = integerize_scales(wok.params.scales, 8);
  auto tampered = set;
  tampered.int_scales[0] += 1;
  CHECK_THROWS_AS(gemm_integer_scale(x, wok, tampered), ParamError);
}

static void test_overflow_rig() {  // test_gemm.cpp:345-407
  MatF xf = MatF::Constant(1, 4096, 127.0f);
  auto x = quantize(xf, 8, Scheme::symmetric, Granularity::per_token());
  MatF wf = MatF::Constant(4096, 2, -8.0f);
  auto w = quantize(wf, 4, Scheme::symmetric, Granularity::group_of(128));
  auto set = integerize_scales(w.params.scales, 1024);
  CHECK(x.params.scales[0] == 1.0);
  CHECK(w.values.minCoeff() == -7 && w.values.maxCoeff() == -7);
  CHECK(set.int_scales.minCoeff() == 1170 && set.int_scales.maxCoeff() == 1170);
  auto r = gemm_integer_scale(x, w, set);
  CHECK(r.stats.overflow_detected);
  CHECK(r.stats.max_abs_accumulator == std::int64_t{113792} * 1170 * 32);
  auto report = overflow_analyzer(4096, 128, 8, 4, set);
  CHECK(!report.safe);
  GemmOptions strict;
  strict.overflow = OverflowMode::strict;
  bool threw = false;
  try {
    gemm_integer_scale(x, w, set, strict);
  } catch (const OverflowError& e) {
    threw = std::string(e.what()).find("(0, 0)") != std::string::npos;
  }
  CHECK(threw);
  PathConfig path{PathKind::integer_scale, &set, nullptr};
  auto fb = run_layer(x, w, path, FallbackPolicy::float_scale_on_overflow_risk);
  CHECK(fb.stats.fallback_applied);
  auto rf = gemm_float_scale(x, w);
  CHECK(fb.output == rf.output);
  CHECK(fb.stats.int_to_float_conversions == 2 * 32);
  auto rn = run_layer(x, w, path, FallbackPolicy::none);
  CHECK(!rn.stats.fallback_applied && rn.stats.overflow_detected);
}

static void test_quantizer_pins() {  // test_quantize.cpp:92-97, :330-339
  MatF one(1, 1);
  one(0, 0) = 1.0f;
  auto q8 = quantize(one, 8, Scheme::symmetric, Granularity::per_token());
  CHECK(q8.params.scales[0] == 1.0 / 127.0);
  CHECK(q8.values(0, 0) == 127);
  MatF x(3, 2);
  x(0, 0) = 1.0f; x(0, 1) = -2.0f; x(1, 0) = 0.5f; x(1, 1) = 0.25f; x(2, 0) = 0.0f; x(2, 1) = 0.0f;
  auto q = quantize(x, 8, Scheme::symmetric, Granularity::per_token());
  CHECK(q.params.scales[0] == 2.0 / 127.0);
  CHECK(q.params.scales[1] == 0.5 / 127.0);
  CHECK(q.params.scales[2] == 1.0);
  CHECK(q.values(0, 1) == -127);
  MatF w1(2, 2);  // test_integer_scale.cpp:127-132 (ties away: -3.5 -> -4)
  w1(0, 0) = 0.875f; w1(0, 1) = 3.5f; w1(1, 0) = -0.4375f; w1(1, 1) = -1.75f;
  auto qw = quantize(w1, 4, Scheme::symmetric, Granularity::group_of(2));
  CHECK(qw.params.scales[0] == 0.125 && qw.params.scales[1] == 0.5);
  CHECK(qw.values(0, 0) == 7 && qw.values(1, 0) == -4 && qw.values(0, 1) == 7 && qw.values(1, 1) == -4);
}

static void test_integer_scale_pins() {  // test_integer_scale.cpp:26-66
  CHECK(search_amplifier(VecD{0.3, 0.9, 5.0}) == 4);
  CHECK(search_amplifier(VecD{0.5}) == 2);
  CHECK(search_amplifier(VecD{1.5, 2.0}) == 1);
  CHECK(search_amplifier(VecD{0x1.0p-10}) == 1024);
  CHECK(search_amplifier_exponent(VecD{0x1.0p-10, 0.25}) == 10);
  CHECK_THROWS_AS(search_amplifier(VecD{}), ParamError);
  CHECK_THROWS_AS(search_amplifier(VecD{1e-300}), ParamError);
  auto s = integerize_scales(VecD{0.25, 0.125}, 8);
  CHECK(s.amplifier == 8 && s.exponent == 3 && s.int_scales[0] == 2 && s.int_scales[1] == 1);
  CHECK(integerize_scales(VecD{0.0001}, 1024).int_scales[0] == 1);
  CHECK(integerize_scales(VecD{2.5 / 1024}, 1024).int_scales[0] == 3);
  CHECK_THROWS_AS(integerize_scales(VecD{0.5}, 3), ParamError);
  CHECK_THROWS_AS(integerize_scales(VecD{3.0e6}, 1024), OverflowError);
}

static void test_nibble_pins() {  // test_tensor_io.cpp:65-86
  MatQ v(1, 2);
  v(0, 0) = -8; v(0, 1) = 7;
  auto p = pack_signed4(v);
  CHECK(p.size() == 1 && p[0] == 0x78);
  CHECK(unpack_signed4(p, 1, 2) == v);
  MatQ v8(1, 8);
  const int vals[8] = {-8, -1, 0, 1, 2, -2, 7, -7};
  for (int i = 0; i < 8; ++i) v8(0, i) = static_cast<std::int16_t>(vals[i]);
  CHECK((pack_signed4(v8) == std::vector<std::uint8_t>{0xf8, 0x10, 0xe2, 0x97}));
  CHECK(unpack_signed4({0xf8, 0x10, 0xe2, 0x97}, 1, 8) == v8);
  MatQ bad(1, 1);
  bad(0, 0) = 8;
  CHECK_THROWS_AS(pack_signed4(bad), ValueError);
  CHECK_THROWS_AS(unpack_signed4({0xf8}, 1, 3), LengthError);
}

static void test_overflow_bound_pins() {  // test_analysis.cpp:33-62
  IntegerScaleSet one;
  one.int_scales = VecI{1};
  CHECK(overflow_analyzer(128, 128, 8, 4, one).static_bound == 130048);
  IntegerScaleSet s;
  s.int_scales = VecI::Constant(32, 1024);
  s.amplifier = 1024;
  s.exponent = 10;
  auto r = overflow_analyzer(4096, 128, 8, 4, s);
  CHECK(r.static_bound == 4261412864LL && !r.safe);
  IntegerScaleSet f;
  f.int_scales = VecI{1, 2, 3, 4};
  CHECK(overflow_analyzer(4, 2, 4, 4, f).static_bound == 784);
}

// acceptance.cpp:86-128 (criterion 1): dyadic scales => integer and float paths agree.
static void test_dyadic_agreement() {
  std::mt19937_64 rng(1001);
  auto below = [&](std::int64_t n) { return static_cast<std::int64_t>(rng() % n); };
  std::int64_t worst = 0;
  for (int trial = 0; trial < 40; ++trial) {
    const Index m = 1 + below(16), n = 1 + below(40), k = 4 * (1 + below(16));
    const Index g_choices[] = {1, 2, 4, k};
    const Index g = g_choices[below(4)];
    const Index units = (k / g) * n;
    VecD ws(units), xs(m);
    for (Index u = 0; u < units; ++u) ws[u] = double(1 + below(4096)) / 1024.0;
    for (Index i = 0; i < m; ++i) xs[i] = double(1 + below(1024)) / 256.0;
    QuantizedTensor x, w;
    x.values.resize(m, k);
    for (Index i = 0; i < m * k; ++i) x.values.data()[i] = static_cast<std::int16_t>(below(255) - 127);
    x.params = {8, Scheme::symmetric, Granularity::per_token(), xs, VecI()};
    w.values.resize(k, n);
    for (Index i = 0; i < k * n; ++i) w.values.data()[i] = static_cast<std::int16_t>(below(16) - 8);
    w.params = {4, Scheme::symmetric, Granularity::group_of(g), ws, VecI()};
    auto set = integerize_scales(ws, 1024);
    auto rf = gemm_float_scale(x, w);
    auto ri = gemm_integer_scale(x, w, set);
    for (Index i = 0; i < m * n; ++i)
      worst = std::max(worst, ulp_distance(rf.output.data()[i], ri.output.data()[i]));
  }
  CHECK(worst <= 1);
}

// A LLaMA-shaped layer goes through tcgen05 and matches the exact int64 pass.
static void test_coarse_equals_integer_at_alpha() {  // test_gemm.cpp:137-166
  std::mt19937_64 rng(17);
  auto u01 = [&] { return (rng() >> 11) * 0x1.0p-53; };
  const Index m = 3, k = 8, n = 4, g = 2;
  QuantizedTensor x;
  x.values.resize(m, k);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < k; ++j) x.values(i, j) = static_cast<std::int16_t>(rng() % 255) - 127;
  QuantizedTensor wg;
  wg.values.resize(k, n);
  for (Index i = 0; i < k; ++i)
    for (Index j = 0; j < n; ++j) wg.values(i, j) = static_cast<std::int16_t>(rng() % 16) - 8;
  x.params.bit_width = 8;
  x.params.scheme = Scheme::symmetric;
  x.params.granularity = Granularity::per_token();
  x.params.scales.resize(m);
  for (Index i = 0; i < m; ++i) x.params.scales[i] = 0.25 + u01();
  wg.params.bit_width = 4;
  wg.params.scheme = Scheme::symmetric;
  wg.params.granularity = Granularity::group_of(g);
  wg.params.scales = VecD::Constant((k / g) * n, 1.0);
  QuantizedTensor wc = wg;
  wc.params.granularity = Granularity::per_channel();
  wc.params.scales = VecD::Constant(n, 1.0);
  for (std::int64_t amp : {1, 8, 1024}) {
    auto set = integerize_scales(wg.params.scales, amp);
    auto ri = gemm_integer_scale(x, wg, set);
    auto rc = gemm_coarse(x, wc);
    CHECK(ri.output == rc.output);
  }
  CHECK_THROWS_AS(gemm_coarse(x, wg), ParamError);  // gemm.cpp:267-268
}

static void test_coarse_tensor_core() {
  std::mt19937_64 rng(5);
  auto u01 = [&] { return (rng() >> 11) * 0x1.0p-53; };
  const Index m = 7, k = 1024, n = 256;
  MatF wf(k, n), xf(m, k);
  for (Index i = 0; i < k * n; ++i) wf.data()[i] = static_cast<float>((2.0 * u01() - 1.0) * 0.01);
  for (Index i = 0; i < m * k; ++i) xf.data()[i] = static_cast<float>(4.0 * u01() - 2.0);
  auto w = quantize(wf, 4, Scheme::symmetric, Granularity::per_channel());
  auto x = quantize(xf, 8, Scheme::symmetric, Granularity::per_token());
  auto r = gemm_coarse(x, w);  // throws if the tcgen05 and exact outputs differ
  CHECK(r.stats.tensor_core);
  CHECK(r.stats.int_to_float_conversions == m * n);
}

static void test_tensor_core_layer() {
  std::mt19937_64 rng(42);
  auto u01 = [&] { return (rng() >> 11) * 0x1.0p-53; };
  const Index m = 16, k = 1024, n = 384;
  MatF wf(k, n), xf(m, k);
  for (Index c = 0; c < n; ++c)
    for (Index t = 0; t < k / 128; ++t) {
      const double vmax = 7.0 * std::exp2(-9.99 + 3.94 * u01());
      for (Index r = t * 128; r < (t + 1) * 128; ++r)
        wf(r, c) = static_cast<float>((2.0 * u01() - 1.0) * 0.97 * vmax);
      wf(t * 128, c) = static_cast<float>(vmax);
    }
  for (Index i = 0; i < m * k; ++i) xf.data()[i] = static_cast<float>(4.0 * u01() - 2.0);
  auto w = quantize(wf, 4, Scheme::symmetric, Granularity::group_of(128));
  auto x = quantize(xf, 8, Scheme::symmetric, Granularity::per_token());
  auto set = integerize_scales(w.params.scales, search_amplifier(w.params.scales));
  GemmOptions stats;
  stats.track_accumulator = true;  // opt-in second pass: tcgen05 output checked against int64
  auto r = gemm_integer_scale(x, w, set, stats);  // throws if tcgen05 and int64 outputs differ
  CHECK(r.stats.tensor_core);
  CHECK(r.stats.max_abs_accumulator > 0);
  auto r2 = gemm_integer_scale(x, w, set);  // default: tcgen05 only
  CHECK(r2.output == r.output);
  CHECK(r2.stats.max_abs_accumulator == -1);
}


// Device-resident overloads (include/intscale/gemm.hpp, namespace device): weight packed
// once, activations quantized and consumed in HBM, results equal the host-matrix calls.
static void test_device_entry_points() {
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  const Index m = 40, k = 512, n = 384;
  MatF wf(k, n), xf(m, k);
  for (Index i = 0; i < k * n; ++i) wf.data()[i] = static_cast<float>(0.02 * u(rng));
  for (Index i = 0; i < m * k; ++i) xf.data()[i] = static_cast<float>(2.0 * u(rng));
  auto w = quantize(wf, 4, Scheme::symmetric, Granularity::group_of(128));
  auto x = quantize(xf, 8, Scheme::symmetric, Granularity::per_token());
  auto set = integerize_scales(w.params.scales, 1024);
  const auto host_i = gemm_integer_scale(x, w, set);
  const auto host_f = gemm_float_scale(x, w);

  device::PackedWeight pw(w, &set);
  CHECK(pw.k() == k && pw.n() == n);
  float* xd = nullptr;
  device::Activations xa;
  xa.m = m;
  xa.k = k;
  void *out = nullptr, *ws = nullptr;
  const std::size_t wsb = std::max<std::size_t>(256, device::workspace_bytes(m, pw));
  cudaMalloc(reinterpret_cast<void**>(&xd), m * k * 4);
  cudaMalloc(reinterpret_cast<void**>(&xa.codes), m * k);
  cudaMalloc(reinterpret_cast<void**>(&xa.scales), m * 8);
  cudaMalloc(&out, m * n * 4);
  cudaMalloc(&ws, wsb);
  cudaMemset(ws, 0, wsb);
  cudaMemcpy(xd, xf.data(), m * k * 4, cudaMemcpyHostToDevice);
  device::quantize_per_token(xd, xa);
  std::vector<std::int8_t> codes(m * k);
  std::vector<double> scales(m);
  cudaMemcpy(codes.data(), xa.codes, m * k, cudaMemcpyDeviceToHost);
  cudaMemcpy(scales.data(), xa.scales, m * 8, cudaMemcpyDeviceToHost);
  bool same_codes = true;
  for (Index i = 0; i < m * k; ++i) same_codes &= codes[i] == x.values.data()[i];
  CHECK(same_codes);
  CHECK(std::equal(scales.begin(), scales.end(), x.params.scales.data()));
  MatF y(m, n);
  device::gemm_integer_scale(xa, pw, out, device::OutType::f32, ws, wsb);
  cudaMemcpy(y.data(), out, m * n * 4, cudaMemcpyDeviceToHost);
  CHECK(y == host_i.output);  // bit-identical
  device::gemm_float_scale(xa, pw, out, device::OutType::f32, ws, wsb);
  cudaMemcpy(y.data(), out, m * n * 4, cudaMemcpyDeviceToHost);
  double mag = 0.0, e2 = 0.0;
  for (Index i = 0; i < m * n; ++i) mag = std::max(mag, std::abs(double(host_f.output.data()[i])));
  for (Index i = 0; i < m * n; ++i)
    e2 = std::max(e2, std::abs(double(y.data()[i]) - double(host_f.output.data()[i])));
  CHECK(e2 <= 1e-4 * mag);  // fp32 group accumulation vs the reference's double
  device::PackedWeight moved = std::move(pw);
  CHECK(moved.handle() != nullptr && pw.handle() == nullptr);
  CHECK_THROWS_AS(device::gemm_integer_scale(xa, device::PackedWeight(w), out, device::OutType::f32,
                                             ws, wsb),
                  ParamError);  // no integer scales packed
  cudaFree(xd);
  cudaFree(xa.codes);
  cudaFree(xa.scales);
  cudaFree(out);
  cudaFree(ws);
}

// ------------------------------------------------------------------ QTNS container
namespace fs = std::filesystem;

struct TempDir {  // test_tensor_io.cpp:21-33
  fs::path path;
  explicit TempDir(const std::string& tag) {
    path = fs::temp_directory_path() / ("isb_io_" + tag + "_" + std::to_string(::getpid()));
    fs::create_directories(path);
  }
  ~TempDir() {
    std::error_code ec;
    fs::remove_all(path, ec);
  }
  std::string file(const std::string& name) const { return (path / name).string(); }
};

static std::vector<std::uint8_t> slurp(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  return std::vector<std::uint8_t>(std::istreambuf_iterator<char>(in), {});
}

static void spit(const std::string& p, const std::vector<std::uint8_t>& b) {
  std::ofstream out(p, std::ios::binary);
  out.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
}

static std::vector<std::uint8_t> header_bytes(std::uint8_t dtype, std::uint64_t rows,
                                              std::uint64_t cols) {
  std::vector<std::uint8_t> h = {'Q', 'T', 'N', 'S', 1, 0, dtype, 2};
  for (std::uint64_t d : {rows, cols})
    for (int b = 0; b < 8; ++b) h.push_back(static_cast<std::uint8_t>((d >> (8 * b)) & 0xff));
  return h;
}

static MatQ rowq(std::initializer_list<int> vals) {
  MatQ m(1, static_cast<Index>(vals.size()));
  Index j = 0;
  for (int v : vals) m(0, j++) = static_cast<std::int16_t>(v);
  return m;
}

static void test_qtns_containers() {  // test_tensor_io.cpp:88-161
  TempDir tmp("hdr");
  MatF z(1, 1);
  write_tensor(z, tmp.file("z.qtns"));
  auto expect = header_bytes(0, 1, 1);
  expect.insert(expect.end(), {0, 0, 0, 0});
  CHECK(slurp(tmp.file("z.qtns")) == expect);

  MatF x(2, 3);
  const float xv[] = {0.0f, -1.5f, 3.25e-3f, 1.0e30f, -1.0e-30f, 127.0f};
  for (int i = 0; i < 6; ++i) x.data()[i] = xv[i];
  write_tensor(x, tmp.file("x.qtns"));
  CHECK(read_float_tensor(tmp.file("x.qtns")) == x);

  MatQ q(2, 2);
  q(0, 0) = -128, q(0, 1) = 127, q(1, 0) = 0, q(1, 1) = -1;
  write_tensor(q, DType::signed8, tmp.file("q.qtns"));
  auto d8 = read_tensor(tmp.file("q.qtns"));
  auto* p8 = std::get_if<QuantizedPayload>(&d8);
  CHECK(p8 && p8->bit_width == 8 && p8->values == q);

  MatQ q4 = rowq({-8, 7, -1});
  write_tensor(q4, DType::packed_signed4, tmp.file("q4.qtns"));
  auto d4 = read_tensor(tmp.file("q4.qtns"));
  auto* p4 = std::get_if<QuantizedPayload>(&d4);
  CHECK(p4 && p4->bit_width == 4 && p4->values == q4);
  CHECK(fs::file_size(tmp.file("q4.qtns")) == 26);

  std::vector<std::uint8_t> v = {'Q', 'T', 'N', 'S', 1, 0, 1, 1, 5, 0, 0, 0, 0, 0, 0, 0,
                                 0x80, 0xff, 0x00, 0x01, 0x7f};
  spit(tmp.file("v.qtns"), v);
  auto dv = read_tensor(tmp.file("v.qtns"));
  auto* pv = std::get_if<QuantizedPayload>(&dv);
  CHECK(pv && pv->values.rows() == 1 && pv->values.cols() == 5);
  CHECK(pv && pv->values(0, 0) == -128 && pv->values(0, 1) == -1 && pv->values(0, 4) == 127);
}

static void test_qtns_malformed() {  // test_tensor_io.cpp:163-226
  TempDir tmp("bad");
  auto good = header_bytes(0, 1, 1);
  good.insert(good.end(), {0, 0, 0, 0});
  const std::string f = tmp.file("bad.qtns");
  auto with = [&](std::size_t i, std::uint8_t val) {
    auto b = good;
    b[i] = val;
    spit(f, b);
  };
  with(0, 'X');
  CHECK_THROWS_AS(read_tensor(f), FormatError);
  with(4, 2);
  CHECK_THROWS_AS(read_tensor(f), FormatError);
  with(6, 3);
  CHECK_THROWS_AS(read_tensor(f), FormatError);
  with(7, 3);
  CHECK_THROWS_AS(read_tensor(f), FormatError);
  spit(f, header_bytes(0, 0, 1));
  CHECK_THROWS_AS(read_tensor(f), FormatError);
  spit(f, std::vector<std::uint8_t>(good.begin(), good.end() - 1));
  CHECK_THROWS_AS(read_tensor(f), LengthError);
  spit(f, std::vector<std::uint8_t>(good.begin(), good.begin() + 10));
  CHECK_THROWS_AS(read_tensor(f), FormatError);
  auto trailing = good;
  trailing.push_back(0);
  spit(f, trailing);
  CHECK_THROWS_AS(read_tensor(f), LengthError);
  auto nan = header_bytes(0, 1, 1);
  nan.insert(nan.end(), {0x00, 0x00, 0xc0, 0x7f});
  spit(f, nan);
  CHECK_THROWS_AS(read_tensor(f), ValueError);
  CHECK_THROWS_AS(read_tensor(tmp.file("absent.qtns")), IoError);

  MatF xn(1, 1);
  xn(0, 0) = std::numeric_limits<float>::quiet_NaN();
  CHECK_THROWS_AS(write_tensor(xn, tmp.file("nan.qtns")), ValueError);
  MatQ big(1, 1);
  big(0, 0) = 200;
  CHECK_THROWS_AS(write_tensor(big, DType::signed8, tmp.file("big.qtns")), ValueError);
  big(0, 0) = 8;
  CHECK_THROWS_AS(write_tensor(big, DType::packed_signed4, tmp.file("big4.qtns")), ValueError);
  big(0, 0) = 1;
  CHECK_THROWS_AS(write_tensor(big, DType::real32, tmp.file("real.qtns")), ParamError);
}

static void test_quantized_sidecars() {  // test_quantize.cpp:284-328
  TempDir tmp("persist");
  std::mt19937_64 rng(9);
  auto u01 = [&] { return (rng() >> 11) * 0x1.0p-53; };
  MatF x(128, 4);
  for (Index i = 0; i < x.rows(); ++i)
    for (Index j = 0; j < x.cols(); ++j) x(i, j) = static_cast<float>(2.0 * u01() - 1.0);

  auto q = quantize(x, 4, Scheme::symmetric, Granularity::group_of(32));
  write_quantized(q, tmp.file("w.qtns"));
  CHECK(fs::exists(tmp.file("w.qtns") + ".json"));
  CHECK(fs::file_size(tmp.file("w.qtns")) == 24 + 256);
  auto back = read_quantized(tmp.file("w.qtns"));
  CHECK(back.values == q.values);
  CHECK(back.params.bit_width == 4);
  CHECK(back.params.scheme == Scheme::symmetric);
  CHECK(back.params.granularity.kind == GranKind::group);
  CHECK(back.params.granularity.group_size == 32);
  CHECK(back.params.scales == q.params.scales);

  // asymmetric codes (built by hand: the B200 quantizer is symmetric-only) survive
  // the signed container through the fold / unfold
  for (int bits : {4, 8}) {
    QuantizedTensor a;
    a.values.resize(3, 5);
    for (Index i = 0; i < a.values.size(); ++i)
      a.values.data()[i] = static_cast<std::int16_t>((i * 7) % (1 << bits));
    a.params.bit_width = bits;
    a.params.scheme = Scheme::asymmetric;
    a.params.granularity = Granularity::per_token();
    a.params.scales = VecD{0.5, 0.25, 1e-3};
    a.params.zero_points = VecI{1, 2, 3};
    write_quantized(a, tmp.file("a.qtns"));
    auto ab = read_quantized(tmp.file("a.qtns"));
    CHECK(ab.values == a.values);
    CHECK(ab.params.zero_points == a.params.zero_points);
    CHECK(ab.params.scales == a.params.scales);
  }

  const std::string side = tmp.file("w.qtns") + ".json";
  auto put = [&](const std::string& s) { spit(side, std::vector<std::uint8_t>(s.begin(), s.end())); };
  put("{not json");
  CHECK_THROWS_AS(read_quantized(tmp.file("w.qtns")), FormatError);
  put(R"({"bit_width": 8, "scheme": "symmetric", "granularity": {"kind": "group", "group_size": 32},
          "scales": [], "zero_points": []})");
  CHECK_THROWS_AS(read_quantized(tmp.file("w.qtns")), FormatError);
  put(R"({"bit_width": 4, "scheme": "skewed", "granularity": {"kind": "group", "group_size": 32},
          "scales": [], "zero_points": []})");
  CHECK_THROWS_AS(read_quantized(tmp.file("w.qtns")), ParamError);
  put(R"({"bit_width": 4, "scheme": "symmetric", "granularity": {"kind": "group", "group_size": 32},
          "scales": [1.0], "zero_points": []})");
  CHECK_THROWS_AS(read_quantized(tmp.file("w.qtns")), FormatError);
  fs::remove(side);
  CHECK_THROWS_AS(read_quantized(tmp.file("w.qtns")), IoError);
}

static void test_dual_quant() {  // test_gemm.cpp:183-226
  auto x = make_activation({{1}}, {1.0});
  QuantizedTensor w_outer = make_weight({{5}}, {1.0}, 8, Granularity::per_channel());
  DualInnerQuant inner;
  inner.group_size = 1;
  inner.values = w_outer.values;
  inner.scales = VecD::Constant(1, 0.5);
  inner.zero_points = VecI::Constant(1, 3);
  auto r = gemm_dual_quant(x, w_outer, inner);
  CHECK(r.output(0, 0) == 1.0f);
  CHECK(r.stats.int_to_float_conversions == 1);
  CHECK(r.stats.elementwise_multiplies == 1);
  CHECK(r.stats.elementwise_subtractions == 1);
  CHECK(r.stats.integer_multiply_adds == 0);
  CHECK(r.stats.max_abs_accumulator == 0);

  std::mt19937_64 rng(19);
  const Index m = 3, k = 8, n = 3;
  MatQ xq(m, k), wq(k, n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < k; ++j) xq(i, j) = static_cast<std::int16_t>(rng() % 255) - 127;
  for (Index i = 0; i < k; ++i)
    for (Index j = 0; j < n; ++j) wq(i, j) = static_cast<std::int16_t>(rng() % 16);
  QuantizedTensor x2;
  x2.values = xq;
  x2.params.bit_width = 8;
  x2.params.scheme = Scheme::symmetric;
  x2.params.granularity = Granularity::per_token();
  x2.params.scales = VecD::Constant(m, 0.125);
  QuantizedTensor outer2;
  outer2.values = wq;
  outer2.params.bit_width = 8;
  outer2.params.scheme = Scheme::symmetric;
  outer2.params.granularity = Granularity::per_channel();
  outer2.params.scales = VecD::Constant(n, 0.25);
  DualInnerQuant ident;
  ident.group_size = k;
  ident.values = wq;
  ident.scales = VecD::Ones(n);
  ident.zero_points = VecI::Zero(n);
  auto rd = gemm_dual_quant(x2, outer2, ident);
  // the coarse path's expression (gemm.cpp:293) on the host: the B200 coarse kernel
  // packs 4-bit weights, and this identity stage is over 8-bit codes in [0, 15]
  MatF rc(m, n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      std::int64_t acc = 0;
      for (Index kk = 0; kk < k; ++kk) acc += std::int64_t{xq(i, kk)} * std::int64_t{wq(kk, j)};
      rc(i, j) = static_cast<float>(static_cast<double>(acc) * 0.25 * 0.125);
    }
  CHECK(rd.output == rc);
  PathConfig pd{PathKind::dual_quant, nullptr, &ident};
  CHECK(run_layer(x2, outer2, pd, FallbackPolicy::none).output == rd.output);

  // dual_inner_quantize: codes in [0, 15]; groups straddling zero reconstruct within
  // half a step (test_gemm.cpp:228-250)
  MatF wf(16, 6);
  std::mt19937_64 r2(20);
  for (Index i = 0; i < wf.size(); ++i) wf.data()[i] = static_cast<float>(((r2() >> 11) * 0x1.0p-53) * 2.0 - 1.0);
  auto w8 = quantize(wf, 8, Scheme::symmetric, Granularity::per_channel());
  auto in = dual_inner_quantize(w8, 4);
  CHECK(in.values.minCoeff() >= 0 && in.values.maxCoeff() <= 15);
  CHECK(in.scales.size() == 24);
  for (Index j = 0; j < 6; ++j)
    for (Index t = 0; t < 4; ++t) {
      std::int16_t lo = 127, hi = -127;
      for (Index r = t * 4; r < t * 4 + 4; ++r) {
        lo = std::min(lo, w8.values(r, j));
        hi = std::max(hi, w8.values(r, j));
      }
      if (lo > 0 || hi < 0) continue;
      const Index u = j * 4 + t;
      for (Index r = t * 4; r < t * 4 + 4; ++r) {
        const double recon = (double(in.values(r, j)) - double(in.zero_points[u])) * in.scales[u];
        // half a step, up to the rounding of a code clamped at 15 (this synthetic
        // weight, unlike the reference's seed-20 instance, hits that edge)
        CHECK(std::abs(recon - double(w8.values(r, j))) <= in.scales[u] / 2 * (1 + 1e-12));
      }
    }
  QuantizedTensor w4 = make_weight({{1}}, {1.0}, 4, Granularity::per_channel());
  CHECK_THROWS_AS(dual_inner_quantize(w4, 1), ParamError);
}

int main() {
  const std::pair<const char*, std::function<void()>> tests[] = {
      {"scalar_hand_example", test_scalar_hand_example},
      {"unit_scales", test_unit_scales},
      {"validation", test_validation},
      {"overflow_rig", test_overflow_rig},
      {"quantizer_pins", test_quantizer_pins},
      {"integer_scale_pins", test_integer_scale_pins},
      {"nibble_pins", test_nibble_pins},
      {"overflow_bound_pins", test_overflow_bound_pins},
      {"dyadic_agreement", test_dyadic_agreement},
      {"tensor_core_layer", test_tensor_core_layer},
      {"device_entry_points", test_device_entry_points},
      {"coarse_equals_integer_at_alpha", test_coarse_equals_integer_at_alpha},
      {"coarse_tensor_core", test_coarse_tensor_core},
      {"qtns_containers", test_qtns_containers},
      {"qtns_malformed", test_qtns_malformed},
      {"quantized_sidecars", test_quantized_sidecars},
      {"dual_quant", test_dual_quant},
  };
  for (const auto& [name, fn] : tests) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
