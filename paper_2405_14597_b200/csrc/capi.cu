// extern "C" boundary of libintscale_b200 (include/intscale_b200.h). Maps
// failures onto the reference exception taxonomy (types.hpp:29-67) as status
// codes; the C++ drop-in layer turns them back into exceptions.
#include <atomic>
#include <bit>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return ISB_OK;
  } catch (const Failure& f) {
    g_err = f.what();
    return f.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ISB_ERROR;
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int num_sms() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (static_cast<int>(cache.size()) <= dev) cache.resize(dev + 1, 0);
  if (!cache[dev]) {
    cuda_check(cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev),
               "cudaDeviceGetAttribute");
  }
  return cache[dev];
}

// Per-device scratch int used as the "non-finite / bad code" flag when the
// caller does not ask for the check (written, never read).
int* scratch_flag() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static std::vector<int*> flags;
  std::lock_guard<std::mutex> lk(mu);
  if (static_cast<int>(flags.size()) <= dev) flags.resize(dev + 1, nullptr);
  if (!flags[dev]) cuda_check(cudaMalloc(&flags[dev], 64), "cudaMalloc(flag)");
  return flags[dev];
}

// Synchronous flag check for the offline / checked entry points.
struct DeviceFlag {
  int* d = nullptr;
  explicit DeviceFlag(cudaStream_t s) {
    cuda_check(cudaMalloc(&d, sizeof(int)), "cudaMalloc(flag)");
    cuda_check(cudaMemsetAsync(d, 0, sizeof(int), s), "cudaMemsetAsync");
  }
  ~DeviceFlag() { cudaFree(d); }
  bool raised(cudaStream_t s) {
    int h = 0;
    cuda_check(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s), "flag copy");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return h != 0;
  }
};

int exponent_of(int64_t amp) {
  if (amp < 1 || (amp & (amp - 1)) != 0)
    fail(ISB_PARAM, "amplifier must be a power of two >= 1, got " + std::to_string(amp));
  return std::countr_zero(static_cast<uint64_t>(amp));
}

void require_positive_scales(const double* s, int64_t n) {  // integer_scale.cpp:13-18
  if (n == 0) fail(ISB_PARAM, "scale list is empty");
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(s[i]) || s[i] <= 0.0)
      fail(ISB_PARAM, "scale " + std::to_string(i) + " is not a positive finite number");
}

isb_weight* pack_common(const int16_t* codes, const uint8_t* s4, int64_t k, int64_t n,
                        int64_t group, const double* scales, const int32_t* int_scales,
                        int64_t amplifier, cudaStream_t s) {
  if (k < 1 || n < 1) fail(ISB_PARAM, "shape must be at least 1x1");
  if (group < 1) fail(ISB_PARAM, "group size must be >= 1");
  if (k % group != 0)
    fail(ISB_PARAM, "group size " + std::to_string(group) +
                        " does not divide the reduction dimension " + std::to_string(k));
  if (!scales) fail(ISB_PARAM, "weight scales are required");
  auto* w = new isb_weight();
  try {
    w->k = k;
    w->n = n;
    w->group = group;
    w->groups = k / group;
    w->amplifier = int_scales ? amplifier : 1;
    w->exponent = int_scales ? exponent_of(amplifier) : 0;
    w->has_int_scales = int_scales != nullptr;
    w->kblocks = (k + kBlockK - 1) / kBlockK;
    w->n_tiles = (n + kTileN - 1) / kTileN;
    w->packed_bytes = w->n_tiles * w->kblocks * kBlockBytes;
    const int64_t units = n * w->groups;
    cuda_check(cudaMalloc(&w->packed, w->packed_bytes), "cudaMalloc(packed)");
    cuda_check(cudaMalloc(&w->scales, units * sizeof(double)), "cudaMalloc(scales)");
    cuda_check(cudaMemcpyAsync(w->scales, scales, units * sizeof(double), cudaMemcpyDefault, s),
               "copy scales");
    if (int_scales) {
      cuda_check(cudaMalloc(&w->int_scales, units * sizeof(int32_t)), "cudaMalloc(int_scales)");
      cuda_check(cudaMemcpyAsync(w->int_scales, int_scales, units * sizeof(int32_t),
                                 cudaMemcpyDefault, s),
                 "copy int scales");
      std::vector<int32_t> h(static_cast<size_t>(units));
      cuda_check(cudaMemcpyAsync(h.data(), int_scales, units * sizeof(int32_t), cudaMemcpyDefault,
                                 s),
                 "copy int scales to host");
      cuda_check(cudaStreamSynchronize(s), "sync");
      int32_t mx = 0;
      for (int32_t v : h) {
        if (v < 1) fail(ISB_PARAM, "integer scales must be >= 1");
        mx = std::max(mx, v);
      }
      w->max_int_scale = mx;
      // static bound max_col sum_g g*127*8*k_g (A_max 127, W_max 8), saturated
      int64_t worst = 0;
      for (int64_t c = 0; c < n; ++c) {
        int64_t col = 0;
        for (int64_t g = 0; g < w->groups; ++g) {
          col += group * 127 * 8 * static_cast<int64_t>(h[static_cast<size_t>(c * w->groups + g)]);
          if (col > (int64_t{1} << 62)) break;
        }
        worst = std::max(worst, col);
      }
      w->static_bound = worst;
      // K-chunking for unsafe layers: the fewest equal group ranges whose bounds fit int32
      w->safe_chunks = 1;
      if (worst > std::numeric_limits<int32_t>::max()) {
        w->safe_chunks = 0;
        for (int c = 2; c <= kMaxChunks && c <= w->groups; ++c) {
          int64_t wc = 0;
          for (int64_t col = 0; col < n && wc <= std::numeric_limits<int32_t>::max(); ++col)
            for (int q = 0; q < c; ++q) {
              int64_t b = 0;
              for (int64_t g = q * w->groups / c; g < (q + 1) * w->groups / c; ++g)
                b += group * 127 * 8 * static_cast<int64_t>(h[static_cast<size_t>(col * w->groups + g)]);
              wc = std::max(wc, b);
            }
          if (wc <= std::numeric_limits<int32_t>::max()) {
            w->safe_chunks = c;
            break;
          }
        }
      }
    }
    DeviceFlag bad(s);
    launch_pack(codes, s4, k, n, w->packed, w->kblocks, w->n_tiles, bad.d, s);
    if (w->tensor_core_ok()) {
      const int64_t tiled = w->n_tiles * w->groups * kTileN;
      cuda_check(cudaMalloc(&w->fscale_tiled, tiled * sizeof(float)), "cudaMalloc(fscale)");
      if (int_scales)
        cuda_check(cudaMalloc(&w->kscale_tiled, tiled * sizeof(int32_t)), "cudaMalloc(kscale)");
      launch_tile_scales(w->int_scales, w->scales, n, w->groups, w->n_tiles, w->kscale_tiled,
                         w->fscale_tiled, s);
    }
    if (bad.raised(s)) {
      if (codes) fail(ISB_VALUE, "weight codes outside signed 4-bit range [-8, 7]");
      fail(ISB_VALUE, "packed payload decodes outside [-8, 7]");
    }
  } catch (...) {
    isb_weight_destroy(w);
    throw;
  }
  return w;
}

// ISB_NO_FOLD=1 forces the per-group kernel at prefill sizes (A/B measurements).
bool fold_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("ISB_NO_FOLD");
    return e && e[0] == '1';
  }();
  return off;
}

// ISB_NO_PG=1 keeps prefill-M calls that cannot fold (k_g > 16, float scale) on the
// decode-family MT=128 kernel (A/B measurements).
bool pg_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("ISB_NO_PG");
    return e && e[0] == '1';
  }();
  return off;
}

int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }

// Unsafe layers (static bound > int32) on the integer path: K-chunk accumulators.
bool chunked_exact(const isb_weight& w) {
  return w.static_bound > std::numeric_limits<int32_t>::max() && w.safe_chunks > 1 &&
         w.tensor_core_ok() && w.group == kBlockK;
}

int64_t gemm_workspace_bytes(int64_t m, const isb_weight& w) {
  if (!w.tensor_core_ok()) return 0;
  int64_t b = std::max(plan_gemm(m, w, num_sms(), ISB_PATH_INTEGER_SCALE).workspace_bytes,
                       plan_gemm(m, w, num_sms(), ISB_PATH_FLOAT_SCALE).workspace_bytes);
  if (chunked_exact(w)) b = std::max<int64_t>(b, int64_t{w.safe_chunks} * m * w.n * 4);
  return b;
}

// act-fused two-kernel form: GEMM workspace, then s_a [m] doubles, then codes [m][k].
int64_t act_fused_workspace_bytes(int64_t m, const isb_weight& w) {
  return align256(gemm_workspace_bytes(m, w)) + align256(8 * m) + align256(m * w.k);
}

void require_gemm_args(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                       const isb_weight* w, int out_dtype) {
  if (!w) fail(ISB_PARAM, "null weight handle");
  if (!xq || !sa) fail(ISB_PARAM, "null activation pointer");
  if (m < 1) fail(ISB_PARAM, "shape must be at least 1x1");
  if (k != w->k)
    fail(ISB_DIMENSION,
         "activation K=" + std::to_string(k) + " vs weight rows " + std::to_string(w->k));
  if (out_dtype != ISB_F32 && out_dtype != ISB_BF16 && out_dtype != ISB_F16 &&
      out_dtype != ISB_I32)
    fail(ISB_PARAM, "unsupported output dtype");
}

// The tensor-core integer path accumulates sum_g P_g k_g in int32 (TMEM, registers,
// the int32 split-K exchange). That equals the reference's int64 acc only while
// overflow_analyzer's static bound fits int32 (analysis.cpp:24-59); otherwise the
// device sum could wrap where the reference flags / throws (gemm.cpp:42-52, :90-98).
// Unsafe layers run as K-chunks whose own bounds fit int32 (raw int32 accumulators per
// chunk, then an exact int64 sum + Eq. 2: finalize_chunks_kernel); only layers no split
// up to kMaxChunks makes safe, and raw int32 output (which cannot hold the sum), are
// refused with ISB_OVERFLOW (the exact scalar path is isb_gemm_checked).
void require_int32_safe(const isb_weight* w, int out_dtype) {
  if (w->static_bound > std::numeric_limits<int32_t>::max() &&
      (out_dtype == ISB_I32 || !chunked_exact(*w)))
    fail(ISB_OVERFLOW, "static overflow bound " + std::to_string(w->static_bound) +
                           " exceeds int32: the tensor-core integer-scale GEMM cannot be exact "
                           "for this layer (use isb_gemm_checked or the float-scale fallback)");
}

void gemm_tc(int path, const int8_t* xq, const double* sa, int64_t m, int64_t k,
             const isb_weight* w, void* out, int out_dtype, void* ws, int64_t ws_bytes,
             void* stream) {
  require_gemm_args(xq, sa, m, k, w, out_dtype);
  if (!w->tensor_core_ok())
    fail(ISB_PARAM, "tcgen05 path needs K % 128 == 0 and group % 128 == 0 (use isb_gemm_checked)");
  if (path == ISB_PATH_INTEGER_SCALE && !w->has_int_scales)
    fail(ISB_PARAM, "integer-scale path needs an IntegerScaleSet");
  if (out_dtype == ISB_I32 && path != ISB_PATH_INTEGER_SCALE)
    fail(ISB_PARAM, "raw int32 accumulator output exists only on the integer-scale path");
  if (path == ISB_PATH_INTEGER_SCALE) require_int32_safe(w, out_dtype);
  if (m > std::numeric_limits<int>::max() || w->n > std::numeric_limits<int>::max())
    fail(ISB_PARAM, "shape too large");
  if (path == ISB_PATH_INTEGER_SCALE && chunked_exact(*w)) {
    // the exact tensor-core path of an unsafe layer: C per-group-epilogue launches over
    // equal group ranges into int32 chunk accumulators, one int64 sum + Eq. 2 launch
    const int c = w->safe_chunks;
    const int64_t need = int64_t{c} * m * w->n * 4;
    if (!ws || ws_bytes < need)
      fail(ISB_PARAM, "workspace too small: need " + std::to_string(need) + " bytes");
    int32_t* acc = static_cast<int32_t*>(ws);
    for (int q = 0; q < c; ++q) {
      const int64_t g0 = q * w->groups / c, g1 = (q + 1) * w->groups / c;
      launch_gemm_pg(path, xq, sa, m, *w, acc + q * m * w->n, ISB_I32, num_sms(), as_stream(stream),
                     g0, g1 - g0);
    }
    launch_finalize_chunks(acc, c, sa, m, w->n, std::ldexp(1.0, -w->exponent), out, out_dtype,
                           as_stream(stream));
    return;
  }
  const GemmPlan pl = plan_gemm(m, *w, num_sms(), path);
  if (!ws || ws_bytes < pl.workspace_bytes)
    fail(ISB_PARAM, "workspace too small: need " + std::to_string(pl.workspace_bytes) + " bytes");
  if (fold_eligible(m, *w, path) && !fold_disabled()) {
    // 1-CTA SS kernel (gemm_fold.cu) by default; debug flag kDbgPair selects the CTA-pair
    // experiment (gemm_pair.cu) for A/B measurements in one process.
    // M >= 512: CTA-pair kernel with tokens as the MMA M (gemm_sp.cu); below, the 1-CTA
    // SS kernel (gemm_fold.cu; debug flag kDbgFoldSS forces it for A/B measurements).
    if (m >= kSpMinM && !(g_dbg & kDbgFoldSS))
      launch_gemm_sp(xq, sa, m, *w, out, out_dtype, num_sms(), as_stream(stream));
    else
      launch_gemm_fold(xq, sa, m, *w, out, out_dtype, num_sms(), as_stream(stream));
    return;
  }
  if (pg_eligible(m, *w) && !pg_disabled()) {  // prefill M: any k_g, and K4
    launch_gemm_pg(path, xq, sa, m, *w, out, out_dtype, num_sms(), as_stream(stream));
    return;
  }
  launch_gemm_tc(path, xq, sa, m, *w, out, out_dtype, ws, pl, as_stream(stream));
}

}  // namespace

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int64_t gemm_workspace_size(int64_t m, const isb_weight& w) { return gemm_workspace_bytes(m, w); }

void gemm_dispatch(int path, const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                   void* out, int out_dtype, void* ws, int64_t ws_bytes, cudaStream_t s) {
  gemm_tc(path, xq, sa, m, w.k, &w, out, out_dtype, ws, ws_bytes, s);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ISB_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

}  // namespace isb

using namespace isb;

extern "C" {

const char* isb_last_error(void) { return g_err.c_str(); }
int isb_version(void) { return 1; }
int64_t isb_launch_count(void) { return g_launches.load(); }

int isb_quantize_per_token(const void* x, int x_dtype, int64_t m, int64_t k, int8_t* codes,
                           double* scales, int check_finite, void* stream) {
  return guarded([&] {
    if (m < 1 || k < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    if (!x || !codes || !scales) fail(ISB_PARAM, "null pointer");
    cudaStream_t s = as_stream(stream);
    if (check_finite) {
      DeviceFlag bad(s);
      launch_quantize_per_token(x, x_dtype, m, k, codes, scales, bad.d, s);
      if (bad.raised(s)) fail(ISB_VALUE, "input has non-finite values");
    } else {
      launch_quantize_per_token(x, x_dtype, m, k, codes, scales, scratch_flag(), s);
    }
  });
}

int isb_quantize_weight_groups(const float* w, int64_t k, int64_t n, int64_t group,
                               int bit_width, int16_t* codes, double* scales, void* stream) {
  return guarded([&] {
    if (bit_width != 4 && bit_width != 8)
      fail(ISB_PARAM, "bit width must be 4 or 8, got " + std::to_string(bit_width));
    if (k < 1 || n < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    if (group < 1) fail(ISB_PARAM, "group size must be >= 1");
    if (k % group != 0)
      fail(ISB_PARAM, "group size " + std::to_string(group) +
                          " does not divide the reduction dimension " + std::to_string(k));
    cudaStream_t s = as_stream(stream);
    DeviceFlag bad(s);
    launch_quantize_weight_groups(w, k, n, group, bit_width, codes, scales, bad.d, s);
    if (bad.raised(s)) fail(ISB_VALUE, "input has non-finite values");
  });
}

int isb_weight_pack_codes(const int16_t* codes, int64_t k, int64_t n, int64_t group,
                          const double* scales, const int32_t* int_scales, int64_t amplifier,
                          void* stream, isb_weight** out) {
  return guarded([&] {
    if (!codes || !out) fail(ISB_PARAM, "null pointer");
    *out = pack_common(codes, nullptr, k, n, group, scales, int_scales, amplifier,
                       as_stream(stream));
  });
}

int isb_weight_pack_signed4(const uint8_t* bytes, int64_t nbytes, int64_t k, int64_t n,
                            int64_t group, const double* scales, const int32_t* int_scales,
                            int64_t amplifier, void* stream, isb_weight** out) {
  return guarded([&] {
    if (!bytes || !out) fail(ISB_PARAM, "null pointer");
    if (nbytes != (k * n + 1) / 2)  // unpack_signed4 contract, tensor_io.cpp:197-199
      fail(ISB_LENGTH, "packed payload is " + std::to_string(nbytes) + " bytes, expected " +
                           std::to_string((k * n + 1) / 2));
    *out = pack_common(nullptr, bytes, k, n, group, scales, int_scales, amplifier,
                       as_stream(stream));
  });
}

int isb_weight_unpack_codes(const isb_weight* w, int16_t* codes, void* stream) {
  return guarded([&] {
    if (!w || !codes) fail(ISB_PARAM, "null pointer");
    launch_unpack(*w, codes, as_stream(stream));
  });
}

int isb_weight_repack_signed4(const isb_weight* w, uint8_t* bytes, void* stream) {
  return guarded([&] {
    if (!w || !bytes) fail(ISB_PARAM, "null pointer");
    launch_repack_signed4(*w, bytes, as_stream(stream));
  });
}

int isb_weight_destroy(isb_weight* w) {
  if (!w) return ISB_OK;
  cudaFree(w->packed);
  cudaFree(w->kscale_tiled);
  cudaFree(w->fscale_tiled);
  cudaFree(w->int_scales);
  cudaFree(w->scales);
  delete w;
  return ISB_OK;
}

int isb_weight_info(const isb_weight* w, isb_weight_info_t* info) {
  return guarded([&] {
    if (!w || !info) fail(ISB_PARAM, "null pointer");
    info->k = w->k;
    info->n = w->n;
    info->group = w->group;
    info->groups = w->groups;
    info->amplifier = w->amplifier;
    info->exponent = w->exponent;
    info->has_int_scales = w->has_int_scales;
    info->packed_bytes = w->packed_bytes;
    info->scale_bytes = w->tensor_core_ok() ? w->n_tiles * w->groups * kTileN * 4 : 0;
    info->max_int_scale = w->max_int_scale;
    info->tensor_core_ok = w->tensor_core_ok() ? 1 : 0;
  });
}

int isb_gemm_workspace_size(int64_t m, const isb_weight* w, int64_t* bytes) {
  return guarded([&] {
    if (!w || !bytes) fail(ISB_PARAM, "null pointer");
    if (m < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    *bytes = gemm_workspace_bytes(m, *w);
  });
}

int isb_gemm_integer_scale(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                           const isb_weight* w, void* out, int out_dtype, void* workspace,
                           int64_t workspace_bytes, void* stream) {
  return guarded([&] {
    gemm_tc(ISB_PATH_INTEGER_SCALE, xq, sa, m, k, w, out, out_dtype, workspace, workspace_bytes,
            stream);
  });
}

int isb_gemm_float_scale(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                         const isb_weight* w, void* out, int out_dtype, void* workspace,
                         int64_t workspace_bytes, void* stream) {
  return guarded([&] {
    gemm_tc(ISB_PATH_FLOAT_SCALE, xq, sa, m, k, w, out, out_dtype, workspace, workspace_bytes,
            stream);
  });
}

int isb_gemm_coarse(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                    const isb_weight* w, void* out, int out_dtype, void* workspace,
                    int64_t workspace_bytes, void* stream) {
  return guarded([&] {
    require_gemm_args(xq, sa, m, k, w, out_dtype);
    if (out_dtype == ISB_I32) fail(ISB_PARAM, "unsupported output dtype");
    if (w->groups != 1)
      fail(ISB_PARAM, "coarse path requires per-channel weights");  // gemm.cpp:268
    if (!w->tensor_core_ok())
      fail(ISB_PARAM, "tcgen05 path needs K % 128 == 0 (use isb_gemm_checked)");
    if (m > std::numeric_limits<int>::max() || w->n > std::numeric_limits<int>::max())
      fail(ISB_PARAM, "shape too large");
    (void)workspace_bytes;
    const GemmPlan pl = plan_gemm(m, *w, num_sms(), ISB_PATH_COARSE);
    launch_gemm_tc(ISB_PATH_COARSE, xq, sa, m, *w, out, out_dtype, workspace, pl,
                   as_stream(stream));
  });
}

int isb_gemm_act_fused(int path, const void* x, int x_dtype, int64_t m, int64_t k,
                       const isb_weight* w, void* out, int out_dtype, double* sa_out,
                       void* workspace, int64_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!w) fail(ISB_PARAM, "null weight handle");
    if (!x || !out) fail(ISB_PARAM, "null pointer");
    if (m < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    if (k != w->k)
      fail(ISB_DIMENSION,
           "activation K=" + std::to_string(k) + " vs weight rows " + std::to_string(w->k));
    if (x_dtype != ISB_F32 && x_dtype != ISB_BF16)
      fail(ISB_PARAM, "activations must be float32 or bfloat16");
    if (path != ISB_PATH_INTEGER_SCALE && path != ISB_PATH_FLOAT_SCALE)
      fail(ISB_PARAM, "unknown path");
    if (path == ISB_PATH_INTEGER_SCALE && !w->has_int_scales)
      fail(ISB_PARAM, "integer-scale path needs an IntegerScaleSet");
    if (path == ISB_PATH_INTEGER_SCALE) require_int32_safe(w, out_dtype);
    if (out_dtype != ISB_F32 && out_dtype != ISB_BF16 && out_dtype != ISB_F16)
      fail(ISB_PARAM, "unsupported output dtype");
    cudaStream_t s = as_stream(stream);
    // K1 into the caller's workspace (after the GEMM's part), then the GEMM, PDL-chained:
    // faster than a single-GEMM kernel quantizing its own slice (15.2 vs 8.3 us at M = 16,
    // 4096 x 4096, scripts/fused_timing.py). The one-launch fused form is the grouped
    // layer launch (isb_group_plan_*), which amortizes the quantize phase over all linears.
    const int64_t gemm_ws = gemm_workspace_bytes(m, *w);
    if (!workspace || workspace_bytes < act_fused_workspace_bytes(m, *w))
      fail(ISB_PARAM, "workspace too small: need " +
                          std::to_string(act_fused_workspace_bytes(m, *w)) +
                          " bytes (isb_gemm_act_fused_workspace_size)");
    auto* base = static_cast<uint8_t*>(workspace);
    // the scales go straight to sa_out when the caller wants them (no copy node)
    double* sa = sa_out ? sa_out : reinterpret_cast<double*>(base + align256(gemm_ws));
    int8_t* codes = reinterpret_cast<int8_t*>(base + align256(gemm_ws) + align256(8 * m));
    launch_quantize_per_token(x, x_dtype, m, k, codes, sa, scratch_flag(), s);
    gemm_tc(path, codes, sa, m, k, w, out, out_dtype, workspace, gemm_ws, stream);
  });
}

int isb_gemm_act_fused_workspace_size(int64_t m, const isb_weight* w, int64_t* bytes) {
  return guarded([&] {
    if (!w || !bytes) fail(ISB_PARAM, "null pointer");
    if (m < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    *bytes = act_fused_workspace_bytes(m, *w);
  });
}

int isb_group_plan_create(const isb_group_problem* problems, int32_t nprob, int32_t path,
                          int32_t out_dtype, isb_group_plan** plan) {
  return guarded([&] {
    if (!plan) fail(ISB_PARAM, "null plan pointer");
    if (!problems) fail(ISB_PARAM, "null problem list");
    *plan = reinterpret_cast<isb_group_plan*>(
        group_plan_create(problems, nprob, path, out_dtype, num_sms()));
  });
}

int isb_group_run(isb_group_plan* plan, void* stream) {
  return guarded([&] {
    if (!plan) fail(ISB_PARAM, "null plan");
    group_plan_run(reinterpret_cast<GroupPlan*>(plan), as_stream(stream));
  });
}

int isb_group_plan_info(const isb_group_plan* plan, isb_group_info_t* info) {
  return guarded([&] {
    if (!plan || !info) fail(ISB_PARAM, "null argument");
    group_plan_info(reinterpret_cast<const GroupPlan*>(plan), info);
  });
}

int isb_group_nonfinite(isb_group_plan* plan, int32_t clear, int32_t* raised) {
  return guarded([&] {
    if (!plan || !raised) fail(ISB_PARAM, "null argument");
    *raised = group_plan_nonfinite(reinterpret_cast<GroupPlan*>(plan), clear != 0);
  });
}

int isb_group_plan_destroy(isb_group_plan* plan) {
  return guarded([&] { group_plan_destroy(reinterpret_cast<GroupPlan*>(plan)); });
}

int isb_gemm_dense(const void* x, const void* w, int dtype, int64_t m, int64_t n, int64_t k,
                   void* out, int out_dtype, void* stream) {
  return guarded([&] {
    if (!x || !w || !out) fail(ISB_PARAM, "null pointer");
    if (m < 1 || n < 1 || k < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    if (dtype != ISB_F16 && dtype != ISB_BF16) fail(ISB_PARAM, "dense inputs must be fp16 or bf16");
    if (out_dtype != ISB_F32 && out_dtype != ISB_BF16 && out_dtype != ISB_F16)
      fail(ISB_PARAM, "unsupported output dtype");
    if (k % 64 != 0) fail(ISB_PARAM, "dense GEMM needs K % 64 == 0");
    if (reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(w) % 16)
      fail(ISB_PARAM, "dense GEMM operands must be 16-byte aligned");
    if (m > std::numeric_limits<int>::max() || n > std::numeric_limits<int>::max())
      fail(ISB_PARAM, "shape too large");
    launch_gemm_dense(x, w, m, n, k, out, out_dtype, dtype == ISB_BF16, num_sms(), as_stream(stream));
  });
}

// Measurement only: the dense kernel's pipeline on kind::i8 (int8 x int8 -> float32),
// x [M][K], w [N][K], K % 128 == 0 — the SS-form upper bound for an int8 K3.
extern "C" int isb_debug_gemm_dense_i8(const void* x, const void* w, int64_t m, int64_t n,
                                       int64_t k, float* out, void* stream) {
  return guarded([&] {
    if (k % 128 != 0) fail(ISB_PARAM, "K % 128");
    launch_gemm_dense_i8(x, w, m, n, k, out, num_sms(), as_stream(stream));
  });
}

int isb_dual_inner_quantize(const int16_t* w8, int64_t k, int64_t n, int64_t group,
                            int16_t* codes, double* scales, int32_t* zero_points, void* stream) {
  return guarded([&] {
    if (!w8 || !codes || !scales || !zero_points) fail(ISB_PARAM, "null pointer");
    if (k < 1 || n < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    if (group < 1 || k % group != 0) fail(ISB_PARAM, "group size must divide the reduction dimension");
    launch_dual_inner_quantize(w8, k, n, group, codes, scales, zero_points, as_stream(stream));
  });
}

int isb_gemm_dual_quant(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                        const int16_t* codes, const double* scales, const int32_t* zero_points,
                        int64_t group, const double* outer_scales, int64_t n, float* out,
                        double* out_f64, void* stream) {
  return guarded([&] {
    if (!xq || !sa || !codes || !scales || !zero_points || !outer_scales || !out)
      fail(ISB_PARAM, "null pointer");
    if (m < 1 || k < 1 || n < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    if (group < 1 || k % group != 0) fail(ISB_PARAM, "inner group size must divide K");
    cudaStream_t s = as_stream(stream);
    validate_dual(xq, m, k, codes, n, zero_points, scales, group, s);
    launch_gemm_dual_quant(xq, sa, m, k, codes, scales, zero_points, group, outer_scales, n, out,
                           out_f64, s);
  });
}

int isb_finalize_acc(const int32_t* acc, const double* sa, int64_t m, int64_t n,
                     int64_t amplifier, void* out, int out_dtype, void* stream) {
  return guarded([&] {
    if (!acc || !sa || !out) fail(ISB_PARAM, "null pointer");
    if (m < 1 || n < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    if (out_dtype != ISB_F32 && out_dtype != ISB_BF16 && out_dtype != ISB_F16)
      fail(ISB_PARAM, "unsupported output dtype");
    const int e = exponent_of(amplifier);
    launch_finalize_acc(acc, sa, m, n, std::ldexp(1.0, -e), out, out_dtype, as_stream(stream));
  });
}

int isb_row_absmax(const void* x, int x_dtype, int64_t m, int64_t k, float* amax, void* stream) {
  return guarded([&] {
    if (!x || !amax) fail(ISB_PARAM, "null pointer");
    if (m < 1 || k < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    launch_row_absmax(x, x_dtype, m, k, amax, as_stream(stream));
  });
}

int isb_quantize_per_token_amax(const void* x, int x_dtype, int64_t m, int64_t k,
                                const float* amax, int8_t* codes, double* scales, void* stream) {
  return guarded([&] {
    if (!x || !amax || !codes || !scales) fail(ISB_PARAM, "null pointer");
    if (m < 1 || k < 1) fail(ISB_PARAM, "shape must be at least 1x1");
    launch_quantize_amax(x, x_dtype, m, k, amax, codes, scales, as_stream(stream));
  });
}

int isb_gemm_checked(int path, const int8_t* xq, const double* sa, int64_t m, int64_t k,
                     const isb_weight* w, int strict, float* out, double* out_f64, int64_t* acc,
                     int64_t* partials, isb_gemm_stats* stats, void* stream) {
  return guarded([&] {
    require_gemm_args(xq, sa, m, k, w, ISB_F32);
    if (path == ISB_PATH_INTEGER_SCALE && !w->has_int_scales)
      fail(ISB_PARAM, "integer-scale path needs an IntegerScaleSet");
    cudaStream_t s = as_stream(stream);
    unsigned long long* d = nullptr;
    cuda_check(cudaMalloc(&d, 3 * sizeof(unsigned long long)), "cudaMalloc(stats)");
    unsigned long long h[3] = {0ull, ~0ull, ~0ull};
    try {
      cuda_check(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, s), "stats init");
      launch_gemm_checked(path, xq, sa, m, *w, out, out_f64, acc, partials, d, s);
      cuda_check(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s), "stats copy");
      cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    } catch (...) {
      cudaFree(d);
      throw;
    }
    cudaFree(d);
    const int64_t n = w->n;
    isb_gemm_stats st{};
    st.max_abs_accumulator = static_cast<int64_t>(h[0]);
    st.overflow_detected = h[1] != ~0ull;
    st.hard_limit_hit = h[2] != ~0ull;
    st.overflow_i = st.overflow_detected ? static_cast<int64_t>(h[1]) / n : -1;
    st.overflow_j = st.overflow_detected ? static_cast<int64_t>(h[1]) % n : -1;
    if (stats) *stats = st;
    if (st.hard_limit_hit)  // gemm.cpp:49-51
      fail(ISB_ERROR, "accumulator exceeded the 64-bit safety margin at output (" +
                          std::to_string(static_cast<int64_t>(h[2]) / n) + ", " +
                          std::to_string(static_cast<int64_t>(h[2]) % n) + ")");
    if (st.overflow_detected && strict)  // gemm.cpp:96-98
      fail(ISB_OVERFLOW, "integer accumulation left the 32-bit window at output (" +
                             std::to_string(st.overflow_i) + ", " + std::to_string(st.overflow_j) +
                             ")");
  });
}

/* Debug: record a clock64 timeline of one CTA of subsequent tcgen05 GEMM launches
 * into trace (device, 8 x 512 int64; roles: 0 producer issue, 1 transform data
 * ready, 2 MMA commit, 3 transform A ready, 4 epilogue D ready, 5 producer start,
 * 6 CTA end, 7 CTA start). trace = NULL disables. Not part of the stable ABI. */
int isb_debug_set_trace(int64_t* trace, int cta) {
  g_trace = trace;
  g_trace_cta = cta;
  return ISB_OK;
}

int isb_debug_set_flags(int flags) {
  g_dbg = flags;
  return ISB_OK;
}

int isb_overflow_analyzer(int64_t k, int64_t group, int act_bits, int weight_bits,
                          const int32_t* int_scales, int64_t count, int64_t* static_bound,
                          double* headroom_bits, int32_t* safe) {
  // analysis.cpp:24-59
  return guarded([&] {
    if (act_bits != 4 && act_bits != 8) fail(ISB_PARAM, "activation bits must be 4 or 8");
    if (weight_bits != 4 && weight_bits != 8) fail(ISB_PARAM, "weight bits must be 4 or 8");
    if (k < 1 || group < 1 || k % group != 0) fail(ISB_PARAM, "group size must divide K");
    const int64_t groups = k / group;
    if (count < groups || count % groups != 0)
      fail(ISB_PARAM, "integer scale count incompatible with the grouping");
    for (int64_t i = 0; i < count; ++i)
      if (int_scales[i] < 1) fail(ISB_PARAM, "integer scales must be >= 1");
    const int64_t a_max = (int64_t{1} << (act_bits - 1)) - 1;
    const int64_t w_max = int64_t{1} << (weight_bits - 1);
    const auto per_mac = static_cast<unsigned __int128>(group) * a_max * w_max;
    unsigned __int128 worst = 0;
    for (int64_t c = 0; c < count / groups; ++c) {
      unsigned __int128 col = 0;
      for (int64_t g = 0; g < groups; ++g)
        col += per_mac * static_cast<unsigned __int128>(int_scales[c * groups + g]);
      worst = std::max(worst, col);
    }
    const auto cap = static_cast<unsigned __int128>(std::numeric_limits<int64_t>::max());
    const int64_t bound = worst > cap ? std::numeric_limits<int64_t>::max()
                                      : static_cast<int64_t>(worst);
    const int64_t hi = std::numeric_limits<int32_t>::max();
    if (static_bound) *static_bound = bound;
    if (safe) *safe = bound <= hi;
    if (headroom_bits)
      *headroom_bits = std::log2(static_cast<double>(hi)) - std::log2(static_cast<double>(bound));
  });
}

int isb_search_amplifier_exponent(const double* scales, int64_t count, int32_t* exponent) {
  // integer_scale.cpp:21-34: double min(s) until >= 1 (exact doublings).
  return guarded([&] {
    require_positive_scales(scales, count);
    double a = scales[0];
    for (int64_t i = 1; i < count; ++i) a = std::min(a, scales[i]);
    int e = 0;
    while (a < 1.0) {
      if (e >= 62) fail(ISB_PARAM, "smallest scale is too small to amplify");
      a *= 2.0;
      ++e;
    }
    *exponent = e;
  });
}

int isb_integerize_scales(const double* scales, int64_t count, int64_t amplifier,
                          int32_t* int_scales, int32_t* exponent) {
  // integer_scale.cpp:40-59: k = max(1, llround(s * amp)), OverflowError past int32.
  return guarded([&] {
    require_positive_scales(scales, count);
    const int e = exponent_of(amplifier);
    for (int64_t i = 0; i < count; ++i) {
      const int64_t kk = std::llround(scales[i] * static_cast<double>(amplifier));
      if (kk > std::numeric_limits<int32_t>::max())
        fail(ISB_OVERFLOW, "amplified scale " + std::to_string(i) +
                               " exceeds int32; amplifier too large for this scale set");
      int_scales[i] = static_cast<int32_t>(std::max<int64_t>(kk, 1));
    }
    *exponent = e;
  });
}

}  // extern "C"
