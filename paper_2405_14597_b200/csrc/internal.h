// Internal declarations shared by the translation units of libintscale_b200.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/intscale_b200.h"

struct isb_weight {
  int64_t k = 0, n = 0, group = 0, groups = 0, amplifier = 1;
  int32_t exponent = 0;
  int32_t has_int_scales = 0;
  int32_t max_int_scale = 0;
  int64_t static_bound = 0;  // overflow_analyzer bound of the int scales (analysis.cpp:24-59)
  // fewest equal K-chunks (by groups) whose own bounds fit int32 (1 when static_bound does;
  // 0 when none up to kMaxChunks does): the exact tensor-core path for unsafe layers
  int32_t safe_chunks = 1;
  int64_t kblocks = 0;   // ceil(K / 128)
  int64_t n_tiles = 0;   // ceil(N / 128)
  uint8_t* packed = nullptr;        // n_tiles * kblocks * 8 KiB
  int32_t* kscale_tiled = nullptr;  // [n_tiles][groups][128] int32 (group % 128 == 0 only)
  float* fscale_tiled = nullptr;    // [n_tiles][groups][128] float(s) / 16
  int32_t* int_scales = nullptr;    // raw [N * groups] (reference unit order)
  double* scales = nullptr;         // raw [N * groups]
  int64_t packed_bytes = 0;
  bool tensor_core_ok() const { return group % 128 == 0 && k % 128 == 0; }
};

namespace isb {

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ISB_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void count_launch(int n = 1);
// Programmatic dependent launch on every kernel (env ISB_NO_PDL=1 disables; A/B only).
bool pdl_enabled();

// Kernel launchers (defined in the .cu files).
void launch_quantize_per_token(const void* x, int x_dtype, int64_t m, int64_t k, int8_t* codes,
                               double* scales, int* bad_flag, cudaStream_t s);
void launch_quantize_weight_groups(const float* w, int64_t k, int64_t n, int64_t group, int bits,
                                   int16_t* codes, double* scales, int* bad_flag, cudaStream_t s);
void launch_pack(const int16_t* codes, const uint8_t* signed4, int64_t k, int64_t n,
                 uint8_t* packed, int64_t kblocks, int64_t n_tiles, int* bad_flag, cudaStream_t s);
void launch_tile_scales(const int32_t* int_scales, const double* scales, int64_t n,
                        int64_t groups, int64_t n_tiles, int32_t* kscale, float* fscale,
                        cudaStream_t s);
void launch_unpack(const isb_weight& w, int16_t* codes, cudaStream_t s);
void launch_repack_signed4(const isb_weight& w, uint8_t* bytes, cudaStream_t s);

// Tensor-parallel helpers (tp.cu).
void launch_row_absmax(const void* x, int x_dtype, int64_t m, int64_t k, float* amax,
                       cudaStream_t s);
void launch_quantize_amax(const void* x, int x_dtype, int64_t m, int64_t k, const float* amax,
                          int8_t* codes, double* scales, cudaStream_t s);
void launch_finalize_chunks(int32_t* acc, int chunks, const double* sa, int64_t m, int64_t n,
                            double inv_amp, void* out, int out_dtype, cudaStream_t s);
void launch_finalize_acc(const int32_t* acc, const double* sa, int64_t m, int64_t n,
                         double inv_amp, void* out, int out_dtype, cudaStream_t s);

struct GemmPlan {
  int mt = 0;         // tokens per tile (UMMA N)
  int m_tiles = 0;
  int tiles = 0;
  int64_t units = 0;  // tiles * groups
  int grid = 0;
  int maxc = 1;       // max CTAs contributing to one tile
  int cluster = 1;    // split-K ways (thread-block cluster size)
  int64_t workspace_bytes = 0;
  bool fused = false; // per-token activation quantization fused into the GEMM (gemm_tc.cu XQ)
};
extern int64_t* g_trace;  // debug timeline buffer (8 x 512 int64), nullptr = off
extern int g_trace_cta;
extern int g_dbg;
GemmPlan plan_gemm(int64_t m, const isb_weight& w, int num_sms, int path, bool fused = false);
// Fused act-quant GEMM (decode M <= 64) possible for this weight (resident K slice fits).
bool act_fused_eligible(int64_t m, int64_t k, const isb_weight& w);
// 2-D TMA map over int8 activations [m][k], box 128 (K) x mt (rows), SWIZZLE_128B.
CUtensorMap make_x_map(const int8_t* xq, int64_t m, int64_t k, int mt);
// Prefill K3 with k_g folded into the weight expansion (gemm_fold.cu).
constexpr int64_t kFoldMinM = 256;
bool fold_eligible(int64_t m, const isb_weight& w, int path);
void launch_gemm_fold(const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                      void* out, int out_dtype, int num_sms, cudaStream_t s);
// Prefill K3 fold, CTA pair with tokens as the MMA M (gemm_sp.cu).
constexpr int kDbgFoldSS = 1 << 22;  // isb_debug_set_flags: force gemm_fold.cu at M >= 512 (A/B)
constexpr int64_t kSpMinM = 512;   // one pair tile = 512 tokens
constexpr int kSpTileTokens = 512;
void launch_gemm_sp(const int8_t* xq, const double* sa, int64_t m, const isb_weight& w, void* out,
                    int out_dtype, int num_sms, cudaStream_t s);
struct SpGroupPlan;
SpGroupPlan* sp_group_create(const isb_group_problem* probs, int nprob, int out_dtype, int num_sms);
void sp_group_run(SpGroupPlan* pl, cudaStream_t s);
double sp_group_balance(const SpGroupPlan* pl);
void sp_group_destroy(SpGroupPlan* pl);
// Prefill per-group-epilogue K3 (any k_g) / K4 on the SS skeleton (gemm_pg.cu).
constexpr int64_t kPgMinM = 128;
constexpr int kMaxChunks = 16;  // K-chunk limit of the exact tensor-core path for unsafe layers
bool pg_eligible(int64_t m, const isb_weight& w);
// kb0 / kbn: the 128-K blocks [kb0, kb0 + kbn) of the weight (kbn < 0: all), for the
// K-chunked exact path of unsafe layers (ISB_I32 raw chunk accumulators).
void launch_gemm_pg(int path, const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                    void* out, int out_dtype, int num_sms, cudaStream_t s, int64_t kb0 = 0,
                    int64_t kbn = -1);
// Dense fp16/bf16 baseline (gemm_f16.cu): out = x[M][K] * w[N][K]^T, K % 64 == 0.
void launch_gemm_dense(const void* x, const void* w, int64_t m, int64_t n, int64_t k, void* out,
                       int out_dtype, bool bf16, int num_sms, cudaStream_t s);
void launch_gemm_dense_i8(const void* x, const void* w, int64_t m, int64_t n, int64_t k, void* out,
                          int num_sms, cudaStream_t s);  // measurement only (SS int8 bound)
// Dual quantization comparison path (dual.cu, gemm.cpp:311-412).
void launch_dual_inner_quantize(const int16_t* w8, int64_t k, int64_t n, int64_t group,
                                int16_t* codes, double* scales, int32_t* zps, cudaStream_t s);
void validate_dual(const int8_t* xq, int64_t m, int64_t k, const int16_t* codes, int64_t n,
                   const int32_t* zps, const double* scales, int64_t group, cudaStream_t s);
void launch_gemm_dual_quant(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                            const int16_t* codes, const double* scales, const int32_t* zps,
                            int64_t group, const double* s_outer, int64_t n, float* out,
                            double* out_f64, cudaStream_t s);
void launch_gemm_tc(int path, const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                    void* out, int out_dtype, void* workspace, const GemmPlan& plan,
                    cudaStream_t s, const void* xf = nullptr, int x_dtype = 0,
                    double* sa_out = nullptr);
// The single-GEMM dispatch of isb_gemm_integer_scale / isb_gemm_float_scale (capi.cu).
int64_t gemm_workspace_size(int64_t m, const isb_weight& w);
void gemm_dispatch(int path, const int8_t* xq, const double* sa, int64_t m, const isb_weight& w,
                   void* out, int out_dtype, void* ws, int64_t ws_bytes, cudaStream_t s);
// Grouped layer launch (gemm_group.cu).
struct GroupPlan;
GroupPlan* group_plan_create(const isb_group_problem* probs, int nprob, int path, int out_dtype,
                             int num_sms);
void group_plan_run(GroupPlan* pl, cudaStream_t s);
void group_plan_info(const GroupPlan* pl, isb_group_info_t* info);
int group_plan_nonfinite(GroupPlan* pl, bool clear);
void group_plan_destroy(GroupPlan* pl);
void launch_gemm_checked(int path, const int8_t* xq, const double* sa, int64_t m,
                         const isb_weight& w, float* out, double* out_f64, int64_t* acc,
                         int64_t* partials, unsigned long long* stats_dev, cudaStream_t s);

}  // namespace isb
