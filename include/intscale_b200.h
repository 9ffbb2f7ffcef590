/*
 * intscale_b200 — C ABI of the B200 (sm_100a) integer-scale W4A8 path.
 *
 * The reference (arXiv 2405.14597, /root/reference/proj) exposes its hot path
 * as C++ free functions in namespace intscale (no FFI, no plugin registry). Each
 * entry point below names the reference interface it replaces (file:line). The
 * C++ drop-in layer (include/intscale/ headers) re-exposes the reference
 * signatures on top of this ABI; the Python mirror binds it with ctypes.
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers unless the name says _host.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls are stream-ordered and asynchronous unless documented otherwise,
 *    reentrant, and never allocate device memory on the hot path (the GEMM
 *    workspace is caller-owned; see isb_gemm_workspace_size).
 *  - Return value: ISB_OK or an error code mapping 1:1 onto the reference
 *    exception types (types.hpp:29-67); isb_last_error() gives the message
 *    (thread-local).
 *  - Data layouts are the reference's: activations row-major M x K, weights
 *    row-major K x N (quantize.hpp:128-134, gemm.cpp:226), group scales with
 *    unit = n * (K/g) + k/g (quantize.cpp:51), outputs row-major M x N.
 */
#ifndef INTSCALE_B200_H_
#define INTSCALE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum isb_status {
  ISB_OK = 0,
  ISB_PARAM = 1,     /* ParamError      types.hpp:55 */
  ISB_DIMENSION = 2, /* DimensionError  types.hpp:50 */
  ISB_VALUE = 3,     /* ValueError      types.hpp:44 */
  ISB_OVERFLOW = 4,  /* OverflowError   types.hpp:61 */
  ISB_LENGTH = 5,    /* LengthError     types.hpp:39 */
  ISB_FORMAT = 6,    /* FormatError     types.hpp:34 */
  ISB_ERROR = 7,     /* Error           types.hpp:29 */
  ISB_CUDA = 8       /* CUDA runtime / launch failure (no reference analogue) */
};

/* ISB_I32 (GEMM output only, integer-scale path): the raw int32 scaled
 * accumulator acc = sum_g P_g * k_g, before the Eq. 2 epilogue — the value a
 * row-parallel (K-sharded) layer all-reduces exactly; see isb_finalize_acc. */
enum isb_dtype { ISB_F32 = 0, ISB_BF16 = 1, ISB_F16 = 2, ISB_I32 = 3 };

/* ISB_PATH_COARSE: per-channel W4A8 (gemm_coarse, gemm.hpp:97) — the paper's
 * coarse-grained comparison; internal to isb_gemm_coarse. */
enum isb_path { ISB_PATH_FLOAT_SCALE = 0, ISB_PATH_INTEGER_SCALE = 1, ISB_PATH_COARSE = 2 };

const char* isb_last_error(void);
int isb_version(void);
/* Number of kernel launches this library has issued on the calling host
 * thread's process since load (bench evidence; monotonic). */
int64_t isb_launch_count(void);

/* --------------------------------------------------------------------------
 * K1 — per-token symmetric int8 activation quantizer.
 * Replaces quantize(x, 8, Scheme::symmetric, Granularity::per_token())
 * (quantize.hpp:146 / quantize.cpp:93-145). Bit-exact: codes are
 * llround(double(x)/s) with s = max|x_row| / 127 (s = 1 for an all-zero row),
 * never -128. Non-finite input => ISB_VALUE (checked: a device flag is read
 * back, so this call synchronizes the stream when check_finite != 0).
 */
int isb_quantize_per_token(const void* x, int x_dtype, int64_t m, int64_t k, int8_t* codes,
                           double* scales, int check_finite, void* stream);

/* Group-wise symmetric weight quantizer, the offline step that feeds the
 * packer: quantize(w, bits, symmetric, group_of(g)) (quantize.cpp:93-145,
 * unit = n*(K/g) + k/g) for float32 K x N weights; codes written as int16
 * (the reference MatQ container, types.hpp:21). per-channel == g = K. */
int isb_quantize_weight_groups(const float* w, int64_t k, int64_t n, int64_t group,
                               int bit_width, int16_t* codes, double* scales, void* stream);

/* --------------------------------------------------------------------------
 * K2 — offline int4 weight packer into the device layout.
 * Source: reference int16 codes K x N (QuantizedTensor::values,
 * quantize.hpp:128-130) or the reference packed_signed4 byte stream
 * (tensor_io.hpp:62-66, tensor_io.cpp:179-193). Scales: the reference double
 * group scales (n*(K/g)+k/g) and the IntegerScaleSet it was integerized into
 * (integer_scale.hpp:17-21); int_scales may be NULL (float-scale only).
 * Codes outside [-8, 7] => ISB_VALUE (pack_signed4 contract).
 * The handle owns its device memory; destroy with isb_weight_destroy.
 */
typedef struct isb_weight isb_weight;

int isb_weight_pack_codes(const int16_t* codes, int64_t k, int64_t n, int64_t group,
                          const double* scales, const int32_t* int_scales, int64_t amplifier,
                          void* stream, isb_weight** out);
int isb_weight_pack_signed4(const uint8_t* bytes, int64_t nbytes, int64_t k, int64_t n,
                            int64_t group, const double* scales, const int32_t* int_scales,
                            int64_t amplifier, void* stream, isb_weight** out);
/* Device verifier: writes the K x N int16 codes back (unpack_signed4,
 * tensor_io.cpp:195-208, through the device layout). */
int isb_weight_unpack_codes(const isb_weight* w, int16_t* codes, void* stream);
/* Reference-order packed_signed4 bytes (ceil(K*N/2)) regenerated from the
 * device layout; equals pack_signed4(codes) byte for byte. */
int isb_weight_repack_signed4(const isb_weight* w, uint8_t* bytes, void* stream);
int isb_weight_destroy(isb_weight* w);

typedef struct {
  int64_t k, n, group, groups, amplifier;
  int32_t exponent;
  int32_t has_int_scales;
  int64_t packed_bytes;   /* HBM bytes of the int4 payload (padded to 128x128 tiles) */
  int64_t scale_bytes;    /* HBM bytes of the per-tile int32 scales read by K3 */
  int32_t max_int_scale;  /* max k_g (the k<=16 fold band) */
  int32_t tensor_core_ok; /* 1 if group % 128 == 0 and K % 128 == 0 (K3/K4 eligible) */
} isb_weight_info_t;
int isb_weight_info(const isb_weight* w, isb_weight_info_t* info);

/* --------------------------------------------------------------------------
 * K3 / K4 — fused W4A8 GEMM on tcgen05 (kind::i8, TMEM accumulators).
 * K3 replaces gemm_integer_scale (gemm.hpp:92, gemm.cpp:205-262):
 *   out[i,j] = (double(sum_g P_g * k_g) / 2^e) * s_a[i], P_g int32 on the
 *   tensor core, sum_g in int32 (exact when overflow_analyzer says safe).
 * K4 replaces gemm_float_scale (gemm.hpp:82, gemm.cpp:156-203) in the
 *   Atom-style fp32 form: acc += float(P_g) * float(s_g), one I2F + FFMA per
 *   group and output.
 * xq: int8 codes M x K; sa: double[M]. out: M x N in out_dtype.
 * Requires K % 128 == 0 and group % 128 == 0 (isb_weight_info.tensor_core_ok);
 * other shapes => ISB_PARAM (use isb_gemm_checked).
 * Overflow: the integer path accumulates in int32, which is exact iff the
 * weight's overflow_analyzer bound (analysis.cpp:24-59, computed at pack time)
 * fits int32. An unsafe weight runs as the fewest equal K-chunks (by groups,
 * at most 16) whose own bounds fit int32: per-chunk int32 accumulators in the
 * workspace, then one exact int64 sum + Eq. 2 — the reference's int64 result
 * (gemm.cpp:205-262). ISB_OVERFLOW only for raw int32 output (cannot hold the
 * sum) or a layer no such split makes safe (exact scalar path:
 * isb_gemm_checked; run_layer falls back to float scale, gemm.cpp:489-516).
 * workspace: caller-owned device buffer of isb_gemm_workspace_size() bytes,
 * zero-filled once before first use (the kernels leave it zeroed).
 */
int isb_gemm_workspace_size(int64_t m, const isb_weight* w, int64_t* bytes);
int isb_gemm_integer_scale(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                           const isb_weight* w, void* out, int out_dtype, void* workspace,
                           int64_t workspace_bytes, void* stream);
int isb_gemm_float_scale(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                         const isb_weight* w, void* out, int out_dtype, void* workspace,
                         int64_t workspace_bytes, void* stream);

/* --------------------------------------------------------------------------
 * K1 (+) K3/K4 — per-token activation quantization + GEMM in one call
 * (BASELINE config C3 "per-token act quant fused"): x is the float32 / bf16
 * M x K activation; the codes and scales are exactly those of quantize(x, 8,
 * symmetric, per_token) (quantize.cpp:93-145) and the output equals
 * isb_quantize_per_token followed by isb_gemm_integer_scale / isb_gemm_float_scale.
 * sa_out (nullable) receives the per-token scales. Runs K1 into the caller's
 * workspace then the GEMM (PDL-chained): measured faster than a single-GEMM kernel
 * that quantizes its own K slice. The one-launch fused form is the grouped launch
 * (isb_group_plan_*, every problem M <= 64), which quantizes inside the kernel.
 */
int isb_gemm_act_fused(int path, const void* x, int x_dtype, int64_t m, int64_t k,
                       const isb_weight* w, void* out, int out_dtype, double* sa_out,
                       void* workspace, int64_t workspace_bytes, void* stream);
/* Workspace for isb_gemm_act_fused: the GEMM's plus room for the int8 codes and
 * double scales of the two-kernel form (never allocated inside the call). */
int isb_gemm_act_fused_workspace_size(int64_t m, const isb_weight* w, int64_t* bytes);

/* --------------------------------------------------------------------------
 * Grouped layer launch — K1 (+) K3/K4 for up to ISB_GROUP_MAX_PROBLEMS GEMMs in
 * ONE persistent kernel (the linears of a decoder layer that share an input
 * step, or the experts of a MoE layer). Per problem p the result is exactly
 * quantize(x_p, 8, symmetric, per_token) (quantize.cpp:93-145) followed by
 * gemm_integer_scale (gemm.cpp:205-262) or gemm_float_scale (gemm.cpp:156-203)
 * — bit-identical to isb_quantize_per_token + isb_gemm_integer_scale /
 * isb_gemm_float_scale on the same inputs.
 *  - x != NULL (every problem): float32 / bf16 activations [m][k], quantized
 *    inside the launch; xq / sa (nullable) receive the codes and scales (the
 *    plan owns buffers for the NULL ones).
 *  - x == NULL (every problem): xq / sa are the int8 codes and double scales.
 *  - m may differ per problem (0 = no work: an expert with no routed token).
 *  - weights: group == 128, K % 128 == 0; integer path: overflow_analyzer
 *    bound within int32, else ISB_OVERFLOW (the K-chunked exact path of
 *    isb_gemm_integer_scale is single-GEMM only).
 * Routes (chosen at creation; isb_group_plan_info.tile_tokens tells which):
 *  - every M <= 64: ONE persistent launch, K1 folded in (tile_tokens 16 / 32);
 *  - every M >= 512, integer scale, every k_g <= 16: K1 per problem (x given) + ONE
 *    grouped CTA-pair fold launch over all problems' tiles (tile_tokens 512);
 *  - otherwise with some M > 64: K1 per problem + the single-GEMM kernels in turn
 *    (tile_tokens 0).
 * The plan binds every pointer at creation (it allocates its schedule, counters
 * and any owned buffers there, never in isb_group_run) and may be replayed any
 * number of times, including inside CUDA graphs; one run at a time per plan.
 * Non-finite activations raise a sticky device flag, read (synchronously) with
 * isb_group_nonfinite — the in-launch analogue of isb_quantize_per_token's
 * check_finite.
 */
#define ISB_GROUP_MAX_PROBLEMS 8
typedef struct {
  const isb_weight* w;
  int64_t m;
  const void* x;   /* float32 / bf16 [m][k] or NULL */
  int32_t x_dtype; /* ISB_F32 / ISB_BF16 */
  int8_t* xq;      /* int8 codes [m][k] */
  double* sa;      /* token scales [m] */
  void* out;       /* [m][n] out_dtype */
} isb_group_problem;
typedef struct {
  int32_t grid, cluster, tile_tokens, quantize;
  double makespan_steps; /* planner's per-cluster makespan (steps of 4 x 8 KiB) */
} isb_group_info_t;
typedef struct isb_group_plan isb_group_plan;
int isb_group_plan_create(const isb_group_problem* problems, int32_t nprob, int32_t path,
                          int32_t out_dtype, isb_group_plan** plan);
int isb_group_run(isb_group_plan* plan, void* stream);
int isb_group_plan_info(const isb_group_plan* plan, isb_group_info_t* info);
int isb_group_nonfinite(isb_group_plan* plan, int32_t clear, int32_t* raised);
int isb_group_plan_destroy(isb_group_plan* plan);

/* --------------------------------------------------------------------------
 * Dense fp16 / bf16 baseline GEMM (no reference analogue; BASELINE.json north
 * star: "an fp16 cuBLAS-free dense baseline kernel ... reported for the paper's
 * speedup claims"): out[M][N] = x[M][K] * w[N][K]^T (nn.Linear weight layout),
 * hand-written tcgen05 kind::f16 with fp32 accumulation, TMA-fed, split-K over a
 * cluster at decode M. x and w share `dtype` (ISB_F16 or ISB_BF16); K % 64 == 0;
 * 16-byte aligned operands.
 */
int isb_gemm_dense(const void* x, const void* w, int dtype, int64_t m, int64_t n, int64_t k,
                   void* out, int out_dtype, void* stream);

/* --------------------------------------------------------------------------
 * QServe-style dual quantization (the paper's comparison path):
 * isb_dual_inner_quantize replaces dual_inner_quantize (gemm.cpp:311-345): the
 * 8-bit per-channel codes w8 (K x N int16, device) -> asymmetric 4-bit group codes
 * (K x N int16 in [0,15]) + double scales and int32 zero points per unit j*G + t.
 * isb_gemm_dual_quant replaces gemm_dual_quant (gemm.cpp:347-412): out = float(
 * (sum_k x * ((w - z) * s_i)) * s_outer[j] * s_a[i]) with the reference's sequential
 * double accumulation, bit-exact; out_f64 (nullable) gets the double value. Values
 * are validated on the device first (ISB_VALUE, as gemm.cpp:114, :366-372); the call
 * synchronises the stream for that check.
 */
int isb_dual_inner_quantize(const int16_t* w8, int64_t k, int64_t n, int64_t group,
                            int16_t* codes, double* scales, int32_t* zero_points, void* stream);
int isb_gemm_dual_quant(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                        const int16_t* codes, const double* scales, const int32_t* zero_points,
                        int64_t group, const double* outer_scales, int64_t n, float* out,
                        double* out_f64, void* stream);

/* --------------------------------------------------------------------------
 * Tensor parallelism (no reference analogue — the reference is one
 * host process). Row-parallel layers shard K on group boundaries: every rank
 * produces the int32 accumulator of its groups (out_dtype = ISB_I32 above),
 * the ranks all-reduce it (integer sum: exact and order-independent), and
 * isb_finalize_acc applies Eq. 2 (gemm.cpp:252): out = float((acc / 2^e) * s_a).
 * A K-sharded activation needs the FULL-row absmax for the per-token scale
 * (quantize.cpp:120-125): isb_row_absmax gives each rank's partial max, the
 * ranks all-reduce MAX, and isb_quantize_per_token_amax quantizes the local
 * slice with that global max — codes bit-identical to quantizing the full row.
 */
int isb_finalize_acc(const int32_t* acc, const double* sa, int64_t m, int64_t n,
                     int64_t amplifier, void* out, int out_dtype, void* stream);
int isb_row_absmax(const void* x, int x_dtype, int64_t m, int64_t k, float* amax, void* stream);
int isb_quantize_per_token_amax(const void* x, int x_dtype, int64_t m, int64_t k,
                                const float* amax, int8_t* codes, double* scales, void* stream);

/* --------------------------------------------------------------------------
 * Coarse-grained (per-channel) W4A8 — replaces gemm_coarse (gemm.hpp:97,
 * gemm.cpp:264-309): out[i,j] = float((double(sum_k x*w) * s_w[j]) * s_a[i]),
 * bit-exact (exact int32 sum on the tensor core, the reference's double
 * epilogue). The weight must be per-channel: packed with group = K.
 */
int isb_gemm_coarse(const int8_t* xq, const double* sa, int64_t m, int64_t k,
                    const isb_weight* w, void* out, int out_dtype, void* workspace,
                    int64_t workspace_bytes, void* stream);

/* --------------------------------------------------------------------------
 * Checked GEMM (CUDA cores, int64): the full reference semantics for any
 * group size dividing K and for layers the static bound calls unsafe:
 * per-group and running-accumulator 32-bit window tracking (gemm.cpp:42-52,
 * :245-247), max_abs_accumulator, the lexicographically first overflowing
 * output, the 2^62 hard limit, and NON-wrapped int64 results in permissive
 * mode (gemm.cpp:90-98, :246-252). Float path: od += double(P_g)*s_g in
 * double, bit-identical to gemm_float_scale.
 * Optional outputs (NULL to skip): out f32, out_f64, acc (int64 M x N, integer
 * path), partials (int64 signed P_g, M x (N*G), index (i, j*G+g)).
 * Synchronous: stats are copied to the host before returning.
 * strict != 0 and an overflow => ISB_OVERFLOW with the reference message
 * "integer accumulation left the 32-bit window at output (i, j)".
 */
typedef struct {
  int64_t max_abs_accumulator;
  int32_t overflow_detected;
  int32_t hard_limit_hit;
  int64_t overflow_i, overflow_j;
} isb_gemm_stats;

int isb_gemm_checked(int path, const int8_t* xq, const double* sa, int64_t m, int64_t k,
                     const isb_weight* w, int strict, float* out, double* out_f64, int64_t* acc,
                     int64_t* partials, isb_gemm_stats* stats, void* stream);

/* Host-side helpers of the offline path (no device work). */
/* overflow_analyzer (analysis.hpp:35, analysis.cpp:24-59). */
int isb_overflow_analyzer(int64_t k, int64_t group, int act_bits, int weight_bits,
                          const int32_t* int_scales_host, int64_t count, int64_t* static_bound,
                          double* headroom_bits, int32_t* safe);
/* search_amplifier_exponent / integerize_scales (integer_scale.cpp:21-59). */
int isb_search_amplifier_exponent(const double* scales_host, int64_t count, int32_t* exponent);
int isb_integerize_scales(const double* scales_host, int64_t count, int64_t amplifier,
                          int32_t* int_scales_host, int32_t* exponent);

#ifdef __cplusplus
}
#endif

#endif /* INTSCALE_B200_H_ */
