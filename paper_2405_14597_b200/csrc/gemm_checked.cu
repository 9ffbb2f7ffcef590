// Checked GEMM on CUDA cores with int64 accumulation: the complete reference
// semantics of gemm_integer_scale / gemm_float_scale (gemm.cpp:156-262) for
// any group size dividing K, including the 32-bit-window tracking of every
// group partial and running accumulator (WorkerState::track, gemm.cpp:42-52),
// max_abs_accumulator, the lexicographically first overflowing output
// (gemm.cpp:90-98) and non-wrapped results in permissive mode. Used by the
// drop-in API for stats, strict mode, record_partials, unsafe layers and
// non-128-multiple group sizes. One thread per output element.
#include <climits>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

constexpr int64_t kWindowLo = INT_MIN;
constexpr int64_t kWindowHi = INT_MAX;
constexpr int64_t kHardLimit = int64_t{1} << 62;

struct Tracker {
  int64_t max_abs = 0;
  bool overflow = false;
  bool hard = false;
  __device__ __forceinline__ void track(int64_t v) {
    const int64_t a = v < 0 ? -v : v;
    max_abs = a > max_abs ? a : max_abs;
    overflow = overflow || v < kWindowLo || v > kWindowHi;
    hard = hard || v < -kHardLimit || v > kHardLimit;
  }
};

__global__ void gemm_checked_kernel(int path, const int8_t* __restrict__ xq,
                                    const double* __restrict__ sa, int64_t M, int64_t K,
                                    int64_t N, int64_t g, int64_t G,
                                    const uint8_t* __restrict__ packed, int64_t kblocks,
                                    const int32_t* __restrict__ ks, const double* __restrict__ s,
                                    double amp, float* __restrict__ out,
                                    double* __restrict__ out_f64, int64_t* __restrict__ acc_out,
                                    int64_t* __restrict__ partials,
                                    unsigned long long* __restrict__ stats) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  const int64_t i = idx / N, j = idx % N;
  const int8_t* xr = xq + i * K;
  // p_worst = g * 128 * 8 (abs_bound uses |qmin|, gemm.cpp:102-104, :228-229)
  const bool check_macs = g * 128 * 8 > kWindowHi;
  Tracker tr;
  int64_t acc = 0;
  double od = 0.0;
  uint4 piece = make_uint4(0, 0, 0, 0);
  int64_t piece_k = -1;
  for (int64_t gi = 0; gi < G; ++gi) {
    int64_t p = 0;
    for (int64_t k = gi * g; k < (gi + 1) * g; ++k) {
      const int64_t kc = k / kChunkK;
      if (kc != piece_k) {
        piece = *reinterpret_cast<const uint4*>(packed + packed_piece_offset(j, k, kblocks));
        piece_k = kc;
      }
      int byte, high;
      packed_nibble_pos(k, &byte, &high);
      const uint32_t word = (&piece.x)[byte >> 2];
      const int nib = (word >> (8 * (byte & 3) + 4 * high)) & 0xF;
      const int wcode = nib >= 8 ? nib - 16 : nib;
      p += static_cast<int64_t>(xr[k]) * wcode;
      if (check_macs) tr.track(p);
    }
    tr.track(p);
    if (path == ISB_PATH_INTEGER_SCALE) {
      acc = static_cast<int64_t>(static_cast<uint64_t>(acc) +
                                 static_cast<uint64_t>(p) * static_cast<uint64_t>(
                                                                static_cast<int64_t>(ks[j * G + gi])));
      tr.track(acc);
    } else {
      od = __dadd_rn(od, __dmul_rn(static_cast<double>(p), s[j * G + gi]));
    }
    if (partials) partials[i * (N * G) + j * G + gi] = p;
  }
  double o;
  if (path == ISB_PATH_INTEGER_SCALE)
    o = __dmul_rn(__ddiv_rn(__ll2double_rn(acc), amp), sa[i]);  // gemm.cpp:252
  else
    o = __dmul_rn(od, sa[i]);                                  // gemm.cpp:193
  if (out) out[idx] = __double2float_rn(o);
  if (out_f64) out_f64[idx] = o;
  if (acc_out) acc_out[idx] = acc;
  atomicMax(&stats[0], static_cast<unsigned long long>(tr.max_abs));
  if (tr.overflow) atomicMin(&stats[1], static_cast<unsigned long long>(idx));
  if (tr.hard) atomicMin(&stats[2], static_cast<unsigned long long>(idx));
}

}  // namespace

void launch_gemm_checked(int path, const int8_t* xq, const double* sa, int64_t m,
                         const isb_weight& w, float* out, double* out_f64, int64_t* acc,
                         int64_t* partials, unsigned long long* stats_dev, cudaStream_t s) {
  const int64_t total = m * w.n;
  const int threads = 128;
  const unsigned blocks = static_cast<unsigned>((total + threads - 1) / threads);
  gemm_checked_kernel<<<blocks, threads, 0, s>>>(
      path, xq, sa, m, w.k, w.n, w.group, w.groups, w.packed, w.kblocks, w.int_scales, w.scales,
      static_cast<double>(w.amplifier), out, out_f64, acc, partials, stats_dev);
  cuda_check(cudaGetLastError(), "gemm_checked launch");
  count_launch();
}

}  // namespace isb
