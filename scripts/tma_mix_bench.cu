// Microbenchmark: per-SM streaming rate when each pipeline stage carries an 8 KiB
// weight bulk copy plus an activation tile (2-D tensor TMA, or a flat bulk copy of
// a pre-swizzled tile) plus a 512 B scale bulk copy — the decode GEMM's mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -o tma_mix_bench tma_mix_bench.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cudaTypedefs.h>

#include "../paper_2405_14597_b200/csrc/common.cuh"

using namespace isb;

template <int STAGES, int MODE>  // MODE 0: W only, 1: W + X tensor TMA, 2: W + X flat bulk, 3: W + X TMA + scale
__global__ void __launch_bounds__(128, 1) mix_stream(const __grid_constant__ CUtensorMap xmap,
                                                      const uint8_t* src, const uint8_t* xflat,
                                                      int64_t per_cta, int kblocks, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES];
  constexpr int kStage = 8192 + 2048 + 1024;
  if (threadIdx.x == 0) {
    prefetch_tensormap(&xmap);
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * per_cta;
  const int64_t n = per_cta / 8192;
  int acc = 0;
  if (threadIdx.x == 0) {
    auto issue = [&](int64_t i, int s) {
      uint32_t bytes = 8192 + (MODE >= 1 ? 2048 : 0) + (MODE == 3 ? 512 : 0);
      mbar_arrive_expect_tx(&full[s], bytes);
      bulk_load(smem + s * kStage, base + i * 8192, 8192, &full[s]);
      const int kb = static_cast<int>((blockIdx.x * 7 + i) % kblocks);
      if (MODE == 1 || MODE == 3) tma_load_2d(smem + s * kStage + 8192, &xmap, &full[s], kb * 128, 0);
      if (MODE == 2) bulk_load(smem + s * kStage + 8192, xflat + kb * 2048, 2048, &full[s]);
      if (MODE == 3) bulk_load(smem + s * kStage + 10240, xflat + kb * 512, 512, &full[s]);
    };
    for (int64_t i = 0; i < STAGES && i < n; ++i) issue(i, i);
    for (int64_t i = 0; i < n; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      acc += smem[s * kStage];
      if (i + STAGES < n) issue(i + STAGES, s);
    }
    atomicAdd(sink, acc);
  }
}

template <int STAGES, int MODE>
void run(const CUtensorMap& map, const uint8_t* buf, const uint8_t* xf, int64_t total, int* sink) {
  const int ctas = 148;
  const int64_t per_cta = (total / ctas) / 8192 * 8192;
  auto k = mix_stream<STAGES, MODE>;
  const int smem = (8192 + 2048 + 1024) * STAGES + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<ctas, 128, smem>>>(map, buf, xf, per_cta, 32, sink);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<ctas, 128, smem>>>(map, buf, xf, per_cta, 32, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("mode %d stages %2d: weight stream %7.1f GB/s  %s\n", MODE, STAGES,
         5.0 * per_cta * ctas / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t total = int64_t(1) << 30;
  uint8_t *buf, *x, *xf;
  int* sink;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  cudaMalloc(&x, 16 * 4096);
  cudaMalloc(&xf, 16 * 4096);
  cudaMalloc(&sink, 4);
  cudaDriverEntryPointQueryResult q{};
  void* f = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  CUtensorMap map;
  const cuuint64_t dims[2] = {4096, 16};
  const cuuint64_t strides[1] = {4096};
  const cuuint32_t box[2] = {128, 16};
  const cuuint32_t estr[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<9, 0>(map, buf, xf, total, sink);
  run<9, 1>(map, buf, xf, total, sink);
  run<9, 2>(map, buf, xf, total, sink);
  run<9, 3>(map, buf, xf, total, sink);
  run<16, 1>(map, buf, xf, total, sink);
  run<16, 3>(map, buf, xf, total, sink);
  return 0;
}
