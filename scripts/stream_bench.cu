// Microbenchmark: HBM -> SMEM streaming rate per SM with cp.async.bulk
// (chunk size x stages), versus plain vectorised LDG. 148 CTAs (one per SM)
// each stream a disjoint slice of a 1 GiB buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2405_14597_b200/csrc/common.cuh"

using namespace isb;

template <int CHUNK, int STAGES, int PER_STAGE, bool HINT>
__global__ void __launch_bounds__(128, 1) bulk_stream(const uint8_t* src, int64_t per_cta, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * per_cta;
  constexpr int kStageBytes = CHUNK * PER_STAGE;
  const int64_t n_stages = per_cta / kStageBytes;
  int acc = 0;
  if (warp == 0 && lane == 0) {
    // prologue: fill all stages
    int64_t issued = 0;
    for (; issued < STAGES && issued < n_stages; ++issued) {
      mbar_arrive_expect_tx(&full[issued], kStageBytes);
      for (int j = 0; j < PER_STAGE; ++j) {
        if (HINT)
          bulk_load_evict_first(smem + issued * kStageBytes + j * CHUNK,
                                base + issued * kStageBytes + j * CHUNK, CHUNK, &full[issued]);
        else
          bulk_load(smem + issued * kStageBytes + j * CHUNK, base + issued * kStageBytes + j * CHUNK,
                    CHUNK, &full[issued]);
      }
    }
    for (int64_t i = 0; i < n_stages; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      acc += smem[s * kStageBytes];
      const int64_t nx = i + STAGES;
      if (nx < n_stages) {
        mbar_arrive_expect_tx(&full[s], kStageBytes);
        for (int j = 0; j < PER_STAGE; ++j) {
          if (HINT)
            bulk_load_evict_first(smem + s * kStageBytes + j * CHUNK, base + nx * kStageBytes + j * CHUNK,
                                  CHUNK, &full[s]);
          else
            bulk_load(smem + s * kStageBytes + j * CHUNK, base + nx * kStageBytes + j * CHUNK, CHUNK,
                      &full[s]);
        }
      }
    }
    atomicAdd(sink, acc);
  }
}

__global__ void __launch_bounds__(512) ldg_stream(const uint4* src, int64_t per_cta_vec, int* sink) {
  const uint4* base = src + blockIdx.x * per_cta_vec;
  uint32_t acc = 0;
  for (int64_t i = threadIdx.x; i < per_cta_vec; i += 512 * 4) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      v[j] = (i + j * 512 < per_cta_vec) ? __ldcs(base + i + j * 512) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc ^= v[j].x ^ v[j].w;
  }
  if (acc == 0x12345) atomicAdd(sink, 1);
}

template <int CHUNK, int STAGES, int PER_STAGE, bool HINT>
void run_bulk(const uint8_t* buf, int64_t total, int* sink) {
  const int ctas = 148;
  const int64_t per_cta = (total / ctas) / (CHUNK * PER_STAGE) * (CHUNK * PER_STAGE);
  auto k = bulk_stream<CHUNK, STAGES, PER_STAGE, HINT>;
  const int smem = CHUNK * PER_STAGE * STAGES;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<ctas, 128, smem>>>(buf, per_cta, sink);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<ctas, 128, smem>>>(buf, per_cta, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("bulk chunk=%5d stages=%2d per_stage=%d hint=%d (in flight %6d B): %7.1f GB/s  %s\n", CHUNK,
         STAGES, PER_STAGE, HINT, CHUNK * PER_STAGE * STAGES, 5.0 * per_cta * ctas / (ms * 1e6),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t total = int64_t(1) << 30;
  uint8_t* buf;
  int* sink;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  cudaMalloc(&sink, 4);
  run_bulk<8192, 4, 1, true>(buf, total, sink);
  run_bulk<8192, 6, 1, true>(buf, total, sink);
  run_bulk<8192, 6, 1, false>(buf, total, sink);
  run_bulk<8192, 8, 1, false>(buf, total, sink);
  run_bulk<8192, 12, 1, false>(buf, total, sink);
  run_bulk<8192, 16, 1, false>(buf, total, sink);
  run_bulk<16384, 6, 1, false>(buf, total, sink);
  run_bulk<16384, 8, 1, false>(buf, total, sink);
  {
    const int ctas = 148 * 2;
    const int64_t per = total / 16 / ctas;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ldg_stream<<<ctas, 512>>>(reinterpret_cast<const uint4*>(buf), per, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) ldg_stream<<<ctas, 512>>>(reinterpret_cast<const uint4*>(buf), per, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg.128 x4 unroll, 296 CTAs x 512 thr: %7.1f GB/s\n", 5.0 * per * 16 * ctas / (ms * 1e6));
  }
  return 0;
}
