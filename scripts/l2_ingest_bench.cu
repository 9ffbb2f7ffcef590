// Microbenchmark: per-SM ingest from an L2-resident buffer (4 MiB, re-read) via
// TMA bulk copies only, cp.async (LDGSTS, 16 B per thread) only, or both at once
// into disjoint smem rings. Tells whether the ~25 B/clk/SM streaming ceiling is the
// TMA engine or the SM's L2->SMEM port.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -o l2_ingest_bench l2_ingest_bench.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2405_14597_b200/csrc/common.cuh"
using namespace isb;

constexpr int kChunk = 8192, kStages = 8;

template <bool TMA, bool LSU>
__global__ void __launch_bounds__(256, 1) ingest(const uint8_t* src, int64_t span, int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kStages];
  uint8_t* ring_t = smem;                          // TMA ring
  uint8_t* ring_l = smem + kStages * kChunk;       // LSU ring (4 x 8 KiB per round)
  if (threadIdx.x == 0) { for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1); fence_barrier_init(); }
  __syncthreads();
  const uint8_t* base = src + (blockIdx.x * 8192LL * 7) % span;
  int acc = 0;
  if (TMA && threadIdx.x == 0) {
    for (int i = 0; i < kStages && i < iters; ++i) {
      mbar_arrive_expect_tx(&full[i], kChunk);
      bulk_load(ring_t + i * kChunk, base + (i * kChunk) % span, kChunk, &full[i]);
    }
    for (int i = 0; i < iters; ++i) {
      const int s = i % kStages;
      mbar_wait(&full[s], (i / kStages) & 1);
      acc += ring_t[s * kChunk];
      if (i + kStages < iters) {
        mbar_arrive_expect_tx(&full[s], kChunk);
        bulk_load(ring_t + s * kChunk, base + ((int64_t)(i + kStages) * kChunk) % span, kChunk, &full[s]);
      }
    }
  }
  if (LSU && threadIdx.x >= 32) {
    // 224 threads, each 16 B per copy, 4 rounds in flight
    const int t = threadIdx.x - 32;
    const uint32_t dst0 = smem_u32(ring_l) + t * 16;
    for (int i = 0; i < iters; ++i) {
      const uint8_t* g = base + ((int64_t)i * 224 * 16 + t * 16) % span;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst0 + (i % 4) * 224 * 16), "l"(g) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 3;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    acc += ring_l[t];
  }
  if (acc == 0x7fffffff) atomicAdd(sink, acc);
}

template <bool TMA, bool LSU>
void run(const uint8_t* buf, int64_t span, int* sink) {
  const int iters = 4000;
  auto k = ingest<TMA, LSU>;
  const int smem = kStages * kChunk + 4 * 224 * 16;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148, 256, smem>>>(buf, span, 10, sink);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 256, smem>>>(buf, span, iters, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double bytes = 148.0 * iters * ((TMA ? kChunk : 0) + (LSU ? 224 * 16 : 0));
  printf("TMA=%d LSU=%d: %8.1f GB/s total  (%5.1f B/clk/SM @1.965GHz)  %s\n", TMA, LSU,
         bytes / (ms * 1e6), bytes / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t span = 4 << 20;  // L2-resident
  uint8_t* buf; int* sink;
  cudaMalloc(&buf, span); cudaMemset(buf, 1, span); cudaMalloc(&sink, 4);
  run<true, false>(buf, span, sink);
  run<false, true>(buf, span, sink);
  run<true, true>(buf, span, sink);
  return 0;
}
