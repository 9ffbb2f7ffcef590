// Microbenchmark: tcgen05.mma throughput (kind::i8 / f16) by shape, with the
// issue loop free of index arithmetic; plus the cost of tcgen05.commit and of
// mbarrier.try_wait on an already-completed phase.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -o mma_bench mma_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2405_14597_b200/csrc/common.cuh"

using namespace isb;

__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// VAR: 0 = i8 SS, 1 = i8 TS, 3 = f16 SS. NACC accumulators round robin. MODE:
// 0 plain MMAs, 1 + 3 commits per 4*NACC MMAs, 2 + 3 try_waits (completed) per 4*NACC MMAs.
template <int M, int N, int VAR, int NACC, int MODE>
__global__ void bench(int64_t* out, int iters) {
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ uint64_t bar, done_bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  constexpr uint32_t idesc = VAR == 3 ? idesc_f16(M, N) : make_idesc_i8(M, N);
  const uint64_t bdesc = make_sw128_kmajor_desc(smem_u32(dsmem));
  const uint64_t adesc = make_sw128_kmajor_desc(smem_u32(dsmem + 32768));
  if (warp == 0) {
    if (elect_one()) {
      mbar_arrive(&done_bar);  // complete phase 0 of done_bar for the try_wait probes
      const int64_t t0 = clock64_();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int j = 0; j < NACC; ++j) {
            const uint32_t d = tb + 256 + j * N;
            if (VAR == 0) mma_i8_ss(d, adesc + c * 2, bdesc + c * 2, idesc, 1);
            if (VAR == 1) mma_i8_ts(d, tb + c * 8, bdesc + c * 2, idesc, 1);
            if (VAR == 3) mma_f16_ss(d, adesc + c * 2, bdesc + c * 2, idesc, 1);
          }
        }
        if (MODE == 1) {
          mma_commit(&bar);
          mma_commit(&bar);
          mma_commit(&bar);
        }
        if (MODE == 2) {
          mbar_wait(&done_bar, 0);
          mbar_wait(&done_bar, 0);
          mbar_wait(&done_bar, 0);
        }
      }
      const int64_t t1 = clock64_();
      out[0] = t1 - t0;
      out[1] = 0;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

template <int M, int N, int VAR, int NACC, int MODE>
void run(int iters) {
  int64_t* d;
  cudaMalloc(&d, 16);
  auto k = bench<M, N, VAR, NACC, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<<<1, 128, 65536>>>(d, iters);
  int64_t h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  const char* vn[] = {"i8-SS", "i8-TS", "", "f16-SS"};
  const double n_mma = double(iters) * 4 * NACC;
  const double macs = double(M) * N * (VAR == 3 ? 16 : 32);
  printf("%-6s M=%3d N=%3d nacc=%d mode=%d: %6.1f cyc/mma, %6.0f MAC/clk (%s)\n", vn[VAR], M, N,
         NACC, MODE, double(h[0]) / n_mma, macs * n_mma / double(h[0]), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<128, 16, 1, 1, 0>(64);
  run<128, 16, 1, 4, 0>(64);
  run<128, 16, 0, 1, 0>(64);
  run<128, 32, 1, 1, 0>(64);
  run<128, 64, 1, 1, 0>(64);
  run<128, 128, 1, 1, 0>(64);
  run<128, 256, 1, 1, 0>(64);
  run<128, 256, 0, 1, 0>(64);
  run<128, 256, 3, 1, 0>(64);
  run<64, 256, 0, 1, 0>(64);
  run<128, 16, 1, 1, 1>(64);
  run<128, 16, 1, 1, 2>(64);
  run<128, 128, 1, 1, 1>(64);
  return 0;
}
