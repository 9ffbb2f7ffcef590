// Microbenchmark: tcgen05.ld throughput per SM (32x32b.xN, W warps).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -o tmem_bench tmem_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2405_14597_b200/csrc/common.cuh"

using namespace isb;

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* v);
template <>
__device__ __forceinline__ void ld<16>(uint32_t taddr, uint32_t* v) {
  tmem_ld_x16_(taddr, *reinterpret_cast<uint32_t(*)[16]>(v));
}

__device__ __forceinline__ void ld64(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "
      "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
        "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]),
        "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]),
        "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]),
        "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
        "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]),
        "=r"(v[62]), "=r"(v[63])
      : "r"(taddr)
      : "memory");
}

template <int W, int X, bool IMAD>
__global__ void bench(int64_t* out, int iters, int* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot + (((warp % 4) * 32) << 16) + (warp / 4) * 64;
  uint32_t acc = 0;
  __syncthreads();
  const int64_t t0 = clock64_();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[64];
    if (X == 16) {
      ld<16>(tb + (i & 3) * 16, v);
      tmem_wait_ld();
#pragma unroll
      for (int t = 0; t < 16; ++t) acc = IMAD ? v[t] * 7u + acc : acc ^ v[t];
    } else {
      ld64(tb, v);
      tmem_wait_ld();
#pragma unroll
      for (int t = 0; t < 64; ++t) acc = IMAD ? v[t] * 7u + acc : acc ^ v[t];
    }
  }
  __syncthreads();
  const int64_t t1 = clock64_();
  if (acc == 0x1234567) atomicAdd(sink, 1);
  if (threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int W, int X, bool IMAD>
void run(int iters) {
  int64_t* d;
  int* sink;
  cudaMalloc(&d, 16);
  cudaMalloc(&sink, 4);
  bench<W, X, IMAD><<<1, W * 32>>>(d, iters, sink);
  int64_t h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = double(iters) * W * 32 * X * 4;
  printf("warps=%2d x%d imad=%d: %.1f B/clk (%.1f cyc per warp-load) %s\n", W, X, IMAD,
         bytes / h, double(h) / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4, 16, false>(2000);
  run<8, 16, false>(2000);
  run<16, 16, false>(2000);
  run<4, 64, false>(1000);
  run<16, 64, false>(1000);
  run<16, 16, true>(2000);
  run<16, 64, true>(1000);
  return 0;
}
