// Throughput of the epilogue conversion / FP64 ops on one SM (64 threads = 2 warps,
// like the grouped kernel's reduction warps, and 512 threads).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_bench fp64_bench.cu
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>

template <int OP>
__global__ void k(const int* in, float* out, int iters, long long* cyc) {
  int a = in[threadIdx.x];
  double s = 1.0 + threadIdx.x * 1e-3, acc = 0.0;
  float facc = 0.f;
  unsigned short h = 0;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) { acc += __dmul_rn(static_cast<double>(a + i) * 0.0009765625, s); }       // I2F.F64 + 2 DMUL
    if (OP == 1) { facc += __double2float_rn(s * (double)i); }                           // DMUL + F2F.F32.F64
    if (OP == 2) { h ^= __bfloat16_as_ushort(__float2bfloat16_rn(facc + i)); }           // F2F.BF16
    if (OP == 3) { acc = __dmul_rn(acc, s); }                                            // DMUL chain
    if (OP == 4) { facc += static_cast<float>(static_cast<double>(a + i)); }             // I2F.F64 + F2F
    if (OP == 5) { acc = fma(acc, s, 1.0); }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc + facc + h;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int* in; float* out; long long* cyc;
  cudaMalloc(&in, 4096); cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  cudaMemset(in, 1, 4096);
  const char* names[] = {"I2F.F64+2xDMUL", "DMUL+F2F.F32.F64", "F2F.BF16.F32", "DMUL dep chain", "I2F.F64+F2F", "DFMA"};
  for (int threads : {64, 512}) {
    for (int op = 0; op < 6; ++op) {
      const int iters = 4096;
      auto run = [&](auto kern) { kern<<<1, threads>>>(in, out, iters, cyc); };
      if (op == 0) run(k<0>); if (op == 1) run(k<1>); if (op == 2) run(k<2>);
      if (op == 3) run(k<3>); if (op == 4) run(k<4>); if (op == 5) run(k<5>);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("threads %3d %-20s: %6.2f cycles per iteration per warp-instr, %7.2f thread-ops/clk/SM\n", threads,
             names[op], (double)c / iters, (double)threads * iters / c);
    }
  }
  return 0;
}
