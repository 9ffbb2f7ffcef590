// Throughput of the Eq. 2 epilogue building blocks on one SM (independent work per
// thread, ILP 8): DADD, DMUL, F2F.F32.F64, I2F.F64, F2FP.BF16 pack, and the full
// per-output sequences of the prefill epilogue (F2F form and integer-rounding form).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cvt_bench cvt_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t eq2_bits(uint32_t acc, double sa2) {
  const double d = __hiloint2double(0x43300000, static_cast<int>(acc ^ 0x80000000u)) - 4503601774854144.0;
  const double prod = d * sa2;
  const uint32_t ph = static_cast<uint32_t>(__double2hiint(prod));
  const double c = __hiloint2double(static_cast<int>((ph & 0x7FF00000u) + (29u << 20) + (1u << 19)), 0);
  const double r = __dadd_rn(__dadd_rn(prod, c), -c);
  const uint32_t rh = static_cast<uint32_t>(__double2hiint(r));
  const uint32_t rl = static_cast<uint32_t>(__double2loint(r));
  return __funnelshift_l(rl, (rh & 0x7FFFFFFFu) - (896u << 20), 3) | (rh & 0x80000000u);
}

template <int OP>
__global__ void k(const uint32_t* in, uint32_t* out, int iters, long long* cyc) {
  uint32_t a[8];
  double x[8];
  for (int i = 0; i < 8; ++i) { a[i] = in[threadIdx.x] + i; x[i] = 1.0 + a[i] * 1e-3; }
  const double s = 1.0 + threadIdx.x * 1e-7;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = x[i] + s;                                             // DADD
      if (OP == 1) x[i] = x[i] * s;                                             // DMUL
      if (OP == 2) acc += __float_as_uint(__double2float_rn(x[i] + it));       // DADD + F2F.F32.F64
      if (OP == 3) x[i] = static_cast<double>(static_cast<int>(a[i] + it));     // I2F.F64
      if (OP == 4) { __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(a[i] + it), __uint_as_float(a[i] ^ it));
                     acc += *reinterpret_cast<uint32_t*>(&b); }                 // F2FP.BF16 pack
      if (OP == 5) { const double d = __hiloint2double(0x43300000, static_cast<int>((a[i] + it) ^ 0x80000000u)) - 4503601774854144.0;
                     acc += __float_as_uint(__double2float_rn(d * s)); }        // epilogue, F2F form
      if (OP == 6) acc += eq2_bits(a[i] + it, s);                               // epilogue, integer form
    }
  }
  long long t1 = clock64();
  double xs = 0; for (int i = 0; i < 8; ++i) xs += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + (uint32_t)xs;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 1024);
  cudaMemset(in, 1, 4096 * 4);
  const char* names[] = {"DADD", "DMUL", "DADD+F2F.F32.F64", "I2F.F64", "F2FP.BF16 (2 outs)", "epi F2F form", "epi int form"};
  for (int threads : {256, 512}) {
    for (int op = 0; op < 7; ++op) {
      const int iters = 2048;
      auto run = [&](auto kern) { kern<<<1, threads>>>(in, out, iters, cyc); };
      if (op == 0) run(k<0>); if (op == 1) run(k<1>); if (op == 2) run(k<2>); if (op == 3) run(k<3>);
      if (op == 4) run(k<4>); if (op == 5) run(k<5>); if (op == 6) run(k<6>);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("threads %3d %-22s: %7.2f per clk per SM\n", threads, names[op], (double)threads * iters * 8 / c);
    }
  }
  return 0;
}
