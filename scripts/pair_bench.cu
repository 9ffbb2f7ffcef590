// Microbenchmark for the prefill skeleton choice (prefill):
//  (1) single-CTA SS kind::i8 M=128 N=256 MMA rate while other warps load the
//      shared-memory port (st.shared / ld.shared / bulk-copy writes): does operand
//      staging traffic slow the tensor core?
//  (2) CTA-pair (cta_group::2) kind::i8 M=256 rate, A from TMEM (TS) or SMEM (SS),
//      N = 256 / 192, with and without the same contention.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -o pair_bench pair_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2405_14597_b200/csrc/common.cuh"

using namespace isb;

__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void mma1_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void mma1_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc)
      : "memory");
}

// PAIR: 0 single CTA, 1 CTA pair. TS: A from TMEM. CONT: 0 none, 1 st.shared.v4 by 8
// warps, 2 ld.shared.v4 by 8 warps, 3 bulk copies (L2 -> smem) 8 KiB each, 4 slots.
template <int PAIR, int TS, int N, int CONT>
__global__ void __launch_bounds__(384, 1) bench(int64_t* out, const uint8_t* src, int iters) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done, bfull[4];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bfull[i], 1);
    stop = 0;
    fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&slot)), "r"(512) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(&slot, 512);
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  constexpr int M = PAIR ? 256 : 128;
  constexpr uint32_t idesc = make_idesc_i8(M, N);
  // operands: B at [0, 32K), A at [32K, 48K); contention region [64K, 128K)
  const uint64_t bdesc = make_sw128_kmajor_desc(smem_u32(smem));
  const uint64_t adesc = make_sw128_kmajor_desc(smem_u32(smem + 32768));
  int64_t cont_ops = 0;
  if (warp == 0) {
    if (rank == 0 && elect_one()) {
      const int64_t t0 = clock64_();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t d = tb + 256;
          if (PAIR) {
            if (TS) mma2_ts(d, tb + c * 8, bdesc + c * 2, idesc);
            else mma2_ss(d, adesc + c * 2, bdesc + c * 2, idesc);
          } else {
            if (TS) mma1_ts(d, tb + c * 8, bdesc + c * 2, idesc);
            else mma1_ss(d, adesc + c * 2, bdesc + c * 2, idesc);
          }
        }
      }
      if (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&done)), "h"((uint16_t)3) : "memory");
      else
        mma_commit(&done);
      mbar_wait(&done, 0);
      const int64_t t1 = clock64_();
      out[0] = t1 - t0;
      stop = 1;
    }
    __syncwarp();
  } else if (PAIR && rank == 1 && warp == 1) {
    mbar_wait(&done, 0);
    stop = 1;
  } else if (warp >= 4 && CONT != 0) {
    const int t = threadIdx.x - 128;  // 0..255
    if (CONT == 1 || CONT == 2) {
      const uint32_t base = smem_u32(smem + 65536) + (t * 16);
      uint32_t x = t;
      while (!stop) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t a = base + (j * 4096) % 65536;
          if (CONT == 1) {
            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(x) : "memory");
          } else {
            uint4 v = ld_shared_v4(a);
            x ^= v.x;
          }
        }
        cont_ops += 16;
      }
      if (x == 0x12345) out[3] = x;
    } else if (CONT == 3 && warp == 4) {
      int ph[4] = {0, 0, 0, 0};
      if (elect_one()) {
        for (int s = 0; s < 4; ++s) {
          mbar_arrive_expect_tx(&bfull[s], 8192);
          bulk_load(smem + 65536 + s * 8192, src + s * 8192, 8192, &bfull[s]);
        }
        int i = 0;
        while (!stop) {
          const int s = i & 3;
          mbar_wait(&bfull[s], ph[s]);
          ph[s] ^= 1;
          mbar_arrive_expect_tx(&bfull[s], 8192);
          bulk_load(smem + 65536 + s * 8192, src + ((i * 8192) & ((1 << 22) - 1)), 8192, &bfull[s]);
          ++i;
          cont_ops += 1;
        }
        for (int s = 0; s < 4; ++s) mbar_wait(&bfull[(i + s) & 3], ph[(i + s) & 3]);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (CONT == 1 || CONT == 2) {
    if (warp >= 4) atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)cont_ops * 16);
  } else if (CONT == 3) {
    if (warp == 4 && (threadIdx.x & 31) == 0 && cont_ops) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)cont_ops * 8192);
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512) : "memory");
    } else {
      tmem_dealloc(tb, 512);
    }
  }
}

template <int PAIR, int TS, int N, int CONT>
void run(const char* name, const uint8_t* src, int iters) {
  int64_t* d;
  cudaMalloc(&d, 32);
  cudaMemset(d, 0, 32);
  auto k = bench<PAIR, TS, N, CONT>;
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(PAIR ? 2 : 1);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, d, src, iters);
  cudaError_t e = cudaDeviceSynchronize();
  int64_t h[4] = {0, 0, 0, 0};
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  const int M = PAIR ? 256 : 128;
  const double n_mma = double(iters) * 4;
  const double macs = double(M) * N * 32 / (PAIR ? 2 : 1);  // per SM
  printf("%-28s: %7.1f cyc/mma, %6.0f MAC/clk/SM, contention %6.1f B/clk (%s)\n", name,
         double(h[0]) / n_mma, macs * n_mma / double(h[0]),
         h[0] ? double(h[1]) / double(h[0]) : 0.0, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, 1 << 22);
  cudaMemset(src, 1, 1 << 22);
  const int it = 400;
  run<0, 0, 256, 0>("1cta SS N=256", src, it);
  run<0, 0, 256, 1>("1cta SS N=256 +sts", src, it);
  run<0, 0, 256, 2>("1cta SS N=256 +lds", src, it);
  run<0, 0, 256, 3>("1cta SS N=256 +bulk", src, it);
  run<0, 1, 256, 0>("1cta TS N=256", src, it);
  run<0, 1, 256, 1>("1cta TS N=256 +sts", src, it);
  run<0, 1, 256, 3>("1cta TS N=256 +bulk", src, it);
  run<1, 1, 256, 0>("pair TS N=256", src, it);
  run<1, 1, 256, 1>("pair TS N=256 +sts", src, it);
  run<1, 1, 256, 2>("pair TS N=256 +lds", src, it);
  run<1, 1, 256, 3>("pair TS N=256 +bulk", src, it);
  run<1, 1, 192, 0>("pair TS N=192", src, it);
  run<1, 1, 192, 1>("pair TS N=192 +sts", src, it);
  run<1, 0, 256, 0>("pair SS N=256", src, it);
  run<1, 0, 256, 1>("pair SS N=256 +sts", src, it);
  run<1, 0, 256, 3>("pair SS N=256 +bulk", src, it);
  return 0;
}
