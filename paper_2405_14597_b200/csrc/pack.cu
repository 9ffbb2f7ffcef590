// K2 — offline int4 weight packer (+ device verifiers).
//
// Source formats (reference):
//   * int16 codes, row-major K x N (QuantizedTensor::values, quantize.hpp:128-130)
//   * packed_signed4 bytes: flat row-major index i -> byte i/2, even i in the low
//     nibble, two's complement (tensor_io.cpp:179-208)
// Destination: the tiled device layout of layout.cuh (8 KiB per 128x128 block,
// nibble-interleaved so the GEMM expands a 32-bit word to two int8x4 words with
// one shift and two ANDs, and 32 consecutive threads read 512 contiguous bytes).
#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace isb {
namespace {

__device__ __forceinline__ int code_from_signed4(const uint8_t* bytes, int64_t i) {
  const uint8_t b = bytes[i >> 1];
  int v = (i & 1) ? (b >> 4) : (b & 0xF);
  return v >= 8 ? v - 16 : v;
}

// One thread per 16-byte piece (row r of chunk c of block (nt, kb)).
__global__ void pack_kernel(const int16_t* __restrict__ codes, const uint8_t* __restrict__ s4,
                            int64_t K, int64_t N, uint8_t* __restrict__ packed, int64_t kblocks,
                            int64_t pieces, int* __restrict__ bad) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= pieces) return;
  const int64_t r = p % kTileN;
  const int64_t c = (p / kTileN) % 4;
  const int64_t blk = p / (kTileN * 4);  // nt * kblocks + kb
  const int64_t kb = blk % kblocks, nt = blk / kblocks;
  const int64_t n = nt * kTileN + r;
  const int64_t k0 = kb * kBlockK + c * kChunkK;
  uint32_t words[4];
  bool ok = true;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t k = k0 + 8 * w + j;
      int v = 0;
      if (n < N && k < K) {
        v = codes ? static_cast<int>(codes[k * N + n]) : code_from_signed4(s4, k * N + n);
        ok = ok && v >= -8 && v <= 7;
      }
      const int byte = j & 3, high = j >> 2;
      word |= (static_cast<uint32_t>(v) & 0xFu) << (8 * byte + 4 * high);
    }
    words[w] = word;
  }
  if (!ok) atomicExch(bad, 1);
  *reinterpret_cast<uint4*>(packed + blk * kBlockBytes + c * (kTileN * 16) + r * 16) =
      make_uint4(words[0], words[1], words[2], words[3]);
}

__device__ __forceinline__ int packed_code(const uint8_t* packed, int64_t n, int64_t k,
                                           int64_t kblocks) {
  int byte_in_piece, high;
  packed_nibble_pos(k, &byte_in_piece, &high);
  const uint8_t b = packed[packed_piece_offset(n, k, kblocks) + byte_in_piece];
  const int v = high ? (b >> 4) : (b & 0xF);
  return v >= 8 ? v - 16 : v;
}

__global__ void unpack_kernel(const uint8_t* __restrict__ packed, int64_t K, int64_t N,
                              int64_t kblocks, int16_t* __restrict__ codes) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= K * N) return;
  const int64_t k = i / N, n = i % N;
  codes[i] = static_cast<int16_t>(packed_code(packed, n, k, kblocks));
}

__global__ void repack_signed4_kernel(const uint8_t* __restrict__ packed, int64_t K, int64_t N,
                                      int64_t kblocks, uint8_t* __restrict__ out) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = K * N;
  if (b >= (total + 1) / 2) return;
  const int64_t i0 = 2 * b, i1 = 2 * b + 1;
  const int lo = packed_code(packed, i0 % N, i0 / N, kblocks);
  const int hi = i1 < total ? packed_code(packed, i1 % N, i1 / N, kblocks) : 0;
  out[b] = static_cast<uint8_t>((lo & 0xF) | ((hi & 0xF) << 4));
}

// [n_tile][g][128] tiling of the per-(n, g) scales for coalesced epilogue reads.
__global__ void tile_scales_kernel(const int32_t* __restrict__ ks, const double* __restrict__ s,
                                   int64_t N, int64_t G, int64_t total,
                                   int32_t* __restrict__ kt, float* __restrict__ ft) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t r = i % kTileN;
  const int64_t g = (i / kTileN) % G;
  const int64_t nt = i / (kTileN * G);
  const int64_t n = nt * kTileN + r;
  if (kt) kt[i] = (n < N && ks) ? ks[n * G + g] : 1;
  // s / 16 undoes the x16 of the nibble expansion (exact power-of-two scaling).
  if (ft) ft[i] = n < N ? static_cast<float>(s[n * G + g]) * 0.0625f : 0.0f;
}

unsigned blocks_for(int64_t total, int threads) {
  return static_cast<unsigned>((total + threads - 1) / threads);
}

}  // namespace

void launch_pack(const int16_t* codes, const uint8_t* signed4, int64_t k, int64_t n,
                 uint8_t* packed, int64_t kblocks, int64_t n_tiles, int* bad, cudaStream_t s) {
  const int64_t pieces = n_tiles * kblocks * 4 * kTileN;
  pack_kernel<<<blocks_for(pieces, 256), 256, 0, s>>>(codes, signed4, k, n, packed, kblocks,
                                                       pieces, bad);
  cuda_check(cudaGetLastError(), "pack launch");
  count_launch();
}

void launch_tile_scales(const int32_t* int_scales, const double* scales, int64_t n,
                        int64_t groups, int64_t n_tiles, int32_t* kscale, float* fscale,
                        cudaStream_t s) {
  const int64_t total = n_tiles * groups * kTileN;
  tile_scales_kernel<<<blocks_for(total, 256), 256, 0, s>>>(int_scales, scales, n, groups, total,
                                                             kscale, fscale);
  cuda_check(cudaGetLastError(), "tile_scales launch");
  count_launch();
}

void launch_unpack(const isb_weight& w, int16_t* codes, cudaStream_t s) {
  unpack_kernel<<<blocks_for(w.k * w.n, 256), 256, 0, s>>>(w.packed, w.k, w.n, w.kblocks, codes);
  cuda_check(cudaGetLastError(), "unpack launch");
  count_launch();
}

void launch_repack_signed4(const isb_weight& w, uint8_t* bytes, cudaStream_t s) {
  repack_signed4_kernel<<<blocks_for((w.k * w.n + 1) / 2, 256), 256, 0, s>>>(w.packed, w.k, w.n,
                                                                             w.kblocks, bytes);
  cuda_check(cudaGetLastError(), "repack launch");
  count_launch();
}

}  // namespace isb
