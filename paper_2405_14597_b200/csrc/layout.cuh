// Device data layouts shared by the packer (K2), the GEMM kernels (K3/K4) and
// the checked kernel. See DESIGN.md "Data layout in HBM".
//
// Packed int4 weight W (reference: K x N int16 codes, row-major,
// gemm.hpp:92 / quantize.cpp:93; or packed_signed4 bytes, tensor_io.cpp:179):
//
//   [n_tile = n / 128][kblock = k / 128][chunk c = (k % 128) / 32][row r = n % 128][16 B]
//
// i.e. one contiguous 8 KiB block per (128 output channels x 128 K). Inside a
// 16-byte piece, 32-bit word w (0..3) holds K = 32c + 8w + {0..7} of row r:
//   byte b (0..3): low nibble  = code(k0 + b), high nibble = code(k0 + 4 + b),
// with k0 = 32c + 8w. Nibbles are two's-complement int4 (the reference nibble
// encoding). The expansion to the tcgen05 A operand is then two LOP3-class
// ops per output word and yields 16*code per byte:
//   lo = (word << 4) & 0xF0F0F0F0   -> bytes 16*code(k0 .. k0+3)
//   hi =  word       & 0xF0F0F0F0   -> bytes 16*code(k0+4 .. k0+7)
// so the int8 MMA accumulates exactly 16 * P_g (|16 P_g| <= 2^21, no overflow).
#pragma once

#include <cstdint>

namespace isb {

constexpr int kTileN = 128;       // output channels per tile == UMMA M
constexpr int kBlockK = 128;      // K per packed block == one 128-byte int8 swizzle row
constexpr int kChunkK = 32;       // K per UMMA instruction (kind::i8)
constexpr int kBlockBytes = kTileN * kBlockK / 2;  // 8192

__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Byte offset of the 16-byte piece holding (row n, chunk of k) and the nibble
// position of code(k, n) inside it.
__host__ __device__ inline int64_t packed_piece_offset(int64_t n, int64_t k, int64_t kblocks) {
  const int64_t nt = n / kTileN, r = n % kTileN;
  const int64_t kb = k / kBlockK, c = (k % kBlockK) / kChunkK;
  return ((nt * kblocks + kb) * 4 + c) * (kTileN * 16) + r * 16;
}

__host__ __device__ inline void packed_nibble_pos(int64_t k, int* byte_in_piece, int* high) {
  const int kk = static_cast<int>(k % kChunkK);  // 0..31
  const int w = kk / 8, j = kk % 8;
  *byte_in_piece = w * 4 + (j & 3);
  *high = j >= 4;
}

}  // namespace isb
