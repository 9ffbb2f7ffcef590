// B200 drop-in for proj/include/intscale/tensor_io.hpp:11-75: the QTNS container
// (header layout, readers/writers, error taxonomy of tensor_io.cpp:142-303) and
// the nibble packing. The nibble (un)packing goes through the device layout
// (K2 pack -> device -> reference byte order), so it doubles as a verifier of the
// B200 packer; the container code itself is host byte handling.
#pragma once

#include <cstdint>
#include <filesystem>
#include <variant>
#include <vector>

#include "intscale/types.hpp"

namespace intscale {

enum class DType : std::uint8_t { real32 = 0, signed8 = 1, packed_signed4 = 2 };

struct TensorHeader {
  static constexpr char kMagic[4] = {'Q', 'T', 'N', 'S'};
  static constexpr std::uint16_t kVersion = 1;
  std::uint16_t version = kVersion;
  DType dtype = DType::real32;
  std::vector<std::uint64_t> dims;
  std::uint64_t element_count() const;
  std::size_t payload_bytes() const;
};

struct QuantizedPayload {
  int bit_width = 0;  // 8 for signed8, 4 for packed_signed4
  MatQ values;        // sign-extended
};

using TensorData = std::variant<MatF, QuantizedPayload>;

TensorData read_tensor(const std::filesystem::path& path);
MatF read_float_tensor(const std::filesystem::path& path);
void write_tensor(const MatF& x, const std::filesystem::path& path);
void write_tensor(const MatQ& values, DType dtype, const std::filesystem::path& path);

std::vector<std::uint8_t> pack_signed4(const MatQ& values);
MatQ unpack_signed4(const std::vector<std::uint8_t>& bytes, Index rows, Index cols);

std::vector<std::uint8_t> encode_header(const TensorHeader& h);
TensorHeader decode_header(const std::vector<std::uint8_t>& bytes, std::size_t& offset);

}  // namespace intscale
