// B200 drop-in for the nibble packing of proj/include/intscale/tensor_io.hpp:62-66.
// Both directions go through the device layout (K2 pack -> device -> reference
// byte order), so they double as a verifier of the B200 packer.
#pragma once

#include <cstdint>
#include <vector>

#include "intscale/types.hpp"

namespace intscale {

std::vector<std::uint8_t> pack_signed4(const MatQ& values);
MatQ unpack_signed4(const std::vector<std::uint8_t>& bytes, Index rows, Index cols);

}  // namespace intscale
