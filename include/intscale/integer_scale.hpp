// B200 drop-in for proj/include/intscale/integer_scale.hpp (integer_scale.hpp:17-41).
#pragma once

#include "intscale/types.hpp"

namespace intscale {

struct IntegerScaleSet {
  VecI int_scales;
  std::int64_t amplifier = 1;
  int exponent = 0;
};

constexpr std::int64_t kDefaultAmplifier = 1024;
constexpr std::int64_t default_amplifier() { return kDefaultAmplifier; }

std::int64_t search_amplifier(const VecD& scales);
int search_amplifier_exponent(const VecD& scales);
IntegerScaleSet integerize_scales(const VecD& scales, std::int64_t amplifier);

}  // namespace intscale
