// B200 drop-in for the hot-path part of proj/include/intscale/analysis.hpp:25-79.
#pragma once

#include "intscale/gemm.hpp"
#include "intscale/integer_scale.hpp"

namespace intscale {

struct OverflowReport {
  std::int64_t static_bound = 0;
  std::int64_t observed_max = 0;
  double headroom_bits = 0.0;
  bool safe = false;
};

OverflowReport overflow_analyzer(Index k, Index group_size, int act_bits, int weight_bits,
                                 const IntegerScaleSet& int_scales);

KernelStats expected_counters(PathKind path, Index m, Index n, Index k, Index group);

}  // namespace intscale
