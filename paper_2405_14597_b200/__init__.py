"""B200-native (sm_100a) integer-scale W4A8 fine-grained GEMM (arXiv 2405.14597).

Drop-in for the reference hot path: per-token int8 activation quantize (K1),
offline int4 weight pack (K2), integer-scale group GEMM (K3) with the
float-scale variant (K4) as the speed-up denominator, and a checked int64 GEMM
with the reference's full overflow/stats semantics. All compute runs in
libintscale_b200.so (hand-written CUDA for sm_100a) behind a C ABI.
"""
from ._lib import (CudaError, DimensionError, FormatError, IntscaleError, LengthError,  # noqa
                   OverflowError_, ParamError, ValueError_)
from .ops import (GroupedGemm, IntegerScaleSet, PackedWeight, Workspace, finalize_acc,  # noqa: F401
                  DualInner, dual_inner_quantize, gemm_dual_quant,
                  gemm_act_fused, gemm_checked, gemm_coarse, gemm_dense, gemm_float_scale, gemm_integer_scale,
                  integerize_scales, launch_count, overflow_analyzer, quantize_per_token,
                  quantize_per_token_amax, quantize_weight, row_absmax, search_amplifier,
                  search_amplifier_exponent, workspace_size)

from . import moe, parallel, qtns, runtime  # noqa: F401,E402

__version__ = "0.1.0"
