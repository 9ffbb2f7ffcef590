"""The tensors bench.py actually times, checked against the oracle.

bench.py builds its LLaMA-2-7B layer on the device (llama_like-structured weights,
group-quantized by the device quantizer, integerized at alpha = 1024) and times one
grouped layer launch (K1 folded in) per step. Here the same construction (same seed as
bench's rank 0) is run once and every linear's output of that launch is compared with
the CPU oracle's gemm_integer_scale (gemm.cpp:205-262) on the SAME codes and scales:
bf16 output == RN(oracle float32) for all 4 x 16 x N outputs, and the device weight
codes / scales / integer scales equal the oracle's quantizer / integerizer on them.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402

DEV = torch.device("cuda:0")


def test_benched_layer_matches_oracle():
    m = 16
    layers, xs = bench.build_layers(isb, m, DEV, seed=1234)   # bench.run_ours, rank 0
    lin = layers[0]
    plan = isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(lin, xs)])
    outs = plan.run()
    torch.cuda.synchronize()
    workers = os.cpu_count() or 1
    for (name, k, n, w, max_k), x, out in zip(lin, xs, outs):
        codes = w.unpack_codes().cpu().numpy().astype(np.int16)        # K x N
        scales = w.group_scales.cpu().numpy().astype(np.float64)        # reference unit order
        wo = O.QuantizedTensor(codes, 4, O.SYMMETRIC, O.GROUP, bench.GROUP, scales,
                               np.zeros(0, np.int32))
        so = O.integerize_scales(scales, bench.ALPHA)
        assert int(so.int_scales.max()) == max_k
        xo = O.quantize_per_token(x.cpu().numpy())
        ref = O.gemm_integer_scale(xo, wo, so, workers=workers, record=False)
        ref_bf16 = torch.from_numpy(ref.output).to(torch.bfloat16)
        assert torch.equal(out.cpu(), ref_bf16), f"{name}: grouped bench launch != oracle"
