"""Dense fp16/bf16 baseline GEMM (isb_gemm_dense, tcgen05 kind::f16, no cuBLAS): the
FP16 comparator of the paper's speed-up claims. Checked against a float64 torch
reference of the same fp16/bf16 inputs: the tensor core accumulates in fp32, so
|out - ref| <= K * 2^-23 * sum|x||w| (+ the output rounding) is the stated bound."""
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_14597_b200 as isb  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("m,n,k", [(1, 4096, 4096), (16, 12288, 4096), (16, 4096, 11008),
                                   (33, 300, 1024), (64, 22016, 4096), (200, 1000, 512),
                                   (2048, 4096, 4096), (300, 128, 64)])
def test_dense_matches_fp64_reference(dtype, m, n, k):
    g = torch.Generator(device=DEV)
    g.manual_seed(m * 7 + n + k)
    x = torch.randn((m, k), generator=g, device=DEV).to(dtype)
    w = (torch.randn((n, k), generator=g, device=DEV) * 0.02).to(dtype)
    out = isb.gemm_dense(x, w, out_dtype=torch.float32)
    ref = x.double() @ w.double().t()
    bound = k * 2.0 ** -23 * (x.double().abs() @ w.double().abs().t()) + 1e-30
    err = (out.double() - ref).abs()
    assert bool((err <= 4 * bound).all()), float((err / bound).max())
    # fp16/bf16 outputs are the rounding of the fp32 result
    o16 = isb.gemm_dense(x, w)
    assert o16.dtype == dtype
    assert torch.equal(o16, out.to(dtype))
    assert isb.launch_count() > 0


def test_dense_rejects_bad_arguments():
    x = torch.zeros((4, 96), dtype=torch.float16, device=DEV)
    w = torch.zeros((8, 96), dtype=torch.float16, device=DEV)
    with pytest.raises(isb.ParamError):
        isb.gemm_dense(x, w)  # K % 64 != 0
    with pytest.raises(isb.ParamError):
        isb.gemm_dense(x.float(), w.float())
    with pytest.raises(isb.DimensionError):
        isb.gemm_dense(torch.zeros((4, 128), dtype=torch.float16, device=DEV), w)
