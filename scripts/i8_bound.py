"""Upper bound of an SS-form int8 tcgen05 GEMM on this box: the dense kernel's pipeline
on kind::i8 with pre-expanded int8 weights (isb_debug_gemm_dense_i8), LLaMA-2-7B
linears at prefill M, vs the W4A8 integer-scale K3 on the same shapes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.isb_debug_gemm_dense_i8.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_void_p, C.c_void_p]
dev = torch.device("cuda:0")
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
tot = 0.0
for name, k, n in bench.LAYER:
    ws = [torch.randint(-128, 112, (n, k), dtype=torch.int8, device=dev) for _ in range(3)]
    x = torch.randint(-127, 128, (m, k), dtype=torch.int8, device=dev)
    out = torch.empty((m, n), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def run(r):
        _lib.check(lib.isb_debug_gemm_dense_i8(x.data_ptr(), ws[r].data_ptr(), m, n, k, out.data_ptr(),
                                               st))
    run(0)
    torch.cuda.synchronize()
    ref = (x[:64].float() @ ws[0].float().t())  # exact in fp32 (|acc| < 2^24 for these K)
    ok = torch.equal(out[:64], ref)
    for r in range(3):
        run(r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(12):
        run(i % 3)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 12
    tot += us
    print(f"{name}: M={m} {us:.1f} us  {2*m*n*k/us/1e6:.0f} TOPS  exact={ok}")
flops = sum(2 * m * k * n for _, k, n in bench.LAYER)
print(f"layer {tot:.1f} us  {flops/tot/1e6:.0f} TOPS")
