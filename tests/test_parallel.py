"""Tensor parallelism: column-parallel (N-split + all-gather) and
row-parallel (group-boundary K-split, global per-token max, exact int32
all-reduce, one Eq. 2 epilogue) must reproduce the single-device layer bit for
bit.

* CPU: world sizes 2 and 3 over gloo (uneven shards included), the layers of
  paper_2405_14597_b200.parallel driven with the oracle as the compute backend
  (the checker) — this exercises the partitioning and exchange logic exactly as
  the NCCL path runs it.
* GPU: the same shards through the CUDA kernels on one device (int32
  accumulator output, finalize, row absmax, quantize-with-global-max), combined
  locally, against the unsharded kernel and the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2405_14597_b200 import parallel as par
from tests.instances import llama_problem


# ----------------------------------------------------------------------------- oracle backend
class OracleBackend:
    """Test-only compute backend: the CPU oracle (gemm.cpp / quantize.cpp restated)."""

    def pack(self, codes, group, scales, int_scales, amplifier):
        codes = np.ascontiguousarray(np.asarray(codes, np.int16))
        w = O.QuantizedTensor(codes, 4, O.SYMMETRIC, O.GROUP, group,
                              np.ascontiguousarray(np.asarray(scales, np.float64)),
                              np.zeros(0, np.int32))
        ks = np.ascontiguousarray(np.asarray(int_scales, np.int32))
        e = int(amplifier).bit_length() - 1
        return w, O.IntegerScaleSet(ks, int(amplifier), e)

    @staticmethod
    def _x(xq, sa):
        return O.QuantizedTensor(np.asarray(xq, np.int16), 8, O.SYMMETRIC, O.PER_TOKEN, 0,
                                 np.asarray(sa, np.float64), np.zeros(0, np.int32))

    def gemm(self, xq, sa, w, out_dtype):
        r = O.gemm_integer_scale(self._x(xq, sa), w[0], w[1])
        return torch.from_numpy(r.output.copy())

    def gemm_acc(self, xq, sa, w):
        r = O.gemm_integer_scale(self._x(xq, sa), w[0], w[1], record=True)
        assert np.abs(r.acc).max(initial=0) < 2 ** 31
        return torch.from_numpy(r.acc.astype(np.int32))

    def row_absmax(self, x):
        return torch.from_numpy(np.abs(np.asarray(x, np.float32)).max(axis=1))

    def quantize_amax(self, x, amax):
        # quantize.cpp:120-142 with the row max given: s = amax/127 (1 if 0),
        # q = llround(double(x) / s) (half away from zero), clamp [-128, 127]
        a = np.asarray(amax, np.float64)
        s = np.where(a == 0.0, 1.0, a / 127.0)
        y = np.asarray(x, np.float32).astype(np.float64) / s[:, None]
        q = np.clip(np.sign(y) * np.floor(np.abs(y) + 0.5), -128, 127).astype(np.int8)
        return torch.from_numpy(q), torch.from_numpy(s)

    def finalize(self, acc, sa, amplifier, out_dtype):
        e = int(amplifier).bit_length() - 1
        o = (np.asarray(acc, np.int64).astype(np.float64) * 2.0 ** -e) * np.asarray(sa)[:, None]
        return torch.from_numpy(o.astype(np.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, k, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, w, s, xf, _ = llama_problem(m, k, n, seed_w=5 + n, seed_x=9 + m)
        comm = par.TorchDistComm()
        be = OracleBackend()
        # column-parallel: replicated X, all-gathered output
        col = par.ColumnParallelLinear(w.values, w.scales, s.int_scales, s.amplifier, w.group,
                                       comm, be)
        out_c = col.forward(x.values, x.scales).numpy()
        # row-parallel from the float activation's K-slice (global per-token max)
        row = par.RowParallelLinear(w.values, w.scales, s.int_scales, s.amplifier, w.group,
                                    comm, be)
        xl = xf[:, row.shard.lo:row.shard.hi]
        xq_l, sa_l = row.quantize_local(torch.from_numpy(np.ascontiguousarray(xl)))
        out_r = row.forward_quantized(xq_l.numpy(), sa_l.numpy()).numpy()
        codes_ok = np.array_equal(xq_l.numpy().astype(np.int16),
                                  x.values[:, row.shard.lo:row.shard.hi])
        scales_ok = np.array_equal(sa_l.numpy(), x.scales)
        ref = O.gemm_integer_scale(x, w, s).output
        q.put((rank, np.array_equal(out_c.view(np.int32), ref.view(np.int32)),
               np.array_equal(out_r.view(np.int32), ref.view(np.int32)), codes_ok, scales_ok,
               (row.shard.lo, row.shard.hi), col.shard.widths))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,k,n", [(2, 3, 1024, 256), (3, 5, 1024, 300), (2, 1, 11008, 130)])
def test_tensor_parallel_gloo_matches_single_device(world, m, k, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, k, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    groups = k // 128
    for rank, col_ok, row_ok, codes_ok, scales_ok, (lo, hi), widths in res:
        assert col_ok, f"column-parallel differs on rank {rank}"
        assert row_ok, f"row-parallel differs on rank {rank}"
        assert codes_ok and scales_ok, f"sharded per-token quantization differs on rank {rank}"
        assert lo % 128 == 0 and hi % 128 == 0  # group boundaries
        assert sum(widths) == n
    # shards tile K exactly, even when the group count does not divide (86 groups)
    bounds = sorted(r[5] for r in res)
    assert bounds[0][0] == 0 and bounds[-1][1] == k
    assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
    assert groups >= world


def test_shard_helpers_partition_reference_layouts():
    rng = np.random.default_rng(0)
    k, n, g = 512, 7, 128
    codes = rng.integers(-8, 8, size=(k, n)).astype(np.int16)
    G = k // g
    units = np.arange(n * G, dtype=np.float64)  # unit c*G + t
    cols = [par.column_shard(codes, units, units.astype(np.int32), r, 3) for r in range(3)]
    assert np.array_equal(np.concatenate([c[0] for c in cols], axis=1), codes)
    assert np.array_equal(np.concatenate([c[1] for c in cols]), units)
    rows = [par.row_shard(codes, units, units.astype(np.int32), g, r, 3) for r in range(3)]
    assert np.array_equal(np.concatenate([r[0] for r in rows], axis=0), codes)
    for r in rows:
        g0, g1 = r[3]
        exp = np.array([c * G + t for c in range(n) for t in range(g0, g1)], np.float64)
        assert np.array_equal(r[1], exp)


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("world,m,k,n", [(2, 16, 4096, 1024), (4, 5, 11008, 512), (8, 16, 4096, 640)])
def test_tensor_parallel_shards_on_device_bit_exact(world, m, k, n):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2405_14597_b200 as isb
    dev = torch.device("cuda:0")
    x, w, s, xf, _ = llama_problem(m, k, n, seed_w=17 + n, seed_x=19 + m)
    ref = O.gemm_integer_scale(x, w, s).output
    be = par.CudaBackend(dev)
    codes = torch.from_numpy(w.values)
    xq_full = torch.from_numpy(x.values.astype(np.int8)).to(dev)
    sa_full = torch.from_numpy(x.scales).to(dev)
    # column-parallel
    outs = []
    for r in range(world):
        c, sc, ks, _ = par.column_shard(codes, w.scales, s.int_scales, r, world)
        pw = be.pack(c.contiguous(), w.group, sc, ks, s.amplifier)
        outs.append(be.gemm(xq_full, sa_full, pw, torch.float32))
    out_c = torch.cat(outs, dim=1).cpu().numpy()
    assert np.array_equal(out_c.view(np.int32), ref.view(np.int32))
    # row-parallel from the float activation: partial maxes -> MAX -> local quantize
    xf_d = torch.from_numpy(xf).to(dev)
    shards = [par.row_shard(codes, w.scales, s.int_scales, w.group, r, world) for r in range(world)]
    amaxes = [be.row_absmax(xf_d[:, g0 * 128:g1 * 128]) for *_, (g0, g1) in shards]
    amax = torch.stack(amaxes).max(dim=0).values
    acc = None
    for (c, sc, ks, (g0, g1)) in shards:
        xq_l, sa_l = be.quantize_amax(xf_d[:, g0 * 128:g1 * 128].contiguous(), amax)
        assert torch.equal(xq_l.cpu(), xq_full[:, g0 * 128:g1 * 128].cpu())
        assert torch.equal(sa_l.cpu(), sa_full.cpu())
        pw = be.pack(c.contiguous(), w.group, sc, ks, s.amplifier)
        a = be.gemm_acc(xq_l, sa_l, pw)
        acc = a if acc is None else acc + a
    out_r = be.finalize(acc, sa_full, s.amplifier, torch.float32).cpu().numpy()
    assert np.array_equal(out_r.view(np.int32), ref.view(np.int32))
    full_acc = O.gemm_integer_scale(x, w, s, record=True).acc
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), full_acc)
    # bf16 epilogue of the reduced accumulator == bf16 of the float32 reference
    out_bf = be.finalize(acc, sa_full, s.amplifier, torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(out_bf, torch.from_numpy(ref).to(torch.bfloat16).float().numpy())
    assert isb.launch_count() > 0


def test_row_parallel_refuses_unsafe_layer():
    """The int32 all-reduce is exact only under the WHOLE layer's static bound
    (analysis.cpp:24-59): LLaMA-2-70B down_proj-like K=28672 at alpha=8192 style
    scales (k_g ~ 124) is unsafe although each 1/8 shard alone would be safe."""
    P = par
    from paper_2405_14597_b200._lib import OverflowError_
    k, n, g = 28672, 4, 128
    groups = k // g
    ks = np.full(n * groups, 124, np.int32)
    bound = P.static_bound(ks, groups, g)
    assert bound == groups * 128 * 127 * 8 * 124 and bound > 2**31 - 1
    assert P.static_bound(ks.reshape(n, groups)[:, : groups // 8].ravel(), groups // 8, g) < 2**31
    ref = O.overflow_analyzer(k, g, 8, 4, O.IntegerScaleSet(ks, 8192, 13))
    assert ref["static_bound"] == bound and not ref["safe"]

    class _Comm:
        rank, world = 0, 8

    with pytest.raises(OverflowError_):
        P.RowParallelLinear(np.zeros((k, n), np.int16), np.full(n * groups, 1e-3), ks, 8192, g,
                            _Comm(), OracleBackend())
