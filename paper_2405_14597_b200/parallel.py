"""Tensor parallelism for the integer-scale W4A8 linear layer.

The reference is a single host process (gemm.cpp:55-100 only splits output rows
over std::threads), so there is no reference interface here; this module is the
multi-GPU layer the north star asks for, built on the same C ABI kernels:

* ColumnParallelLinear — rank r owns output channels [N r/P, N (r+1)/P): its
  int4 codes, its group scales and its integer scales are one contiguous slice
  of the reference layouts (unit c*(K/g) + k/g, quantize.cpp:51). The
  activation is replicated; every rank computes its [M, N/P] slice with the
  integer-scale GEMM and the slices are all-gathered (exact: no cross-rank
  arithmetic).
* RowParallelLinear — rank r owns quantization groups [G r/P, G (r+1)/P) (K is
  split on group boundaries, shards may be uneven, e.g. LLaMA-2-7B down_proj
  has 86 groups). The activation arrives K-sharded, so the per-token scale needs
  the full-row absmax (quantize.cpp:120-125): each rank takes its partial row
  max, the ranks all-reduce MAX, and each rank quantizes its slice with the
  global max — the codes are then exactly the slice of the full-row
  quantization. Each rank produces the raw int32 accumulator of its groups
  (sum_g P_g k_g, gemm.cpp:245-247), the ranks all-reduce SUM in int32 — exact
  and order-independent whenever overflow_analyzer calls the whole layer safe,
  because every partial sum is bounded by the full static bound — and the Eq. 2
  epilogue (gemm.cpp:252) runs once on the reduced accumulator. The output is
  therefore bit-identical to the single-GPU layer.

Collectives go through a small Comm interface; TorchDistComm wraps
torch.distributed (NCCL over NVLink on B200, gloo in the CPU tests). The compute
backend defaults to the CUDA kernels (paper_2405_14597_b200.ops); the CPU tests
inject the oracle as the checker.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops


# ----------------------------------------------------------------------------- partitioning
def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of n units: rank r gets [n r/P, n (r+1)/P)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return n * rank // world, n * (rank + 1) // world


def column_shard(codes, scales, int_scales, rank: int, world: int):
    """Output channels [n0, n1) of a K x N weight: codes[:, n0:n1]; the scales and
    integer scales of those channels are the contiguous slice [n0 G, n1 G) of the
    reference unit order c*G + g (quantize.cpp:51)."""
    k, n = codes.shape
    g_count = len(scales) // n
    n0, n1 = shard_bounds(n, world, rank)
    ks = None if int_scales is None else int_scales[n0 * g_count:n1 * g_count]
    return codes[:, n0:n1], scales[n0 * g_count:n1 * g_count], ks, (n0, n1)


def static_bound(int_scales, groups: int, group: int, act_bits=8, w_bits=4) -> int:
    """overflow_analyzer's bound (analysis.cpp:24-59): max over output channels of
    sum_g group * A_max * W_max * k_g, in exact Python integers."""
    if isinstance(int_scales, torch.Tensor):
        int_scales = int_scales.detach().cpu().numpy()
    ks = np.asarray(int_scales, np.int64).reshape(-1, groups)
    per_mac = group * ((1 << (act_bits - 1)) - 1) * (1 << (w_bits - 1))
    return int(max(int(v) for v in ks.sum(axis=1))) * per_mac if ks.size else 0


def require_int32_safe(int_scales, groups: int, group: int, what: str):
    """The int32 all-reduce of row-parallel partial accumulators equals the
    reference's int64 acc only if the WHOLE layer's static bound fits int32 (each
    shard's bound is smaller, so the per-rank kernels' own gate is not enough)."""
    b = static_bound(int_scales, groups, group)
    if b > (1 << 31) - 1:
        from ._lib import OverflowError_
        raise OverflowError_(f"{what}: static overflow bound {b} exceeds int32 "
                             "(analysis.cpp:24-59); the int32 accumulator exchange "
                             "would not be exact")
    return b


def row_shard(codes, scales, int_scales, group: int, rank: int, world: int):
    """Quantization groups [g0, g1) of a K x N weight (K split on group boundaries):
    codes rows [g0 g, g1 g) and, per output channel c, units c*G + [g0, g1)."""
    k, n = codes.shape
    g_count = k // group
    g0, g1 = shard_bounds(g_count, world, rank)

    def take(u):
        if u is None:
            return None
        if isinstance(u, torch.Tensor):
            return u.reshape(n, g_count)[:, g0:g1].contiguous().reshape(-1)
        return np.ascontiguousarray(np.asarray(u).reshape(n, g_count)[:, g0:g1]).reshape(-1)

    return codes[g0 * group:g1 * group, :], take(scales), take(int_scales), (g0, g1)


# ----------------------------------------------------------------------------- collectives
class Comm:
    """Collectives the layers need; rank order is the concatenation order."""
    rank: int = 0
    world: int = 1

    def all_gather_cols(self, t: torch.Tensor, widths: list[int]) -> torch.Tensor:
        raise NotImplementedError

    def all_reduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError

    def all_reduce_max_(self, t: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError


class TorchDistComm(Comm):
    """torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_cols(self, t, widths):
        # ranks may own different column counts: pad to the widest, gather, trim, concat
        w = max(widths)
        m = t.shape[0]
        buf = torch.zeros((m, w), dtype=t.dtype, device=t.device)
        buf[:, :t.shape[1]] = t
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(parts, buf.contiguous(), group=self.group)
        return torch.cat([p[:, :wi] for p, wi in zip(parts, widths)], dim=1)

    def all_reduce_sum_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_max_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t


# ----------------------------------------------------------------------------- compute backend
class CudaBackend:
    """The product path: every call is a kernel of libintscale_b200.so."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.ws = ops.Workspace()

    def pack(self, codes, group, scales, int_scales, amplifier):
        return ops.PackedWeight.from_codes(torch.as_tensor(codes).to(self.device), group,
                                           scales, int_scales, amplifier)

    def gemm(self, xq, sa, w, out_dtype):
        return ops.gemm_integer_scale(xq, sa, w, out_dtype=out_dtype, workspace=self.ws)

    def gemm_acc(self, xq, sa, w):
        return ops.gemm_integer_scale(xq, sa, w, out_dtype=torch.int32, workspace=self.ws)

    def row_absmax(self, x):
        return ops.row_absmax(x)

    def quantize_amax(self, x, amax):
        return ops.quantize_per_token_amax(x, amax)

    def finalize(self, acc, sa, amplifier, out_dtype):
        return ops.finalize_acc(acc, sa, amplifier, out_dtype=out_dtype)


# ----------------------------------------------------------------------------- layers
@dataclass
class ShardInfo:
    lo: int
    hi: int
    widths: list


class ColumnParallelLinear:
    """N-split integer-scale W4A8 linear; output all-gathered to [M, N]."""

    def __init__(self, codes, scales, int_scales, amplifier: int, group: int, comm: Comm,
                 backend):
        n = codes.shape[1]
        c, s, ks, (n0, n1) = column_shard(codes, scales, int_scales, comm.rank, comm.world)
        self.comm, self.backend, self.amplifier = comm, backend, amplifier
        self.shard = ShardInfo(n0, n1, [shard_bounds(n, comm.world, r)[1] -
                                        shard_bounds(n, comm.world, r)[0]
                                        for r in range(comm.world)])
        self.weight = backend.pack(c, group, s, ks, amplifier)

    def forward(self, xq, sa, out_dtype=torch.bfloat16, gather=True):
        local = self.backend.gemm(xq, sa, self.weight, out_dtype)
        if not gather or self.comm.world == 1:
            return local
        return self.comm.all_gather_cols(local, self.shard.widths)


class RowParallelLinear:
    """K-split (group-boundary) integer-scale W4A8 linear with an exact int32
    all-reduce of the scaled accumulator, then one Eq. 2 epilogue."""

    def __init__(self, codes, scales, int_scales, amplifier: int, group: int, comm: Comm,
                 backend):
        require_int32_safe(int_scales, codes.shape[0] // group, group, "RowParallelLinear")
        c, s, ks, (g0, g1) = row_shard(codes, scales, int_scales, group, comm.rank, comm.world)
        self.comm, self.backend, self.amplifier, self.group = comm, backend, amplifier, group
        self.shard = ShardInfo(g0 * group, g1 * group, [])
        self.weight = backend.pack(c, group, s, ks, amplifier)

    def quantize_local(self, x_local):
        """Per-token int8 quantization of this rank's K-slice with the global row max."""
        amax = self.backend.row_absmax(x_local)
        self.comm.all_reduce_max_(amax)
        return self.backend.quantize_amax(x_local, amax)

    def forward_quantized(self, xq_local, sa, out_dtype=torch.bfloat16):
        acc = self.backend.gemm_acc(xq_local, sa, self.weight)
        self.comm.all_reduce_sum_(acc)
        return self.backend.finalize(acc, sa, self.amplifier, out_dtype)

    def forward(self, x_local, out_dtype=torch.bfloat16):
        xq, sa = self.quantize_local(x_local)
        return self.forward_quantized(xq, sa, out_dtype)
