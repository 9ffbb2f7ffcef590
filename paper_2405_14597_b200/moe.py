"""Expert-sharded Mixtral-style FFN on the integer-scale W4A8 GEMM (BASELINE config
C5, SURVEY §8e "Expert-sharded").

Each expert e owns three integer-scale W4A8 linears — w1 (gate) and w3 (up),
K -> F, fused into one K -> 2F weight, and w2 (down), F -> K — and lives on rank
e % world. A step takes T tokens with top-2 routing: every (token, slot) pair is a
row of its expert's batch, so each expert runs two hot-path GEMM instances on its
own routed rows (gemm.cpp:205-262 per expert, exact per expert):

    rows_e = x[tokens routed to e]                 (dispatch; all-to-all across ranks)
    h_e    = silu(rows_e @ w1_e) * (rows_e @ w3_e)  (K1 + K3 on the fused gate/up weight)
    y_e    = h_e @ w2_e                            (K1 + K3)
    out[t] = sum_slot weight[t, slot] * y_e[t]      (combine, fixed slot order)

Routing, SiLU and the combine are framework glue (torch ops on device); the
reference has no MoE, so only the per-expert GEMMs are hot path.
The combine sums the two slots in slot order on the token's home rank, so the
expert-sharded result is bit-identical to the single-device one.
"""
from __future__ import annotations

import torch

from . import ops


def route_top2(logits: torch.Tensor):
    """Top-2 routing (Mixtral): expert ids [T, 2] and softmax-of-top-2 weights."""
    w, idx = torch.topk(logits.float(), 2, dim=-1)
    return idx, torch.softmax(w, dim=-1)


class Expert:
    """One expert's three linears (w1/w3 fused into K x 2F) as PackedWeights."""

    def __init__(self, w13: ops.PackedWeight, w2: ops.PackedWeight, amplifier: int, act=None):
        self.w13, self.w2, self.amplifier = w13, w2, amplifier
        self.f = w2.k
        self.act = act or (lambda g, u: torch.nn.functional.silu(g) * u)

    def forward(self, rows: torch.Tensor, workspace=None) -> torch.Tensor:
        """rows: float32 [R, K] on device -> float32 [R, K]."""
        if rows.shape[0] == 0:
            return torch.zeros((0, self.w2.n), dtype=torch.float32, device=rows.device)
        xq, sa = ops.quantize_per_token(rows)
        gu = ops.gemm_integer_scale(xq, sa, self.w13, out_dtype=torch.float32, workspace=workspace)
        h = self.act(gu[:, :self.f], gu[:, self.f:])
        hq, hs = ops.quantize_per_token(h.contiguous())
        return ops.gemm_integer_scale(hq, hs, self.w2, out_dtype=torch.float32, workspace=workspace)


class ExpertParallelFFN:
    """Experts sharded over ranks (expert e on rank e % world). With world == 1 (or
    comm=None) every expert is local."""

    def __init__(self, experts_local: dict, n_experts: int, comm=None):
        self.experts = experts_local        # expert id -> Expert (only the local ones)
        self.n_experts = n_experts
        self.comm = comm
        self.world = 1 if comm is None else comm.world
        self.rank = 0 if comm is None else comm.rank
        self.ws = ops.Workspace()

    def owner(self, e: int) -> int:
        return e % self.world

    def forward(self, x: torch.Tensor, idx: torch.Tensor, weight: torch.Tensor) -> torch.Tensor:
        """x: float32 [T, K] (this rank's tokens), idx/weight: [T, 2] routing."""
        T, K = x.shape
        flat_e = idx.reshape(-1)                       # (token, slot) rows in slot order
        rows = x.repeat_interleave(2, dim=0)           # row r = token r // 2, slot r % 2
        y = torch.empty_like(rows)
        if self.world == 1:
            for e in range(self.n_experts):
                sel = torch.nonzero(flat_e == e).reshape(-1)
                if sel.numel():
                    y[sel] = self.experts[e].forward(rows[sel].contiguous(), self.ws)
        else:
            y = self._forward_distributed(rows, flat_e)
        out = y.view(T, 2, K)
        w = weight.to(out.dtype)
        return out[:, 0, :] * w[:, 0:1] + out[:, 1, :] * w[:, 1:2]  # fixed slot order

    def _forward_distributed(self, rows, flat_e):
        import torch.distributed as dist
        dev = rows.device
        owner = flat_e % self.world
        order = torch.argsort(owner * self.n_experts + flat_e, stable=True)
        send = rows[order].contiguous()
        send_e = flat_e[order].contiguous()
        counts = torch.bincount(owner, minlength=self.world).to(torch.int64)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts)
        sc, rc = counts.tolist(), recv_counts.tolist()
        recv = torch.empty((sum(rc), rows.shape[1]), dtype=rows.dtype, device=dev)
        recv_e = torch.empty((sum(rc),), dtype=send_e.dtype, device=dev)
        dist.all_to_all_single(recv, send, rc, sc)
        dist.all_to_all_single(recv_e, send_e, rc, sc)
        yl = torch.empty_like(recv)
        for e, ex in self.experts.items():
            sel = torch.nonzero(recv_e == e).reshape(-1)
            if sel.numel():
                yl[sel] = ex.forward(recv[sel].contiguous(), self.ws)
        back = torch.empty_like(send)
        dist.all_to_all_single(back, yl, sc, rc)
        y = torch.empty_like(rows)
        y[order] = back
        return y
