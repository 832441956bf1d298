"""Data-parallel GSR-GNN training (BASELINE.json configs[3]).

The reference is single-process (SPEC.md:16 puts multi-device training out of
scope); this is the B200 build's one cross-GPU step. Each rank trains
full-batch on its own sampled subgraph — the graphs are disjoint, so the
aggregation needs no halo — and the ranks exchange exactly one message per
step: the all-reduce (average) of the flat FP32 gradient buffer
(`gsrc_grads_device`, the GSRP parameter order). The optimizer then runs
identically on every rank, so the replicas stay bit-identical.

    step = DataParallelStep(ctx, lr=1e-4)     # torch.distributed already initialised
    loss = step()                              # fwd + loss + bwd → all_reduce(avg) → Adam

The backend is anything with `forward_backward() -> float`,
`optimizer_step(lr=...)` and `grads_tensor()` (a torch view of the flat
gradient buffer): the C-ABI `Context` on a GPU (NCCL over NVLink), or the CPU
test double in tests/test_dp_gloo.py (gloo).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def device_grads_tensor(ctx, device: int) -> torch.Tensor:
    """torch view of the context's flat gradient buffer, reduced in place by NCCL."""
    ptr, n = ctx.grads_device()
    return torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{device}")


def average_gradients(grads: torch.Tensor, group=None) -> None:
    """In-place average over the ranks of `group` (C1 in SURVEY.md §2.3).

    NCCL reduces with ReduceOp.AVG in one call; gloo has no AVG, so it sums and
    scales by 1/P (a power of two for P ∈ {1,2,4,8}: the scale is exact).
    """
    world = dist.get_world_size(group)
    if world == 1:
        return
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(grads, op=dist.ReduceOp.AVG, group=group)
    else:
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
        grads.mul_(1.0 / world)


class DataParallelStep:
    """fwd + loss + bwd on the local subgraph → gradient all-reduce → optimizer.

    With one rank (or no process group) this is the fused `train_step` of the
    backend, which a CUDA graph replays as one launch sequence.
    """

    def __init__(self, ctx, lr: float = 1e-3, group=None, grads: torch.Tensor | None = None, **optim):
        self.ctx = ctx
        self.lr = lr
        self.optim = optim
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.grads = grads
        if self.world > 1 and self.grads is None:
            self.grads = ctx.grads_tensor()

    def __call__(self) -> float:
        if self.world == 1:
            return self.ctx.train_step(lr=self.lr, **self.optim)
        loss = self.ctx.forward_backward()
        average_gradients(self.grads, self.group)
        self.ctx.optimizer_step(lr=self.lr, **self.optim)
        return loss


def replicas_identical(params: torch.Tensor, group=None) -> bool:
    """True iff every rank holds bit-identical parameters (max-min over ranks)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return True
    hi = params.clone()
    lo = params.clone()
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    return bool(torch.equal(hi, lo))
