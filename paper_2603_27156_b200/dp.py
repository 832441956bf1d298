"""Data-parallel GSR-GNN training (BASELINE.json configs[3]).

The reference is single-process (SPEC.md:16 puts multi-device training out of
scope); this is the B200 build's one cross-GPU step. Each rank trains
full-batch on its own sampled subgraph — the graphs are disjoint, so the
aggregation needs no halo — and the ranks exchange exactly one message per
step: the all-reduce (average) of the flat FP32 gradient buffer (GSRP
parameter order). The optimizer then runs identically on every rank, so the
replicas stay bit-identical.

    step = DataParallelStep(ctx, lr=1e-4)     # torch.distributed already initialised
    loss = step()                              # fwd + loss + bwd → all_reduce(avg) → Adam

Two paths:
* native (the default for a C-ABI Context under an NCCL process group): the
  library owns an NCCL communicator (gsrc_comm_init; torch.distributed only
  broadcasts the unique id) and gsrc_train_step enqueues forward, backward,
  ncclAllReduce(avg) and Adam on the context's one stream — ordered by the
  stream itself, the forward/backward/optimizer parts replayed as CUDA graphs;
* split (gloo, the CPU test double of tests/test_dp_gloo.py, or fused=False):
  forward_backward → torch all_reduce on grads_tensor() → host sync of the
  reducing stream → optimizer_step, so Adam never reads a partly reduced
  buffer and the next step's zero_grads never races the reduction.
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


def average_gradients(grads: torch.Tensor, group=None, force: bool = False) -> None:
    """In-place average over the ranks of `group` (C1 in SURVEY.md §2.3), complete on return.

    NCCL reduces with ReduceOp.AVG in one call; gloo has no AVG, so it sums and
    scales by 1/P (a power of two for P ∈ {1,2,4,8}: the scale is exact). On a
    device tensor the reducing stream is synchronised before returning, so work
    the caller enqueues on another stream (the context's) sees the result.
    `force` runs the collective even for one rank (tests of the split path).
    """
    world = dist.get_world_size(group)
    if world == 1 and not force:
        return
    if dist.get_backend(group) == "nccl":
        work = dist.all_reduce(grads, op=dist.ReduceOp.AVG, group=group, async_op=True)
        work.wait()
    else:
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
        grads.mul_(1.0 / world)
    if grads.is_cuda:
        torch.cuda.current_stream(grads.device).synchronize()


def init_native_comm(ctx, group=None) -> None:
    """Give the context its own NCCL communicator over the ranks of `group`:
    rank 0 of the group creates the unique id, torch.distributed broadcasts it."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = [ctx.comm_unique_id() if rank == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    ctx.comm_init(obj[0], world, rank)


class DataParallelStep:
    """fwd + loss + bwd on the local subgraph → gradient all-reduce → optimizer.

    One rank: the backend's fused `train_step`. Several ranks under NCCL with a
    C-ABI Context: the native path (see the module docstring). Otherwise, or
    with fused=False: the split path.
    """

    def __init__(self, ctx, lr: float = 1e-3, group=None, grads: torch.Tensor | None = None, fused: bool | None = None, **optim):
        self.ctx = ctx
        self.lr = lr
        self.optim = optim
        self.group = group
        ddp = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if ddp else 1
        nccl = ddp and dist.get_backend(group) == "nccl"
        self.native = bool(nccl and hasattr(ctx, "comm_init") and fused is not False and self.world > 1)
        self.split = fused is False or (self.world > 1 and not self.native)
        self.grads = grads
        if self.native:
            init_native_comm(ctx, group)
        elif self.split and self.grads is None:
            self.grads = ctx.grads_tensor()

    def __call__(self) -> float:
        if not self.split:
            return self.ctx.train_step(lr=self.lr, **self.optim)
        loss = self.ctx.forward_backward()
        average_gradients(self.grads, self.group, force=True)
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
