"""Data-parallel step (paper_2603_27156_b200/dp.py) at world_size 2 on CPU (gloo).

The GPU backend is replaced by a CPU double that runs the oracle (the checker)
for fwd + loss + bwd and Adam, so the DP orchestration — one all-reduce of the
flat gradient buffer per step, then the same optimizer on every rank — is
checked here without a GPU against the SURVEY.md §8e parity rule: the oracle
computes each rank's gradient sequentially and averages them in rank order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

L, D, C, K, D_IN = 2, 32, 2, 4, 8
LR = 1e-3
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(rank):
    from paper_2603_27156_b200 import synth
    return synth.generate_synthetic(synth.SynthConfig(n=300, hub_fraction=0.01, hub_degree_range=(10, 40), seed=rank))


class OracleBackend:
    """CPU stand-in for the C-ABI Context: same methods DataParallelStep uses."""

    def __init__(self, rank):
        from oracle import oracle as o
        from paper_2603_27156_b200 import MODE_GSRC, init_params
        self.o = o
        g, nd = _inputs(rank)
        self.og = o.Graph(g.row_ptr, g.col_idx, norm=1)
        self.nd = nd
        self.net = o.Net(self.og, MODE_GSRC, L, D, C, K, D_IN, dtype=np.float32)
        self.net.set_params(init_params(MODE_GSRC, L, D, C, D_IN, seed=1))
        P = self.net.P
        self.g = torch.zeros(P, dtype=torch.float32)
        self.m = np.zeros(P, np.float32)
        self.v = np.zeros(P, np.float32)
        self.t = 0

    def forward_backward(self):
        loss, grads, _, _ = self.net.loss_grads(self.nd.features, self.nd.labels, self.nd.train_mask)
        self.g.copy_(torch.from_numpy(grads))
        return loss

    def grads_tensor(self):
        return self.g

    def optimizer_step(self, lr):
        self.t += 1
        p = self.net.params()
        self.o.adam(p, self.g.numpy(), self.m, self.v, self.t, lr=lr)
        self.net.set_params(p)

    def train_step(self, lr):
        loss = self.forward_backward()
        self.optimizer_step(lr)
        return loss


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_27156_b200.dp import DataParallelStep, replicas_identical
    be = OracleBackend(rank)
    step = DataParallelStep(be, lr=LR)
    losses = [step() for _ in range(STEPS)]
    p = torch.from_numpy(be.net.params())
    same = replicas_identical(p)
    np.save(os.path.join(out_dir, f"p{rank}.npy"), p.numpy())
    np.save(os.path.join(out_dir, f"l{rank}.npy"), np.array(losses + [float(same)]))
    dist.destroy_process_group()


def _sequential_reference(world):
    """Oracle-only: per-rank gradients averaged in fixed rank order, one Adam."""
    from oracle import oracle as o
    backs = [OracleBackend(r) for r in range(world)]
    m = np.zeros(backs[0].net.P, np.float32)
    v = np.zeros_like(m)
    p = backs[0].net.params()
    for t in range(1, STEPS + 1):
        gs = []
        for b in backs:
            b.net.set_params(p)
            b.forward_backward()
            gs.append(b.g.numpy().copy())
        g = gs[0].copy()
        for x in gs[1:]:
            g += x
        g *= np.float32(1.0 / world)
        o.adam(p, g, m, v, t, lr=LR)
    return p


def test_dp_gloo_world2_matches_sequential_average(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    p0 = np.load(tmp_path / "p0.npy")
    p1 = np.load(tmp_path / "p1.npy")
    assert np.array_equal(p0, p1), "replicas diverged"
    assert np.load(tmp_path / "l0.npy")[-1] == 1.0 and np.load(tmp_path / "l1.npy")[-1] == 1.0
    ref = _sequential_reference(world)
    scale = np.abs(ref).max()
    assert np.abs(p0 - ref).max() <= 1e-5 * scale
    # each rank's loss is its own subgraph's loss: they differ
    assert np.load(tmp_path / "l0.npy")[0] != np.load(tmp_path / "l1.npy")[0]


def test_dp_single_rank_is_fused_train_step():
    from paper_2603_27156_b200.dp import DataParallelStep
    be = OracleBackend(0)
    calls = []
    be.train_step = lambda lr: calls.append(lr) or 0.0
    DataParallelStep(be, lr=LR)()
    assert calls == [LR]


def test_average_gradients_sum_then_exact_scale():
    from paper_2603_27156_b200 import dp
    assert not dist.is_initialized()
    x = torch.ones(4)
    with pytest.raises(Exception):
        dp.average_gradients(x)  # no process group: refuses instead of silently skipping


class _FakeCommCtx:
    """Records what init_native_comm hands the C-ABI (gsrc_comm_unique_id / gsrc_comm_init)."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def comm_unique_id(self):
        return bytes([7] * 128)

    def comm_init(self, uid, nranks, rank):
        self.calls.append((uid, nranks, rank))


def _comm_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_27156_b200.dp import DataParallelStep, init_native_comm
    c = _FakeCommCtx(rank)
    init_native_comm(c)
    assert c.calls == [(bytes([7] * 128), world, rank)]
    # gloo never takes the native path (it needs NCCL): the split path with a CPU gradient view
    be = OracleBackend(rank)
    step = DataParallelStep(be, lr=LR)
    assert step.split and not step.native
    np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([1]))
    dist.destroy_process_group()


def test_native_comm_id_broadcast_world2(tmp_path):
    world = 2
    mp.spawn(_comm_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}.npy").exists() for r in range(world))
