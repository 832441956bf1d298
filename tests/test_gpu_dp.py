"""Data-parallel step on the device path (paper_2603_27156_b200/dp.py).

With one B200 the NCCL process group has one rank, but every call still runs:
* the split path — forward_backward → torch NCCL all_reduce(AVG) on the
  context's gradient buffer (Context.grads_tensor(), a zero-copy view) → host
  sync of the reducing stream → optimizer_step — must give bit-identical
  losses and parameters to the fused gsrc_train_step;
* the native path — the library's own communicator (gsrc_comm_init), the
  all-reduce enqueued on the context stream between backward and Adam — must
  too (AVG over one rank is the identity).
A two-rank NCCL run needs two GPUs; it is skipped on a one-GPU box (the CPU
gloo test at world size 2, tests/test_dp_gloo.py, covers the host logic).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

L, D, C, K, D_IN = 3, 256, 4, 16, 8


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _ctx(graph=True, seed=0):
    from paper_2603_27156_b200 import GEMM_TF32, MODE_GSRC, Context, model, synth
    g, nd = synth.generate_synthetic(synth.SynthConfig(n=20000, hub_fraction=0.002, hub_degree_range=(20, 900), seed=seed))
    c = Context(0)
    c.graph_upload(g.row_ptr, g.col_idx, norm=1)
    c.model_init(MODE_GSRC, L, D, C, K, D_IN, gemm=GEMM_TF32)
    c.set_params(model.init_params(MODE_GSRC, L, D, C, D_IN, seed=1))
    c.data_upload(nd.features, nd.labels, nd.train_mask)
    c.set_graph_capture(graph)
    return c


def _run(step, ctx, n=3):
    losses = [step() for _ in range(n)]
    return losses, ctx.params().copy()


def test_split_path_matches_fused_train_step(pg):
    from paper_2603_27156_b200.dp import DataParallelStep
    a = _ctx()
    fused = DataParallelStep(a, lr=1e-3)
    assert not fused.split and not fused.native
    la, pa = _run(fused, a)
    b = _ctx()
    split = DataParallelStep(b, lr=1e-3, fused=False)
    assert split.split and split.grads.data_ptr() == b.grads_device()[0]
    lb, pb = _run(split, b)
    assert la == lb
    assert np.array_equal(pa.view(np.uint32), pb.view(np.uint32))
    a.close()
    b.close()


def test_native_comm_matches_train_step(pg):
    from paper_2603_27156_b200 import Context
    from paper_2603_27156_b200.dp import init_native_comm
    a = _ctx()
    la, pa = _run(lambda: a.train_step(lr=1e-3), a)
    b = _ctx()
    init_native_comm(b)
    lb, pb = _run(lambda: b.train_step(lr=1e-3), b)
    assert la == lb
    assert np.array_equal(pa.view(np.uint32), pb.view(np.uint32))
    # the explicit all-reduce entry point (split path inside the library)
    g0 = b.grads().copy()
    b.comm_allreduce_grads()
    assert np.array_equal(g0, b.grads())
    b.comm_destroy()
    with pytest.raises(Exception):
        b.comm_allreduce_grads()
    uid = Context.comm_unique_id()
    assert len(uid) == 128
    a.close()
    b.close()


def test_stream_binding_orders_torch_work():
    """The context stream is exposed (gsrc_get_stream) so torch can order its
    work with the library's; binding to the legacy default stream is refused."""
    from paper_2603_27156_b200 import ConfigError
    c = _ctx(graph=False)
    s_own = c.stream_ptr()
    assert s_own != 0
    with pytest.raises(ConfigError):
        c.set_stream(0)
    ts = torch.cuda.Stream()
    c.set_stream(ts.cuda_stream)
    assert c.stream_ptr() == ts.cuda_stream
    with torch.cuda.stream(ts):
        g = c.grads_tensor()
        l0 = c.forward_backward()
        g.mul_(0.0)                      # enqueued on ts after the backward
        c.optimizer_step(lr=1e-3)        # Adam on ts sees zero gradients
    assert np.isfinite(l0)
    assert not np.any(c.grads())
    c.set_stream(None)
    assert c.stream_ptr() == s_own
    c.close()


def test_optim_state_roundtrip_exact_resume():
    """Adam m, v and the step count restore exactly: a resumed run continues the
    interrupted trajectory bit for bit (SPEC.md:293 checkpoint + optimizer state)."""
    a = _ctx()
    for _ in range(2):
        a.train_step(lr=1e-3)
    p, (m, v, t) = a.params().copy(), a.optim_state()
    assert t == 2 and np.any(m) and np.any(v)
    la = [a.train_step(lr=1e-3) for _ in range(2)]
    b = _ctx()
    b.set_params(p)
    b.set_optim_state(m, v, t)
    lb = [b.train_step(lr=1e-3) for _ in range(2)]
    assert la == lb
    assert np.array_equal(a.params().view(np.uint32), b.params().view(np.uint32))
    a.close()
    b.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_native_comm_two_ranks():
    import torch.multiprocessing as mp
    port = _port()
    mp.spawn(_two_rank_worker, args=(port,), nprocs=2, join=True)


def _two_rank_worker(rank, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=2, device_id=torch.device("cuda", rank))
    from paper_2603_27156_b200.dp import DataParallelStep, replicas_identical
    from paper_2603_27156_b200 import GEMM_TF32, MODE_GSRC, Context, model, synth
    g, nd = synth.generate_synthetic(synth.SynthConfig(n=20000, seed=rank))
    c = Context(rank)
    c.graph_upload(g.row_ptr, g.col_idx, norm=1)
    c.model_init(MODE_GSRC, L, D, C, K, D_IN, gemm=GEMM_TF32)
    c.set_params(model.init_params(MODE_GSRC, L, D, C, D_IN, seed=1))
    c.data_upload(nd.features, nd.labels, nd.train_mask)
    step = DataParallelStep(c, lr=1e-3)
    assert step.native
    for _ in range(3):
        step()
    p = torch.from_numpy(c.params()).cuda(rank)
    assert replicas_identical(p)
    dist.destroy_process_group()
