"""Device WorkCounter against the oracle's, and the SPEC's work
scaling acceptance.

The device counts the SPEC operations each entry point executes with the
oracle's accounting (include/gsr_cuda.h gsrc_work_counter): a layer forward or
inverse, a full training step (forward + backward with inverse recomputation),
and the op-level spmm / spmm_sparse / gsr_forward_block / gsr_backward_block
must give exactly the oracle's scalar multiply-adds on the same graph.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2603_27156_b200 import Context
    return Context(0)


def _graph(n=3000, seed=0):
    from paper_2603_27156_b200 import synth
    return synth.generate_synthetic(synth.SynthConfig(n=n, hub_fraction=0.005, hub_degree_range=(20, 200), seed=seed))


@pytest.mark.parametrize("mode_name,C,use_weight", [("gsrc", 4, True), ("gsrc", 4, False), ("alg12", 2, True), ("alg12", 2, False), ("rev", 4, True)])
def test_step_and_layer_work_match_oracle(ctx, oracle, mode_name, C, use_weight):
    from paper_2603_27156_b200 import GEMM_FP32, MODE_ALG12, MODE_GSRC, MODE_REV, model
    mode = {"gsrc": MODE_GSRC, "alg12": MODE_ALG12, "rev": MODE_REV}[mode_name]
    g, nd = _graph()
    L, D, k, d_in = 2, 64, 4, 8
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(mode, L, D, C, k, d_in, use_weight=use_weight, gemm=GEMM_FP32)
    p = model.init_params(mode, L, D, C, d_in, seed=1)
    ctx.set_params(p)
    ctx.data_upload(nd.features, nd.labels, nd.train_mask)
    og = oracle.Graph(g.row_ptr, g.col_idx, norm=1)
    net = oracle.Net(og, mode, L, D, C, k, d_in, use_weight=use_weight, dtype=np.float32)
    net.set_params(p)
    # one training step (forward + loss + backward with inverse recomputation)
    ctx.work_reset()
    ctx.forward_backward()
    oracle.work_reset()
    net.loss_grads(nd.features, nd.labels, nd.train_mask)
    step_ma, _ = ctx.work_counter()
    assert step_ma == oracle.work_muladds()
    if mode != MODE_REV:
        assert step_ma > 0
    # a single layer forward (and, for the reversible modes, its inverse)
    x = np.random.default_rng(2).normal(size=(g.n, D)).astype(np.float32)
    ctx.set_activation(x)
    ctx.work_reset()
    ctx.layer_forward(0)
    oracle.work_reset()
    y = net.layer_forward(0, x)
    assert ctx.work_counter()[0] == oracle.work_muladds()
    if mode != MODE_ALG12:
        ctx.work_reset()
        ctx.layer_inverse(0)
        oracle.work_reset()
        net.layer_inverse(0, y)
        assert ctx.work_counter()[0] == oracle.work_muladds()


def test_op_work_match_oracle_and_scaling(ctx, oracle):
    """spmm e·cols, spmm_sparse e·k (+ n rows each), gsr_forward_block e·k + n·w²,
    gsr_backward_block e·k + n·w² + e·w; and SPEC acceptance 6: the aggregation
    stage's count for k vs 4k differs by exactly 4×, for k = 4 vs 64 by 16×."""
    g, _ = _graph(n=2000, seed=3)
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    og = oracle.Graph(g.row_ptr, g.col_idx, norm=1)
    rng = np.random.default_rng(4)
    w = 64
    x = rng.normal(size=(g.n, w)).astype(np.float32)
    W = rng.normal(size=(w, w)).astype(np.float32) * 0.1

    def both(dev_fn, ora_fn):
        ctx.work_reset()
        dev_fn()
        oracle.work_reset()
        ora_fn()
        dev = ctx.work_counter()
        assert dev[0] == oracle.work_muladds(), (dev, oracle.work_muladds())
        return dev

    ma, rows = both(lambda: ctx.spmm(x), lambda: oracle.spmm(og, x))
    assert ma == g.e * w and rows == g.n
    agg = {}
    for k in (4, 16, 64):
        vals, idx = oracle.gs_topk(x, k)
        ma, rows = both(lambda: ctx.spmm_sparse(vals, idx, w), lambda: oracle.spmm_sparse(og, vals, idx, w))
        assert rows == g.n
        agg[k] = ma
        both(lambda: ctx.block_forward(vals, idx, W, width=w, use_weight=True), lambda: oracle.block_fwd(og, vals, idx, W, width=w))
        both(lambda: ctx.block_forward(vals, idx, W, width=w, use_weight=False), lambda: oracle.block_fwd(og, vals, idx, W, width=w, use_weight=False))
        both(lambda: ctx.block_backward(x, idx, vals, idx, W), lambda: oracle.block_bwd(og, x, idx, vals, idx, W))
    assert agg[16] == 4 * agg[4] and agg[64] == 16 * agg[4]
