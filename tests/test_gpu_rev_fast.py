"""rev-baseline (RevGNN-style dense blocks) on the
tcgen05 fast path in TF32 mode: FWD / INV with a dense Â·relu(u) aggregation
(k_fast<W, *, -1>, dense hub rows by k_hub_seg_dense + k_hub_fold with relu)
and BIN with S = relu(u) and the mask u > 0 (k_bin2<W, 2, true>), against the
TF32 oracle (dW in the device's relu(u)ᵀ·(Âᵀ·G) form).

Bounds: no GS masks here, so the only difference is the tensor core's
accumulation order inside each TF32 transform (and the rare relu mask of a u
within rounding of 0): rows within 1e-4 of scale, parameter gradients within
1e-3. The inverse is exact on the residual grid: forward then inverse returns
the layer input bit for bit."""
import os

import numpy as np
import pytest

from tests.gpu_helpers import block_max_rel, make_graph

pytestmark = pytest.mark.gpu

ROW_RTOL = 1e-4
GRAD_RTOL = 1e-3


@pytest.fixture(scope="module")
def ctx():
    from paper_2603_27156_b200 import Context
    return Context(0)


@pytest.fixture
def oracle_tf32(oracle):
    oracle.set_tf32(True)
    yield oracle
    oracle.set_tf32(False)


def _rel_rows(a, b):
    return np.abs(a - b).max(axis=1) / max(float(np.abs(b).max()), 1e-30)


@pytest.mark.parametrize("D,C,bias", [(256, 4, False), (128, 4, True), (64, 2, False), (256, 8, False)])
def test_rev_fast_layer_fwd_inv_bwd(ctx, oracle_tf32, D, C, bias):
    from paper_2603_27156_b200 import GEMM_TF32, MODE_REV, model
    oracle = oracle_tf32
    n = 6000
    g = make_graph(n, seed=D + C)
    assert np.diff(g.row_ptr).max() > 8                     # dense hub rows on both directions
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    og = oracle.Graph(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(MODE_REV, 1, D, C, 4, 8, use_bias=bias, gemm=GEMM_TF32)
    net = oracle.Net(og, MODE_REV, 1, D, C, 4, 8, use_bias=bias, dtype=np.float32)
    p = model.init_params(MODE_REV, 1, D, C, 8, seed=7)
    ctx.set_params(p)
    net.set_params(p)
    rng = np.random.default_rng(D)
    x = (np.round(rng.normal(size=(n, D)) * 2.0 ** 20) * 2.0 ** -20).astype(np.float32)   # on the residual grid
    ctx.set_activation(x)
    l0 = ctx.kernel_launches()
    ctx.layer_forward(0)
    assert ctx.kernel_launches() > l0
    y = ctx.activation()
    ry = net.layer_forward(0, x)
    err = _rel_rows(y, ry)
    print(f"rev D={D} C={C}: forward rows max {err.max():.2e}")
    assert err.max() <= ROW_RTOL
    # the inverse runs the forward's kernels on the same inputs: the input comes back bit for bit
    ctx.layer_inverse(0)
    assert np.array_equal(ctx.activation(), x)
    # backward: inverse + dW/db + masked input gradient
    G = rng.normal(size=(n, D)).astype(np.float32)
    ctx.set_activation(y)
    ctx.set_gradient(G)
    ctx.zero_grads()
    net.zero_grads()
    ctx.layer_backward(0)
    rx, rg = net.layer_backward(0, y, G)
    assert _rel_rows(ctx.activation(), rx).max() <= ROW_RTOL
    gerr = _rel_rows(ctx.gradient(), rg)
    print(f"rev D={D} C={C}: input gradient rows max {gerr.max():.2e}")
    assert gerr.max() <= 10 * ROW_RTOL
    lay = model.param_layout(MODE_REV, 1, D, C, 8)
    perr = block_max_rel(ctx.grads(), net.grads(), lay)
    print(f"rev D={D} C={C}: dW/db block max {perr:.2e}")
    assert perr <= GRAD_RTOL


def test_rev_fast_train_step_matches_oracle(ctx, oracle_tf32):
    """a 4-layer rev-baseline step: loss and gradients vs the TF32 oracle, and
    the fast kernels are the ones that ran (k_tile would be the fallback)"""
    from paper_2603_27156_b200 import GEMM_TF32, MODE_REV, model, synth
    oracle = oracle_tf32
    g, nd = synth.generate_synthetic(synth.SynthConfig(n=20_000, hub_fraction=0.002, hub_degree_range=(30, 80), seed=3))
    L, D, C = 4, 256, 4
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(MODE_REV, L, D, C, 4, 8, gemm=GEMM_TF32)
    net = oracle.Net(oracle.Graph(g.row_ptr, g.col_idx, norm=1), MODE_REV, L, D, C, 4, 8, dtype=np.float32)
    p = model.init_params(MODE_REV, L, D, C, 8, seed=2)
    ctx.set_params(p)
    net.set_params(p)
    ctx.data_upload(nd.features, nd.labels, nd.train_mask)
    loss = ctx.forward_backward()
    rloss, rgrads, _, _ = net.loss_grads(nd.features, nd.labels, nd.train_mask)
    gerr = block_max_rel(ctx.grads(), rgrads, model.param_layout(MODE_REV, L, D, C, 8))
    print(f"rev step: loss rel {abs(loss - rloss) / abs(rloss):.2e}, grads {gerr:.2e}")
    assert abs(loss - rloss) <= 1e-4 * abs(rloss)
    assert gerr <= GRAD_RTOL
