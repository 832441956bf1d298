"""Pin the CPU oracle against every golden vector in the reference SPEC.

The reference ships no tests or fixtures; the SPEC's
[PAPER]/[TRIVIAL] examples in tests/golden/spec_vectors.json are the only
external anchors. CPU-only.
"""
import numpy as np
import pytest


def _graph(oracle, golden, norm=0):
    g = golden["graph_4_1"]
    return oracle.Graph.from_edges(g["n"], g["edges"], norm=norm)


def test_csr_from_edge_list(oracle, golden):
    g = _graph(oracle, golden)
    rp, ci = g.csr()
    assert rp.tolist() == golden["graph_4_1"]["row_ptr"]
    assert ci.tolist() == golden["graph_4_1"]["col_idx"]


def test_csr_empty_and_dedup(oracle):
    g = oracle.Graph.from_edges(3, np.zeros((0, 2), np.int64))
    rp, ci = g.csr()
    assert rp.tolist() == [0, 0, 0, 0] and ci.size == 0
    g = oracle.Graph.from_edges(3, [[0, 1], [0, 1], [2, 0]])
    rp, ci = g.csr()
    assert rp.tolist() == [0, 1, 1, 2] and ci.tolist() == [1, 0]


def test_split_golden(golden):
    v = golden["split_4_3"]
    x = np.array(v["x"])
    w = x.shape[1] // v["parts"]
    assert np.array_equal(x[:, :w], np.array(v["first"]))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_gs_topk_golden(oracle, golden, dt):
    v = golden["gs_topk_4_3"]
    vals, idx = oracle.gs_topk(np.array(v["x"], dt), v["k"])
    assert np.array_equal(vals, np.array(v["values"], dt))
    assert idx.tolist() == v["indices"]


def test_gs_topk_zero_and_full(oracle, golden):
    v = golden["gs_topk_zero"]
    vals, idx = oracle.gs_topk(np.zeros((v["rows"], v["cols"])), v["k"])
    assert idx.tolist() == v["indices"] and not vals.any()
    x = np.random.default_rng(0).normal(size=(5, 6))
    vals, idx = oracle.gs_topk(x, 6)
    assert (idx == np.arange(6)).all() and np.array_equal(vals, x)


def test_gs_topk_bruteforce(oracle):
    rng = np.random.default_rng(1)
    for _ in range(50):
        w = int(rng.integers(1, 40))
        k = int(rng.integers(1, w + 1))
        x = rng.normal(size=(7, w))
        x[:, ::3] = np.round(x[:, ::3], 1)  # induce magnitude ties
        x[0, :] = -x[0, :]
        vals, idx = oracle.gs_topk(x, k)
        for r in range(7):
            order = sorted(range(w), key=lambda j: (-abs(x[r, j]), j))[:k]
            assert idx[r].tolist() == sorted(order)
            assert np.array_equal(vals[r], x[r, sorted(order)])


def test_scatter_golden(oracle, golden):
    v = golden["scatter_4_1"]
    d = oracle.scatter(np.array(v["values"]), np.array(v["indices"]), v["width"])
    assert np.array_equal(d, np.array(v["dense"]))


def test_spmm_golden(oracle, golden):
    g = _graph(oracle, golden)
    v = golden["spmm_4_1"]
    y = oracle.spmm(g, np.array(v["x"]))
    assert np.abs(y - np.array(v["y"])).max() <= 1e-12


def test_spmm_sparse_golden_bit_exact_f64(oracle, golden):
    """Acceptance criterion 1: bit-exact in 64-bit."""
    g = _graph(oracle, golden)
    v = golden["spmm_sparse_4_1"]
    y = oracle.spmm_sparse(g, np.array(v["values"]), np.array(v["indices"]), v["width"])
    assert np.array_equal(y, np.array(v["y"]))


def test_spmm_sparse_golden_f32(oracle, golden):
    """f32 compares against the f32-rounded oracle (0.79+0.86 != 1.65 in f32)."""
    g = _graph(oracle, golden)
    v = golden["spmm_sparse_4_1"]
    y = oracle.spmm_sparse(g, np.array(v["values"], np.float32), np.array(v["indices"]), v["width"])
    assert np.abs(y - np.array(v["y"], np.float32)).max() <= 1e-6
    assert y[2, 3] == np.float32(0.79) + np.float32(0.86)


def test_dense_block_golden(oracle, golden):
    g = _graph(oracle, golden)
    v = golden["dense_block_4_1"]
    y = oracle.dense_block(g, np.array(v["x"]), use_weight=False, use_bias=False)
    assert np.abs(y - np.array(v["y"])).max() <= 1e-12


def test_gsr_forward_block_golden(oracle, golden):
    g = _graph(oracle, golden)
    v = golden["gsr_forward_block_4_1"]
    y = oracle.block_fwd(g, np.array(v["values"]), np.array(v["indices"]), None, width=4, use_weight=False)
    assert np.array_equal(y, np.array(v["y"]))


def test_gsr_forward_block_identity_graph(oracle):
    """identity-only graph, flags off → scatter(s)."""
    n, w, k = 6, 5, 2
    g = oracle.Graph(np.arange(n + 1), np.arange(n))
    x = np.random.default_rng(3).normal(size=(n, w))
    vals, idx = oracle.gs_topk(x, k)
    y = oracle.block_fwd(g, vals, idx, None, width=w, use_weight=False)
    assert np.array_equal(y, oracle.scatter(vals, idx, w))


def test_mse_hand(oracle, golden):
    v = golden["mse_hand"]
    loss, gy = oracle.mse(np.array(v["yhat"]), np.array(v["y"]), np.array(v["mask"]))
    assert loss == v["loss"] and gy.tolist() == v["grad"]
    with pytest.raises(oracle.OracleError):
        oracle.mse(np.zeros(2), np.zeros(2), np.zeros(2))             # empty mask → error


def test_gs_topk_k_out_of_range(oracle):
    with pytest.raises(oracle.OracleError) as e:
        oracle.gs_topk(np.zeros((2, 3)), 4)
    assert e.value.code == 1


def test_oracle_tf32_operand_truncation(oracle):
    """TF32 transform mode reads operands as the B200 tensor core does: the low
    13 mantissa bits truncated (scratch/tf32_probe.cu measured 128/128)."""
    rp, ci = np.arange(2), np.arange(1)
    g = oracle.Graph(rp, ci, norm=0)
    W = np.ones((1, 1), np.float32)
    cases = [(1 + 2.0 ** -11, 1.0), (1 + 2.0 ** -12, 1.0), (-(1 + 2.0 ** -11), -1.0), (1 + 3 * 2.0 ** -12, 1.0),
             (1 + 2.0 ** -10 + 2.0 ** -11, 1 + 2.0 ** -10)]
    try:
        oracle.set_tf32(True)
        for x, want in cases:
            out = oracle.block_fwd(g, np.array([[x]], np.float32), np.zeros((1, 1), np.int32), W, width=1)
            assert out[0, 0] == np.float32(want), (x, out[0, 0], want)
    finally:
        oracle.set_tf32(False)
    out = oracle.block_fwd(g, np.array([[1 + 2.0 ** -11]], np.float32), np.zeros((1, 1), np.int32), W, width=1)
    assert out[0, 0] == np.float32(1 + 2.0 ** -11)
