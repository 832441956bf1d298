"""SPEC invariants and acceptance criteria checked on the CPU oracle.

Acceptance criteria: 2 reversibility, 3 FD gradients,
4 Alg. 1/2 transcription, 5 sparse/dense bridge, 6 work scaling,
12 determinism. CPU-only.
"""
import numpy as np
import pytest

from paper_2603_27156_b200 import synth


def rand_graph(oracle, n, m, seed, norm=0, self_loops=True):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, size=m)
    v = rng.integers(0, n, size=m)
    if self_loops:
        u = np.concatenate([u, np.arange(n)])
        v = np.concatenate([v, np.arange(n)])
    g = synth.from_edge_list(n, u, v)
    return oracle.Graph(g.row_ptr, g.col_idx, norm=norm)


@pytest.mark.parametrize("norm", [0, 1, 2])
@pytest.mark.parametrize("transpose", [False, True])
def test_bridge_sparse_equals_dense(oracle, norm, transpose):
    """Acceptance 5: spmm_sparse == spmm∘scatter exactly."""
    for seed in range(5):
        rng = np.random.default_rng(seed)
        n, w = int(rng.integers(3, 60)), int(rng.integers(1, 20))
        k = int(rng.integers(1, w + 1))
        g = rand_graph(oracle, n, 4 * n, seed, norm=norm)
        for dt in (np.float64, np.float32):
            x = rng.normal(size=(n, w)).astype(dt)
            vals, idx = oracle.gs_topk(x, k)
            a = oracle.spmm_sparse(g, vals, idx, w, transpose=transpose)
            b = oracle.spmm(g, oracle.scatter(vals, idx, w), transpose=transpose)
            assert np.array_equal(a, b)


def test_spmm_against_densified_adjacency(oracle):
    """random graph vs dense multiply, all norms, both directions."""
    rng = np.random.default_rng(7)
    n, w = 30, 6
    for norm in (0, 1, 2):
        g = rand_graph(oracle, n, 90, 7, norm=norm, self_loops=False)
        rp, ci = g.csr()
        A = np.zeros((n, n))
        for r in range(n):
            A[r, ci[rp[r]:rp[r + 1]]] = 1
        deg = A.sum(1)
        if norm == 1:
            A = A / np.where(deg > 0, deg, 1)[:, None]
        elif norm == 2:
            s = np.where(deg > 0, 1 / np.sqrt(np.maximum(deg, 1)), 0)
            A = s[:, None] * A * s[None, :]
        x = rng.normal(size=(n, w))
        assert np.abs(oracle.spmm(g, x) - A @ x).max() <= 1e-12
        assert np.abs(oracle.spmm(g, x, transpose=True) - A.T @ x).max() <= 1e-12


def test_transpose_symmetric_graph(oracle):
    g = synth.generate_graph(synth.SynthConfig(n=200, hub_fraction=0.01, hub_degree_range=(5, 20), seed=3))
    og = oracle.Graph(g.row_ptr, g.col_idx, norm=0)
    x = np.random.default_rng(0).normal(size=(200, 8))
    assert np.array_equal(oracle.spmm(og, x), oracle.spmm(og, x, transpose=True))


def test_work_scaling(oracle):
    """Acceptance 6: k vs 4k exactly 4×; 4 vs 64 exactly 16×."""
    g = rand_graph(oracle, 300, 1200, 1)
    x = np.random.default_rng(1).normal(size=(300, 64))
    counts = {}
    for k in (4, 16, 64):
        vals, idx = oracle.gs_topk(x, k)
        oracle.work_reset()
        oracle.spmm_sparse(g, vals, idx, 64)
        counts[k] = oracle.work_muladds()
    assert counts[16] == 4 * counts[4] and counts[64] == 16 * counts[4]
    assert counts[4] == g.e * 4


def _net(oracle, g, mode, L, D, C, k, d_in=3, seed=0, dt=np.float64, scale=None, **kw):
    net = oracle.Net(g, mode, L, D, C, k, d_in, dtype=dt, **kw)
    rng = np.random.default_rng(seed)
    w = D // (2 if mode == oracle.MODE_ALG12 else C)
    s = scale if scale is not None else np.sqrt(6.0 / (2 * w))
    net.set_params(rng.uniform(-s, s, size=net.P).astype(dt))
    return net


@pytest.mark.parametrize("mode,C", [(2, 2), (2, 4), (1, 2), (1, 4)])
def test_reversibility(oracle, mode, C):
    """Acceptance 2: per-layer < 1e-10; 100 stacked layers < 1e-6 (f64).
    Applies to the rev baseline (mode 2) and to GSR-C (mode 1), whose blocks are
    GS-sparse; GS masks recomputed on the reconstructed inputs."""
    n, D = 200, 32
    g = rand_graph(oracle, n, 4 * n, 11, norm=1)
    k = (D // C) // 4
    net = _net(oracle, g, mode, 100, D, C, max(k, 1), scale=0.3)
    x = np.random.default_rng(5).normal(size=(n, D))
    y = net.layer_forward(0, x)
    assert np.abs(net.layer_inverse(0, y) - x).max() < 1e-10
    z = x
    for l in range(100):
        z = net.layer_forward(l, z)
    for l in reversed(range(100)):
        z = net.layer_inverse(l, z)
    assert np.abs(z - x).max() < 1e-6


def test_f_zero_identity(oracle):
    """rev_forward_layer with f≡0 → identity; gsr layer f≡0,
    k=D/2 → identity."""
    n, D = 20, 8
    g = rand_graph(oracle, n, 60, 2)
    x = np.random.default_rng(0).normal(size=(n, D))
    for mode, C in ((2, 2), (1, 4), (0, 2)):
        net = oracle.Net(g, mode, 1, D, C, D // 2 if mode == 0 else 1, 3, dtype=np.float64)
        net.set_params(np.zeros(net.P))
        y = net.layer_forward(0, x)
        assert np.array_equal(y, x)


def _fd_check(oracle, net, X0, y, mask, rel=1e-5, h=1e-6, n_params=None, seed=0):
    loss, grads, _, _ = net.loss_grads(X0, y, mask)
    p0 = net.params()
    rng = np.random.default_rng(seed)
    idxs = np.arange(net.P) if n_params is None else rng.choice(net.P, size=n_params, replace=False)
    for i in idxs:
        p = p0.copy(); p[i] += h; net.set_params(p)
        lp = net.loss_grads(X0, y, mask)[0]
        p = p0.copy(); p[i] -= h; net.set_params(p)
        lm = net.loss_grads(X0, y, mask)[0]
        fd = (lp - lm) / (2 * h)
        assert abs(fd - grads[i]) <= rel * max(abs(fd), abs(grads[i])) + 1e-9, (i, fd, grads[i])
    net.set_params(p0)


def test_fd_gradients_rev_baseline(oracle):
    """Acceptance 3: L=2, C=2, D=4, n=6, h=1e-6, rel 1e-5, all params."""
    n = 6
    g = rand_graph(oracle, n, 12, 4, norm=1)
    net = _net(oracle, g, oracle.MODE_REV, 2, 4, 2, 1, d_in=3, use_bias=True, scale=0.8)
    rng = np.random.default_rng(2)
    X0, y = rng.normal(size=(n, 3)), rng.normal(size=n)
    _fd_check(oracle, net, X0, y, np.ones(n, np.uint8))


@pytest.mark.parametrize("C,k", [(2, 2), (4, 1), (2, 1)])
def test_fd_gradients_gsrc(oracle, C, k):
    """GSR-C exact gradient (SURVEY.md §7 hard part 1) checked by central FD in
    f64 (masks are locally constant away from ties)."""
    n, D = 8, 8
    g = rand_graph(oracle, n, 20, 9, norm=1)
    net = _net(oracle, g, oracle.MODE_GSRC, 2, D, C, k, d_in=3, use_bias=True, scale=0.7, seed=C)
    rng = np.random.default_rng(6)
    X0, y = rng.normal(size=(n, 3)), rng.normal(size=n)
    _fd_check(oracle, net, X0, y, np.ones(n, np.uint8))


def test_alg12_transcription_equivalence(oracle):
    """Acceptance 4: modular layers == straight-line Alg. 1/2,
    bit-identical, 100 seeded fuzz cases (n≤64, D≤16, k∈1..D/2, L≤4)."""
    rng = np.random.default_rng(123)
    for case in range(100):
        n = int(rng.integers(2, 65))
        D = int(rng.choice([2, 4, 6, 8, 10, 12, 14, 16]))
        k = int(rng.integers(1, D // 2 + 1))
        L = int(rng.integers(1, 5))
        norm = int(rng.integers(0, 3))
        isrc = int(rng.integers(0, 2))
        g = rand_graph(oracle, n, 3 * n, case, norm=norm)
        dt = np.float64 if case % 2 else np.float32
        kw = dict(use_bias=bool(case % 3 == 0), index_source=isrc)
        a = _net(oracle, g, oracle.MODE_ALG12, L, D, 2, k, seed=case, dt=dt, **kw)
        b = _net(oracle, g, oracle.MODE_ALG12, L, D, 2, k, seed=case, dt=dt, **kw)
        x = rng.normal(size=(n, D)).astype(dt)
        xa, xb = x.copy(), x.copy()
        for l in range(L):
            xa = a.layer_forward(l, xa)
            xb = b.transcribe_forward(l, xb)
            assert np.array_equal(xa, xb), (case, l)
        gm = rng.normal(size=(n, D)).astype(dt)
        ga, gb = gm.copy(), gm.copy()
        for l in reversed(range(L)):
            _, ga = a.layer_backward(l, xa, ga)
            gb = b.transcribe_backward(l, gb)
            assert np.array_equal(ga, gb), (case, l)


def test_alg12_cache_discipline(oracle):
    g = rand_graph(oracle, 10, 30, 0)
    net = _net(oracle, g, oracle.MODE_ALG12, 1, 8, 2, 2)
    x = np.random.default_rng(0).normal(size=(10, 8))
    with pytest.raises(oracle.OracleError) as e:               # backward without forward
        net.layer_backward(0, x, x)
    assert e.value.code == 4
    net.layer_forward(0, x)
    with pytest.raises(oracle.OracleError):                    # double fill
        net.layer_forward(0, x)
    net.layer_backward(0, x, x)                                # consumes
    with pytest.raises(oracle.OracleError):
        net.layer_backward(0, x, x)


def test_alg12_zero_upstream(oracle):
    g = rand_graph(oracle, 12, 40, 1)
    # SPEC.md:401 holds with the default bias-off blocks (a bias makes
    # GSRBlock(GS(0)) = b, so Alg. 2 then propagates -b).
    net = _net(oracle, g, oracle.MODE_ALG12, 1, 8, 2, 2)
    x = np.random.default_rng(0).normal(size=(12, 8))
    net.layer_forward(0, x)
    net.zero_grads()
    _, gout = net.layer_backward(0, x, np.zeros((12, 8)))
    assert not gout.any() and not net.grads().any()


def test_determinism_across_threads(oracle):
    """Acceptance 12: bit-identical across thread counts."""
    cfg = synth.SynthConfig(n=3000, hub_fraction=0.003, hub_degree_range=(20, 200), seed=4)
    gg, nd = synth.generate_synthetic(cfg)
    g = oracle.Graph(gg.row_ptr, gg.col_idx, norm=1)
    outs = []
    for th in (1, 3, 8):
        oracle.set_threads(th)
        for mode in (0, 1):
            net = _net(oracle, g, mode, 2, 32, 4 if mode else 2, 4, d_in=8, dt=np.float32)
            outs.append(net.loss_grads(nd.features, nd.labels, nd.train_mask))
    oracle.set_threads(1)
    for a, b in zip(outs[:2], outs[2:4]):
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    for a, b in zip(outs[:2], outs[4:6]):
        assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_adam_scalar_quadratic(oracle):
    """Adam on a scalar quadratic converges to the minimum."""
    p = np.array([1.0])
    m, v = np.zeros(1), np.zeros(1)
    for t in range(1, 501):
        g = 2 * (p - 0.25)
        oracle.adam(p, g, m, v, t, lr=0.05)
    assert abs(p[0] - 0.25) < 1e-3


def test_gsr_descent(oracle):
    """training loss after 20 epochs below epoch-0 loss (k ≥ 4)."""
    cfg = synth.SynthConfig(n=2000, hub_fraction=0.005, hub_degree_range=(10, 100), seed=1)
    gg, nd = synth.generate_synthetic(cfg)
    g = oracle.Graph(gg.row_ptr, gg.col_idx, norm=1)
    for mode, C in ((0, 2), (1, 4)):
        net = _net(oracle, g, mode, 4, 32, C, 4, d_in=8, dt=np.float32, scale=0.2)
        p = net.params()
        m, v = np.zeros_like(p), np.zeros_like(p)
        losses = []
        for t in range(1, 21):
            loss, grads, _, _ = net.loss_grads(nd.features, nd.labels, nd.train_mask)
            losses.append(loss)
            oracle.adam(p, grads, m, v, t, lr=1e-2)
            net.set_params(p)
        assert losses[-1] < losses[0], (mode, losses)


def test_residual_grid_makes_f32_inverse_exact(oracle):
    """DESIGN.md §3 (exactly invertible residual stream): with the block outputs
    on the 2^-20 grid, 24 f32 GSR-C layers forward then inverse return the input
    bit for bit, and the plain-add variant does not (it drifts)."""
    from paper_2603_27156_b200 import model, synth
    g = synth.generate_graph(synth.SynthConfig(n=3000, hub_fraction=0.01, hub_degree_range=(10, 80), seed=4))
    og = oracle.Graph(g.row_ptr, g.col_idx, norm=1)
    L, D, C, k = 24, 128, 4, 8
    p = model.init_params(1, L, D, C, 8, seed=2)
    rng = np.random.default_rng(0)
    x = (np.round(rng.normal(size=(g.n, D)) * 2 ** 20) / 2 ** 20).astype(np.float32)   # on the grid, like the encoder output
    res = {}
    for q in (20, 0):
        net = oracle.Net(og, 1, L, D, C, k, 8, dtype=np.float32, qshift=q)
        net.set_params(p)
        y = x
        for l in range(L):
            y = net.layer_forward(l, y)
        for l in reversed(range(L)):
            y = net.layer_inverse(l, y)
        res[q] = np.abs(y - x).max()
    assert res[20] == 0.0
    assert res[0] > 0.0
