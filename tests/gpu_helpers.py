"""Shared helpers for the -m gpu parity tests (oracle = the checker)."""
import numpy as np

from paper_2603_27156_b200 import synth


def make_graph(n, seed, hubs=True, self_loops=False, isolated=0):
    """Lattice + hubs (rows longer than a warp's 32-edge batch) + optional
    isolated nodes (empty rows)."""
    cfg = synth.SynthConfig(n=n, base_degree=2, hub_fraction=(0.02 if hubs else 0.0), hub_degree_range=(20, min(n - 1, 90)),
                            seed=seed, self_loops=self_loops)
    g = synth.generate_graph(cfg)
    if isolated:
        # drop all edges of the first `isolated` nodes (both directions)
        rows = np.repeat(np.arange(n), np.diff(g.row_ptr))
        keep = (rows >= isolated) & (g.col_idx >= isolated)
        g = synth.from_edge_list(n, rows[keep], g.col_idx[keep])
    return g


def block_max_rel(a, b, layout):
    """max over parameter blocks of max|a-b| / max|b| (scale-relative)."""
    worst = 0.0
    segs = [layout["enc_w"], layout["enc_b"], layout["head_w"], layout["head_b"]]
    segs += [(o, w * w + w) for _, o, w in layout["blocks"]]
    for o, n in segs:
        ref = np.abs(b[o:o + n]).max()
        if ref == 0:
            continue
        worst = max(worst, float(np.abs(a[o:o + n] - b[o:o + n]).max() / ref))
    return worst


def ties_matrix(rng, n, w):
    x = rng.normal(size=(n, w)).astype(np.float32)
    x[::3, ::2] = np.round(x[::3, ::2], 1)    # magnitude ties
    x[1::4] = -x[1::4]
    x[2::5, :w // 2] = 0.0                    # zero ties
    x[3::7, 1] = -0.0
    x[5::11, :] = 0.0                         # all-zero rows
    return x


def dyadic_case(n, D, C, k, seed, use_bias):
    """Graph with hubs over 1024 edges (norm none: unit edge scales), values on
    a 1/2 grid, signed-permutation transforms. Returns (graph, params, x, y, G).

    Why every dW partial sum is exact: dW_i = Σ_r S_i[r]ᵀ·Y_i[r] with
    Y_i = Âᵀ·G_i. The masked input gradient of block i is added into G_{i-1}
    and grows by up to a hub's in-degree per block, so only blocks 0 and C-1
    carry a (±1) permutation and blocks 1..C-2 have W = 0 (their dW is still
    computed: it does not depend on W). G is ±1/2, ±1 on 10% of rows. Then
    Σ_r |S||Y| stays below ~2^20 on a 1/4 product grid (< 2^24 ulps), and
    every product of TF32 operands is exact, so the tensor core's and the
    oracle's summation orders give the same fp32 result."""
    from paper_2603_27156_b200 import MODE_GSRC, model, synth
    cfg = synth.SynthConfig(n=n, base_degree=2, hub_fraction=4.0 / n, hub_degree_range=(1400, 1500), seed=seed)
    g = synth.generate_graph(cfg)
    lay = model.param_layout(MODE_GSRC, 1, D, C, 8)
    rng = np.random.default_rng(seed)
    p = (rng.integers(-2, 3, lay["P"]) * 0.5).astype(np.float32)   # encoder / head (unused by layer calls)
    w = lay["w"]
    for (_, i), o, _ in lay["blocks"]:
        W = np.zeros((w, w), np.float32)
        if i in (0, C - 1):
            W[rng.permutation(w), np.arange(w)] = rng.choice([-1.0, 1.0], w)
        p[o:o + w * w] = W.ravel()
        p[o + w * w:o + w * w + w] = (rng.integers(-1, 2, w) * 0.5) if use_bias else 0.0
    grid = lambda shape, lo, hi: (rng.integers(lo, hi + 1, shape) * 0.5).astype(np.float32)
    x = grid((n, D), -3, 3)
    y = grid((n, D), -3, 3)
    G = grid((n, D), -2, 2) * (rng.random((n, 1)) < 0.1)
    return g, p, x, y, G.astype(np.float32)
