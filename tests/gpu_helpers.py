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
