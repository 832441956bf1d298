"""Flat parameter layout and seeded initialisation (host side).

Layout = GSRP block order: encoder W (d_in×D) and b (D); for each
layer l, for each block i: W (w×w, row-major, h = Z·W) and b (w); head w (D)
and b (1). Identical on the device (csrc/capi.cu off_block) and in the oracle
(oracle/gsr_oracle.hpp NetCfg), so one host vector initialises both sides.
"""
from __future__ import annotations

import numpy as np

from ._capi import MODE_ALG12


def param_layout(mode, layers, hidden, groups, d_in):
    C = 2 if mode == MODE_ALG12 else groups
    w = hidden // C
    nb = C
    lay = {"enc_w": (0, d_in * hidden), "enc_b": (d_in * hidden, hidden)}
    off = d_in * hidden + hidden
    blocks = []
    for l in range(layers):
        for i in range(nb):
            blocks.append(((l, i), off, w))
            off += w * w + w
    lay["blocks"] = blocks
    lay["head_w"] = (off, hidden)
    lay["head_b"] = (off + hidden, 1)
    lay["P"] = off + hidden + 1
    lay["w"] = w
    return lay


def init_params(mode, layers, hidden, groups, d_in, seed=0, block_scale=None, dtype=np.float32):
    """Glorot encoder / head; block weights uniform ±sqrt(6/(2w))
    divided by sqrt(L·C) by default (depth-scaled so an 80-layer, 4-group
    reversible stack neither explodes nor vanishes at init)."""
    lay = param_layout(mode, layers, hidden, groups, d_in)
    rng = np.random.Generator(np.random.PCG64(seed))
    P = lay["P"]
    p = np.zeros(P, np.float64)
    w = lay["w"]
    s_enc = np.sqrt(6.0 / (d_in + hidden))
    o, n = lay["enc_w"]
    p[o:o + n] = rng.uniform(-s_enc, s_enc, n)
    nb = len(lay["blocks"])
    bs = block_scale if block_scale is not None else np.sqrt(6.0 / (2 * w)) / np.sqrt(max(nb, 1))
    for _, o, w_ in lay["blocks"]:
        p[o:o + w_ * w_] = rng.uniform(-bs, bs, w_ * w_)
    o, n = lay["head_w"]
    s_h = np.sqrt(6.0 / (hidden + 1))
    p[o:o + n] = rng.uniform(-s_h, s_h, n)
    return p.astype(dtype)
