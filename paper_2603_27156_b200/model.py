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


# ---- GSRP parameter checkpoints ---------------------------------
# magic "GSRP", u32 LE version, then u64 LE mode, L, D, C, d_in and the block
# count; per block u64 LE rows, cols, then w (rows × cols) and b (cols) as f64 LE.
# Blocks in GSRP order: encoder (d_in × D), every layer's C blocks (w × w), head (D × 1).
GSRP_VERSION = 1


def _blocks(mode, layers, hidden, groups, d_in):
    lay = param_layout(mode, layers, hidden, groups, d_in)
    out = [(lay["enc_w"][0], d_in, hidden)]
    out += [(o, w, w) for _, o, w in lay["blocks"]]
    out.append((lay["head_w"][0], hidden, 1))
    return out


def write_gsrp(path, p, mode, layers, hidden, groups, d_in):
    p = np.asarray(p, np.float64)
    blocks = _blocks(mode, layers, hidden, groups, d_in)
    with open(path, "wb") as f:
        f.write(b"GSRP")
        f.write(np.array([GSRP_VERSION], "<u4").tobytes())
        f.write(np.array([mode, layers, hidden, groups, d_in, len(blocks)], "<u8").tobytes())
        for o, rows, cols in blocks:
            f.write(np.array([rows, cols], "<u8").tobytes())
            f.write(p[o:o + rows * cols + cols].astype("<f8").tobytes())


def read_gsrp(path):
    """→ (params f32, dict(mode, layers, hidden, groups, d_in)); ValueError on a malformed file."""
    with open(path, "rb") as f:
        buf = f.read()
    if len(buf) < 56 or buf[:4] != b"GSRP":
        raise ValueError(f"{path}: bad GSRP magic")
    if int(np.frombuffer(buf, "<u4", 1, 4)[0]) != GSRP_VERSION:
        raise ValueError(f"{path}: unsupported GSRP version")
    mode, layers, hidden, groups, d_in, nb = (int(x) for x in np.frombuffer(buf, "<u8", 6, 8))
    blocks = _blocks(mode, layers, hidden, groups, d_in)
    if nb != len(blocks):
        raise ValueError(f"{path}: block count {nb} != {len(blocks)}")
    P = param_layout(mode, layers, hidden, groups, d_in)["P"]
    p = np.zeros(P, np.float64)
    off = 56
    for o, rows, cols in blocks:
        if off + 16 > len(buf):
            raise ValueError(f"{path}: truncated GSRP")
        r, c = (int(x) for x in np.frombuffer(buf, "<u8", 2, off))
        if (r, c) != (rows, cols):
            raise ValueError(f"{path}: block shape {(r, c)} != {(rows, cols)}")
        off += 16
        cnt = rows * cols + cols
        if off + 8 * cnt > len(buf):
            raise ValueError(f"{path}: truncated GSRP")
        p[o:o + cnt] = np.frombuffer(buf, "<f8", cnt, off)
        off += 8 * cnt
    if off != len(buf):
        raise ValueError(f"{path}: trailing bytes in GSRP")
    return p.astype(np.float32), dict(mode=mode, layers=layers, hidden=hidden, groups=groups, d_in=d_in)
