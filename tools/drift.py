#!/usr/bin/env python
"""Reconstruction drift and GS-mask flips of the inverse recomputation.

The backward reconstructs every layer's input from its output (Eq. 7,
x_i = y'_i − f_i(u)); each reconstruction rounds, and a rounded input can flip a
near-tie GS top-k mask, after which f_i(u) changes by a whole selected column.
For one training step this reports, per (layer, block), the fraction of
sampled rows whose mask recomputed in the backward differs from the forward's
(gsrc_diag_masks), and the error of the reconstructed encoder output
max|x̂_enc − x_enc| / max|x_enc| after the full backward sweep.

    python tools/drift.py --config c3 [--gemm tf32] [--stride 1] [--lr-sweep 1e-4,3e-5] [--steps 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {"c1": (8, 64, 2, 8), "c2": (28, 128, 4, 8), "c3": (80, 256, 4, 16), "c5": (200, 256, 8, 8)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--gemm", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--lr-sweep", default="")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--qshift", type=int, default=20, help="residual-stream grid 2^-qshift (0 = plain fp32 adds)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    from paper_2603_27156_b200 import GEMM_FP32, GEMM_TF32, MODE_GSRC, Context, model, synth
    L, D, C, k = CONFIGS[a.config]
    t0 = time.time()
    g, nd = synth.generate_synthetic(synth.config_graph(a.config, seed=0))
    d_in = nd.features.shape[1]
    ctx = Context(0)
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(MODE_GSRC, L, D, C, k, d_in, gemm=GEMM_TF32 if a.gemm == "tf32" else GEMM_FP32)
    p = model.init_params(MODE_GSRC, L, D, C, d_in, seed=1)
    ctx.set_params(p)
    ctx.data_upload(nd.features, nd.labels, nd.train_mask)
    ctx.set_residual_quant(a.qshift)
    ctx.diag_masks(True, a.stride)
    loss = ctx.forward_backward()
    flips, rows = ctx.mask_flips()
    xr = ctx.activation()  # the backward sweep leaves the reconstructed encoder output
    # the encoder output itself: a 0-layer model with the same encoder / head on the device
    enc = Context(0)
    enc.graph_upload(g.row_ptr, g.col_idx, norm=1)
    enc.model_init(MODE_GSRC, 0, D, C, k, d_in, gemm=GEMM_TF32 if a.gemm == "tf32" else GEMM_FP32)
    enc.set_residual_quant(a.qshift)
    lay = model.param_layout(MODE_GSRC, L, D, C, d_in)
    enc.set_params(np.concatenate([p[:d_in * D + D], p[lay["head_w"][0]:]]))
    enc.data_upload(nd.features, nd.labels, nd.train_mask)
    enc.forward()
    xenc = enc.activation()
    enc.close()
    err = np.abs(xr - xenc).max(1) / np.abs(xenc).max()
    rate = flips / rows
    res = {
        "config": a.config, "gemm": a.gemm, "qshift": a.qshift, "max_abs_activation": float(np.abs(xr).max()), "n": g.n, "e": g.e, "layers": L, "groups": C, "k": k, "row_stride": a.stride,
        "sampled_rows_per_block": int(rows), "loss": loss,
        "mask_flip_rate": {"mean": float(rate.mean()), "max": float(rate.max()), "total_flipped_rows": int(flips.sum()),
                           "per_layer_mean": [float(x) for x in rate.mean(1)],
                           "block0_mean": float(rate[:, 0].mean()), "blocks_ge1_mean": float(rate[:, 1:].mean())},
        "reconstruction": {"bit_exact": bool(np.array_equal(xr, xenc)), "max_rel": float(err.max()), "rows_over_1e-4": float((err > 1e-4).mean()),
                           "rows_over_1e-6": float((err > 1e-6).mean()), "median_rel": float(np.median(err))},
    }
    ctx.diag_masks(False)
    if a.lr_sweep:
        res["lr_sweep"] = {}
        for lr in [float(x) for x in a.lr_sweep.split(",")]:
            ctx.set_params(p)
            ctx.set_graph_capture(True)
            res["lr_sweep"][str(lr)] = [ctx.train_step(lr=lr) for _ in range(a.steps)]
    res["wall_s"] = time.time() - t0
    line = json.dumps(res)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
