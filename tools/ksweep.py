#!/usr/bin/env python
"""The paper's K sweep (Table 3: 100 layers, 384 hidden,
K ∈ {4, 8, 16, 32, 64}) on one B200 at the c3 graph (1M nodes): GSR-C with
C = 4 (w = 96) for each K (and Alg. 1/2, C = 2, where w = D/2 ≤ 128), and
the rev-baseline (C = 4) once. w > 64 runs on the generic tcgen05 tile kernel
(k_tile, TF32), so this measures that path's speed; the fast thread-per-row
kernels cover w ≤ 64, k ≤ 16 (the bench config). Per run: Eq. 9 breakdown
(forward / backward / total, ms, median of the timed steps) and peak HBM.

    python tools/ksweep.py [--layers 100] [--hidden 384] [--ks 4,8,16,32,64] [--out profiles/r2_ksweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(g, nd, mode, L, D, C, k, steps, warmup, lr):
    import torch
    from paper_2603_27156_b200 import GEMM_TF32, Context, model
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    ctx = Context(0)
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(mode, L, D, C, k, 8, gemm=GEMM_TF32)
    ctx.set_params(model.init_params(mode, L, D, C, 8, seed=1))
    ctx.data_upload(nd.features, nd.labels, nd.train_mask)
    ctx.set_graph_capture(True)
    losses = [ctx.train_step(lr=lr) for _ in range(warmup)]
    rows = []
    for _ in range(steps):
        losses.append(ctx.train_step(lr=lr))
        t = ctx.last_timing()
        rows.append({x: t[f"t_{x}"] * 1e3 for x in ("forward", "backward", "total")})
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    m = ctx.mem_stats()
    ctx.close()
    med = {x: statistics.median(r[x] for r in rows) for x in rows[0]}
    return {"ms": med, "steps_per_s": 1000.0 / med["total"], "arena_peak_active": m["peak_active_bytes"],
            "cudaMemGetInfo_delta": int(free0 - free1), "loss_first_last": [losses[0], losses[-1]]}


def main():
    import bench
    from paper_2603_27156_b200 import MODE_ALG12, MODE_GSRC, MODE_REV
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=100)
    ap.add_argument("--hidden", type=int, default=384)
    ap.add_argument("--ks", default="4,8,16,32,64")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    g, nd = bench.build_inputs("c3", 0)
    L, D = a.layers, a.hidden
    res = {"graph": {"n": g.n, "e": g.e}, "layers": L, "hidden": D, "precision": "TF32 transforms (tcgen05 kind::tf32)", "runs": []}
    base = one(g, nd, MODE_REV, L, D, 4, 4, a.steps, a.warmup, bench.LR)
    res["runs"].append({"model": "rev-baseline", "C": 4, **base})
    for k in [int(x) for x in a.ks.split(",")]:
        for name, mode, C in (("GSR-C", MODE_GSRC, 4), ("Alg. 1/2", MODE_ALG12, 2)):
            if k > D // C or D // C > 128:   # the generic tile kernel covers w ≤ 128 (Alg. 1/2 at D = 384 has w = 192)
                continue
            r = one(g, nd, mode, L, D, C, k, a.steps, a.warmup, bench.LR)
            r["speedup_vs_rev_total"] = base["ms"]["total"] / r["ms"]["total"]
            res["runs"].append({"model": name, "C": C, "k": k, **r})
            print(json.dumps(res["runs"][-1]), flush=True)
    line = json.dumps(res)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
