#!/usr/bin/env python
"""Table-3 analogue on one B200: the
GSR-C network against the rev-baseline (RevGNN-style dense grouped reversible
blocks) at the same config, both on the tcgen05 TF32 fast
path, both O(N·D) activation memory. Per model: the Eq. 9 breakdown of a
training step (forward, backward, copy, optimizer, total; gsrc_timing, CUDA
events, median of K graph-replayed steps after W warm-up steps), steps/s and
peak HBM (arena peak_active and the device cudaMemGetInfo delta).

    python tools/table3.py [--config c3] [--steps 5] [--warmup 3] [--out profiles/r2_table3.json]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(mode_name, cfg_name, steps, warmup, g, nd):
    import torch
    import bench
    from paper_2603_27156_b200 import GEMM_TF32, MODE_GSRC, MODE_REV, Context, model
    mode = {"gsrc": MODE_GSRC, "rev": MODE_REV}[mode_name]
    _, L, D, C, k = bench.CONFIGS[cfg_name]
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    ctx = Context(0)
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(mode, L, D, C, k, 8, gemm=GEMM_TF32)
    ctx.set_params(model.init_params(mode, L, D, C, 8, seed=1))
    ctx.data_upload(nd.features, nd.labels, nd.train_mask)
    ctx.set_graph_capture(True)
    lr = bench.LR_BY_CONFIG.get(cfg_name, bench.LR)
    losses = [ctx.train_step(lr=lr) for _ in range(warmup)]
    ctx.high_water_reset()
    rows = []
    for _ in range(steps):
        losses.append(ctx.train_step(lr=lr))
        t = ctx.last_timing()
        rows.append({k_: t[f"t_{k_}"] * 1e3 for k_ in ("forward", "backward", "copy", "optimizer", "total")})
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    m = ctx.mem_stats()
    med = {k_: statistics.median(r[k_] for r in rows) for k_ in rows[0]}
    res = {"model": {"gsrc": "GSR-C (grouped sparse reversible, GS top-k)", "rev": "rev-baseline (dense grouped reversible, ReLU)"}[mode_name],
           "ms": med, "steps_per_s": 1000.0 / med["total"], "peak_hbm": {"arena_peak_active": m["peak_active_bytes"],
           "cudaMemGetInfo_delta": int(free0 - free1)}, "loss_first_last": [losses[0], losses[-1]], "params": int(ctx.P),
           "kernel_launches": int(ctx.kernel_launches())}
    ctx.close()
    return res


def main():
    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    g, nd = bench.build_inputs(a.config, 0)
    _, L, D, C, k = bench.CONFIGS[a.config]
    out = {"config": {"workload": bench.workload(a.config, "tf32", "gsrc"), "n": g.n, "e": g.e, "layers": L, "hidden": D, "groups": C, "k": k},
           "gsrc": run("gsrc", a.config, a.steps, a.warmup, g, nd), "rev": run("rev", a.config, a.steps, a.warmup, g, nd)}
    out["gsr_speedup_total"] = out["rev"]["ms"]["total"] / out["gsrc"]["ms"]["total"]
    out["gsr_speedup_forward"] = out["rev"]["ms"]["forward"] / out["gsrc"]["ms"]["forward"]
    out["gsr_speedup_backward"] = out["rev"]["ms"]["backward"] / out["gsrc"]["ms"]["backward"]
    line = json.dumps(out)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
