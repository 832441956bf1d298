#!/usr/bin/env python
"""CPU oracle step time vs depth at full N (backs the reference arm's linear-in-L
extrapolation): L in {1, 2, 4, 8} plus one real full-depth
step, on all host threads. Writes one JSON line.

    python tools/cpu_linearity.py --config c3 [--full] [--out profiles/r2_cpu_linearity.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--full", action="store_true", help="also time one real full-depth step")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    from oracle import oracle as o
    _, L, D, C, k = bench.CONFIGS[a.config]
    g, nd = bench.build_inputs(a.config, 0)
    th = bench.host_threads()
    o.set_threads(th)
    depths = [1, 2, 4, 8] + ([L] if a.full else [])
    t = {d: bench._oracle_sample(a.config, g, nd, 1, d) for d in depths}
    x = np.array([1, 2, 4, 8], float)
    y = np.array([t[d] for d in (1, 2, 4, 8)])
    slope, icpt = np.polyfit(x, y, 1)
    fit_err = float(np.abs(np.polyval([slope, icpt], x) - y).max() / y.max())
    ext2 = t[2] + (L - 2) * (t[2] - t[1])     # the reference arm's extrapolation
    res = {"config": a.config, "n": g.n, "e": g.e, "threads": th, "cpu_model": bench.cpu_model(), "seconds_by_layers": t,
           "linear_fit": {"s_per_layer": slope, "intercept_s": icpt, "max_rel_residual": fit_err},
           "extrapolated_full_step_s_from_L1_L2": ext2, "extrapolated_full_step_s_from_fit": icpt + slope * L}
    if a.full:
        res["measured_full_step_s"] = t[L]
        res["extrapolation_error_rel"] = (ext2 - t[L]) / t[L]
    line = json.dumps(res)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
