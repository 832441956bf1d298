"""SPEC acceptance 11 ("quality parity"): matched-seed
synthetic training of GSR-C (k = w/4 per group, the 25% group sparsity of c3)
and of the rev-baseline (dense grouped reversible blocks) through the C++ CLI
(tools/gsrnet-cuda) on one B200; after 100 epochs the test-split Pearson,
Spearman and Kendall tau-b of the two runs must differ by ≤ 0.05 and both
Pearson ≥ 0.5.

    python tools/quality_parity.py [--out profiles/r2_quality_parity.json]
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_quality_parity.json"))
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--epochs", type=int, default=100)
    args = ap.parse_args()
    from paper_2603_27156_b200 import synth
    cfg = synth.SynthConfig(n=args.n, base_degree=2, hub_fraction=0.002, hub_degree_range=(300, 700), seed=0)
    g, nd = synth.generate_synthetic(cfg)
    L, D, C = 8, 128, 4
    k = (D // C) // 4
    cli = os.path.join(ROOT, "tools", "gsrnet-cuda")
    res = {"config": {"n": g.n, "e": g.e, "layers": L, "hidden": D, "groups": C, "k": k, "epochs": args.epochs, "lr": 1e-3, "seed": 7,
                      "precision": "tf32", "criterion": "SPEC.md:665: |metric(gsr, k=D/4) - metric(baseline)| <= 0.05 (Pearson, Spearman, Kendall), both Pearson >= 0.5"}}
    with tempfile.TemporaryDirectory() as td:
        gp, np_ = os.path.join(td, "g.gsrg"), os.path.join(td, "n.gsrn")
        synth.write_graph(gp, g)
        synth.write_node_data(np_, nd)
        for model in ("gsrc", "baseline"):
            rep = os.path.join(td, f"{model}.jsonl")
            r = subprocess.run([cli, "train", "--graph", gp, "--nodes", np_, "--model", model, "--layers", str(L), "--hidden", str(D),
                                "--groups", str(C), "--k", str(k), "--epochs", str(args.epochs), "--lr", "1e-3", "--seed", "7",
                                "--precision", "tf32", "--report", rep], capture_output=True, text=True, timeout=1200)
            if r.returncode != 0:
                raise SystemExit(f"{model}: exit {r.returncode}: {r.stderr[-500:]}")
            recs = [json.loads(x) for x in open(rep)]
            ep = [x for x in recs if x["record"] == "epoch"]
            met = next(x for x in recs if x["record"] == "metrics")
            res[model] = {"test": met["test"], "val": met["val"], "loss_first": ep[0]["train_loss"], "loss_last": ep[-1]["train_loss"],
                          "s_per_epoch": sum(x["t_total"] for x in ep[1:]) / max(1, len(ep) - 1)}
    d = {m: abs(res["gsrc"]["test"][m] - res["baseline"]["test"][m]) for m in ("pearson", "spearman", "kendall")}
    res["abs_diff_test"] = d
    res["pass"] = bool(all(v <= 0.05 for v in d.values()) and res["gsrc"]["test"]["pearson"] >= 0.5 and res["baseline"]["test"]["pearson"] >= 0.5)
    json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
