"""Summary of bench JSON lines (and an optional ncu metrics CSV) for quick A/B runs."""
import collections
import csv
import json
import sys


def bench(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    print(f"{path}: {d['value']:.3f} steps/s, {d['ms_per_step']:.1f} ms/step, phases {d.get('phases_ms_last_step')}")
    for k, v in d.get("kernels", {}).items():
        print(f"    {k:22s} {v['ms']:.4f} ms  blocks {[round(x, 4) for x in v.get('ms_per_block', [])]}  frac {v['frac_hbm']:.3f}")


def ncu(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "")[:40]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a[3] += m.get("smsp__inst_executed.sum", 0)
    tot = sum(a[1] for a in agg.values())
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:42s} n={a[0]:5d} avg={a[1] / a[0] / 1000:8.1f}us share={100 * a[1] / tot:5.1f}% "
              f"MB/launch={a[2] / a[0] / 1e6:7.1f} GB/s={a[2] / max(a[1], 1):7.0f} Minst={a[3] / a[0] / 1e6:6.1f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        (ncu if p.endswith(".csv") else bench)(p)
