"""Summaries of ncu output for profiles/ (markdown).

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of one step
    python tools/ncu_summary.py full <report.ncu-rep> [label]      # --set full capture: per-launch metrics + stalls

The launch list comes from `ncu --metrics gpu__time_duration.sum` over one
un-graphed bench step (cold-cache, serialised: compare shares, not absolutes).
"""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("gsrk::", "").replace("fast::", "").replace("tile::", "").replace("(anonymous namespace)::", "")
    name = name.replace("unnamed>::", "").replace("void ", "")
    return name.strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[i + 1:]:
        if len(r) <= mv or not r[mv]:
            continue
        v = float(r[mv].replace(",", ""))
        if r[mu] == "us":
            v *= 1e3
        elif r[mu] == "ms":
            v *= 1e6
        k = short(r[kn])
        tot[k] += v
        cnt[k] += 1
    all_ns = sum(tot.values())
    print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v / 1e6:.2f} | {100 * v / all_ns:.1f}% |")
    print(f"\n{sum(cnt.values())} launches, {all_ns / 1e6:.1f} ms summed device time (serialised, cold-cache under ncu).")


METRICS = [
    ("gpu__time_duration.sum", "time (us)", lambda v: f"{v / 1e3:.1f}" if v > 1e3 else f"{v:.1f}"),
    ("dram__bytes_read.sum", "DRAM read", None),
    ("dram__bytes_write.sum", "DRAM write", None),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", None),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %", None),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", None),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", None),
    ("sm__inst_executed.avg.per_cycle_active", "IPC", None),
    ("launch__registers_per_thread", "regs", None),
    ("launch__grid_size", "grid", None),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %", None),
]


def full(path, label):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"### {label}\n")
    cols = [(hdr.index(m), name, fmt) for m, name, fmt in METRICS if m in hdr]
    print("| kernel | " + " | ".join(f"{name} ({units[i]})" if units[i] and name not in ('IPC', 'regs', 'grid') else name for i, name, _ in cols) + " | top stalls (cycles/issue) |")
    print("|---" * (len(cols) + 2) + "|")
    for r in rows[2:]:
        vals = []
        for i, name, fmt in cols:
            v = r[i]
            try:
                fv = float(v.replace(",", ""))
                v = f"{fv:.3g}" if fmt is None else v
            except ValueError:
                pass
            vals.append(v)
        st = []
        for j, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[j]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls = ", ".join(f"{n} {v:.1f}" for v, n in sorted(st, reverse=True)[:4])
        print(f"| `{short(r[hdr.index('Kernel Name')])}` | " + " | ".join(vals) + f" | {stalls} |")
    print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[2])
