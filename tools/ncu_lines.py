"""Aggregate an ncu source page (cuda,sass) by CUDA source line: stall samples and executed warp instructions.
Usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-index> [top]"""
import csv
import io
import subprocess
import sys

rep, kid = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip", kid, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname, hdr = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] in ("", "Function Name"):
        continue
    try:
        samp, ins = int(r[4]), int(r[7])
    except (ValueError, IndexError):
        continue
    res.append((samp, ins, fname, r[0], r[1][:100]))
tot = sum(x[0] for x in res) or 1
toti = sum(x[1] for x in res) or 1
print("total samples", tot, "warp instr", toti)
for x in sorted(res, reverse=True)[:top]:
    print(f"{x[0]:7d} {100 * x[0] / tot:5.1f}% ins {100 * x[1] / toti:5.1f}% {x[2]}:{x[3]} {x[4]}")
