"""Refresh the measured head of profiles/r2_summary.md from an evidence pass (tools/gpu_round.sh)
and copy its artefacts into profiles/; the hand-written sections after the ncu tables are kept.

    python tools/profile_summary.py [gpurun_out]
"""
import gzip
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
SUMMARY = os.path.join(PROF, "r2_summary.md")
NAMES = {"fused_block_fwd": "FWD (`k_hub_rows` + `k_fws<64,0,16>`)", "block_bwd_recompute": "INV (`k_hub_rows` + `k_fws<64,1,16>`)",
         "block_bwd_input": "BIN (`k_hub_seg_dense` + `k_hub_fold` + `k_bin2<64,2>`)", "gs_groupsum": "group-sum GS (`k_gs_tma<64>`)"}


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def ncu_md(mode, path, label=None):
    cmd = [sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), mode, path] + ([label] if label else [])
    return subprocess.run(cmd, capture_output=True, text=True, check=True).stdout


def row_bytes(md, kernel):
    for line in md.splitlines():
        if f"`{kernel}`" in line:
            p = [x.strip() for x in line.strip().strip("|").split("|")]
            return (float(p[2]) + float(p[3])) * 1e6
    raise KeyError(kernel)


def main():
    shutil.copy(os.path.join(SRC, "bench_c3.json"), os.path.join(PROF, "r2_bench_c3.json"))
    shutil.copy(os.path.join(SRC, "bench_ref.json"), os.path.join(PROF, "r2_bench_reference.json"))
    with open(os.path.join(SRC, "launches.csv"), "rb") as f, gzip.open(os.path.join(PROF, "r2_launches_c3.csv.gz"), "wb") as g:
        g.write(f.read())
    b = last_json(os.path.join(PROF, "r2_bench_c3.json"))
    r = last_json(os.path.join(PROF, "r2_bench_reference.json"))
    fwd = ncu_md("full", os.path.join(SRC, "prof_fwd.ncu-rep"), "forward, layer 0 (group-sum GS, sparse hub pre-pass, FWD with GS epilogue)")
    bwd = ncu_md("full", os.path.join(SRC, "prof_bwd.ncu-rep"), "backward, blocks of layer 79 (dense hub pre-pass, sparse hub pre-pass, INV, BIN, dW reduction)")
    launches = ncu_md("launches", os.path.join(SRC, "launches.csv"))
    traffic = {"source": "ncu --set full capture of one c3 step, round 2 final (profiles/r2_summary.md: forward layer 0; backward blocks of layer 79); "
                         "DRAM read+write bytes per launch, each class including its hub-row pre-pass launches; FWD is a block with its GS epilogue, "
                         "INV the block without (block C-1)",
               "fused_block_fwd": row_bytes(fwd, "k_hub_rows<64>") + row_bytes(fwd, "k_fws<64, 0, 16>"),
               "block_bwd_recompute": row_bytes(bwd, "k_hub_rows<64>") + row_bytes(bwd, "k_fws<64, 1, 16>"),
               "block_bwd_input": row_bytes(bwd, "k_hub_seg_dense<64>") + row_bytes(bwd, "k_hub_fold<64>") + row_bytes(bwd, "k_bin2<64, 2, 0>"),
               "gs_groupsum": row_bytes(fwd, "k_gs_tma<64>")}
    json.dump(traffic, open(os.path.join(PROF, "r2_traffic.json"), "w"), indent=1)
    rows = [f"| {NAMES[k]} | {v['ms']:.3f} | {' / '.join(f'{x:.3f}' for x in v.get('ms_per_block', [])) or '—'} | {int(v['launches_per_step'])} | "
            f"{v['bytes'] / 1e6:.0f} MB | {v['achieved_gbs']:.0f} | {v['frac_hbm']:.2f} | {traffic[k] / 1e6:.0f} MB | {100 * v['share_of_step']:.1f}% |"
            for k, v in b["kernels"].items()]
    cpu = b["cpu_baseline"]
    ph = b["phases_ms_last_step"]
    head = f"""# Round 2 profiles — GSR-C training step, config c3, 1×B200

Config c3: 1M nodes, 3.99M edges, L = 80, D = 256, C = 4 (w = 64), k = 16, TF32 block transforms.
Peak used for every fraction: the measured 6457.1 GB/s of `MEASURED_PEAKS.json` (driver-written, burst copy).
Everything below is from one evidence pass on one box (`tools/gpu_round.sh`, final round-2 code; refreshed by
`tools/profile_summary.py`), except where a row says otherwise.

## Bench line (`r2_bench_c3.json`, `python bench.py`, defaults)

- **{b['value']:.3f} steps/s** ({b['ms_per_step']:.1f} ms/step); `e2e` {b['e2e']['value']:.3f} steps/s (node inputs copied from pinned host memory each step, loss read back).
- Eq. 9 phases of the last step: forward {ph['forward']:.1f} ms, backward {ph['backward']:.1f} ms, optimizer {ph['optimizer']:.3f} ms.
- Clocks {b['clocks']['sm_mhz']:.0f} MHz of {b['clocks']['sm_max_mhz']:.0f}, no throttle reason; {b['gpu_launches']} kernel launches per timed region.
- Peak HBM (arena) {b['peak_hbm_bytes']['arena_peak_active'] / 1e9:.2f} GB; the depth sweep (L = 20, 80, 200) is in the same line (`peak_hbm_depth_sweep`).
- CPU oracle on {cpu['cores']} host threads ({cpu['cpu_model']}): {cpu['sample']} → {cpu['value']:.4f} steps/s, so **{b['value'] / cpu['value']:.0f}×** on this box
  (the host CPUs differ between boxes: the same sample extrapolated to 137-178 s/step on other evidence boxes this round).
  The linearity of that extrapolation and one measured 80-layer CPU step (164 s) are in `r2_cpu_linearity.json`.
- Reference arm (`r2_bench_reference.json`, `bench.py --impl reference`, the same oracle): {r['value']:.4f} steps/s.
- Round 1 for comparison: 3.235 steps/s (driver `BENCH_r01.json`); the round-2 start (commit c713ef3) measured 3.35-3.40.

## Live per-class timings (CUDA events inside `bench.py`; algorithmic bytes per DESIGN.md §5; each class with its hub pre-pass)

| class | ms / launch | ms per block 0/1/2/3 | launches / step | algorithmic bytes | algorithmic GB/s | frac | measured DRAM / launch | share of step |
|---|---|---|---|---|---|---|---|---|
""" + "\n".join(rows) + """

FWD / INV blocks 0-2 run the GS epilogue (the next block's, or the lower layer's, records); block 3 does not.
BIN's block 0 adds its masked gradient into C − 1 = 3 planes.

## Launch list (one un-graphed step under `ncu --metrics gpu__time_duration.sum`; raw: `r2_launches_c3.csv.gz`)

Cold-cache and serialised: compare shares, not absolute values.

""" + launches + "\n\n## `--set full` captures (`ncu --set full --clock-control none --import-source on`)\n\n" + fwd + "\n" + bwd + "\n"
    old = open(SUMMARY).read()
    tail = old[old.index("`k_fws` FWD ("):]
    open(SUMMARY, "w").write(head + tail)
    print(f"{b['value']:.3f} steps/s, e2e {b['e2e']['value']:.3f}, BIN frac {b['roofline']['frac']:.3f}")


if __name__ == "__main__":
    main()
