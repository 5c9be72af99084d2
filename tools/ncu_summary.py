"""Summarise ncu outputs into profiles/: launch list shares + key metrics of a
--set full capture.  Usage: python tools/ncu_summary.py <launches.csv> <rep>... > profiles/X.md"""
import csv, subprocess, sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0][:90]
                agg[k][0] += 1
                agg[k][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"### Launch list `{path.split('/')[-1]}` (ncu gpu__time_duration.sum, cold/serialised)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1] / 1e6:.1f} | {100 * v[1] / tot:.1f}% |")
    print()


KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem", "Theoretical Occupancy", "Achieved Occupancy",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
       "dram__bytes_read.sum.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "derived__memory_l1_wavefronts_shared_excessive", "smsp__inst_executed.sum",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__average_warp_latency_issue_stalled_barrier",
       "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_wait",
       "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_not_selected",
       "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_dispatch_stall", "smsp__pcsamp_warps_issue_stalled_no_instructions",
       "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_warps_issue_stalled_lg_throttle"]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    name = None
    vals = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in KEYS and d["Metric Name"] not in vals:
            vals[d["Metric Name"]] = f'{d["Metric Value"]} {d.get("Metric Unit", "")}'.strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rawv = {}
    if len(rr) >= 3:
        h, units, v = rr[0], rr[1], rr[2]
        for k in RAW:
            if k in h:
                i = h.index(k)
                rawv[k] = f"{v[i]} {units[i]}".strip()
    print(f"### `{path.split('/')[-1]}`: {name}\n")
    print("| metric | value |\n|---|---|")
    for k in KEYS:
        if k in vals:
            print(f"| {k} | {vals[k]} |")
    for k in RAW:
        if k in rawv:
            print(f"| {k} | {rawv[k]} |")
    print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        if p.endswith(".csv"):
            launches(p)
        else:
            rep(p)
