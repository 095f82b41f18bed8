#!/usr/bin/env python
"""Summarise an ncu capture for profiles/: per kernel in the report, key SOL /
memory / occupancy / stall metrics, DRAM bytes, tensor-pipe activity (tcgen05
kernels), and the hottest source lines (needs -lineinfo builds).

usage: python scripts/ncu_summary.py REPORT.ncu-rep [LAUNCHES.csv] > profiles/<name>.md
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Block Limit Shared Mem", "Block Limit Registers", "Eligible Warps Per Scheduler",
        "No Eligible", "Executed Instructions", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Warp Cycles Per Issued Instruction", "SM Frequency", "Compute (SM) Throughput")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_sector_hit_rate.pct",
       # tcgen05 evidence (M4): tensor pipe busy share, UTC* instruction issue, TMEM loads
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tc.sum", "sm__inst_executed_pipe_tmem.sum",
       "sm__inst_executed_pipe_uniform.sum")


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def func_name(k):
    m = re.search(r"(k_\w+)", k)
    return m.group(1) if m else k.split("(")[0]


def main():
    rep = sys.argv[1]
    print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
    det = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "details", "--csv"]))))
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    by_id = defaultdict(list)
    if det:
        h = det[0]
        ii, ki, mi, ui, vi = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                              h.index("Metric Value"))
        for r in det[1:]:
            by_id[r[ii]].append(r)
    hr, units = (raw[0], raw[1]) if len(raw) > 2 else ([], [])
    done = set()
    for n, (kid, rows) in enumerate(by_id.items()):
        kname = rows[0][ki]
        fn = func_name(kname)
        print(f"## kernel: `{kname[:140]}` (ID {kid})\n")
        print("| metric | value |\n|---|---|")
        seen = set()
        for r in rows:
            if any(k == r[mi] or (k in r[mi] and k.startswith("Block Limit")) for k in KEEP) and r[mi] not in seen:
                seen.add(r[mi])
                print(f"| {r[mi]} | {r[vi]} {r[ui]} |")
        if len(raw) > 2 + n:
            v = raw[2 + n]
            print("\n| raw metric | value |\n|---|---|")
            stalls = []
            for i, name in enumerate(hr):
                if name in RAW:
                    print(f"| {name} | {v[i]} {units[i]} |")
                if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                    try:
                        stalls.append((float(v[i].replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
            tot = sum(s for s, _ in stalls) or 1
            print("\nwarp stall samples (share):",
                  ", ".join(f"{nm} {s / tot:.1%}" for s, nm in sorted(stalls, reverse=True)[:8]))
        if fn in done:
            print()
            continue
        done.add(fn)
        src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                                               "--kernel-name", f"regex:{fn}"]))))
        out, f = [], None
        for r in src:
            if r and r[0] == "File Path":
                f = r[1].split("/")[-1]
            elif len(r) > 8 and r[0].isdigit() and r[2] == "-":
                try:
                    out.append((int(r[7]), int(r[4]), f, int(r[0]), r[1].strip()[:80]))
                except ValueError:
                    pass
        if out:
            ti = sum(x[0] for x in out) or 1
            ts = sum(x[1] for x in out) or 1
            print("\nhottest source lines (by stall samples):\n\n| stall % | inst % | line | source |\n|---|---|---|---|")
            for x in sorted(out, key=lambda t: -t[1])[:15]:
                print(f"| {x[1] / ts:.1%} | {x[0] / ti:.1%} | {x[2]}:{x[3]} | `{x[4]}` |")
        print()
    if len(sys.argv) > 2:
        lines = list(csv.reader(open(sys.argv[2])))
        hdr = [i for i, r in enumerate(lines) if "Kernel Name" in r][0]
        h = lines[hdr]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        agg = defaultdict(list)
        for r in lines[hdr + 1:]:
            if len(r) > vi:
                agg[r[ki].split("(")[0][-40:]].append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        print(f"\nlaunch list `{sys.argv[2].split('/')[-1]}` (gpu__time_duration.sum, cold-cache, serialised):\n")
        print("| kernel | launches | mean µs | share of step |\n|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")


if __name__ == "__main__":
    main()
