#!/usr/bin/env python
"""Print the key ncu --set full sections (SOL, occupancy, warp stalls, instruction
mix) of every kernel in a .ncu-rep, for reading here on the CPU box.
  python tools/ncu_details.py gpurun_out/prof_TAG.ncu-rep [kernel-substring]"""
import csv
import io
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis", "Occupancy",
            "Warp State Statistics", "Launch Statistics", "Scheduler Statistics")
KEEP = ("Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Executed Instructions", "Grid Size", "Block Limit Registers", "Block Limit Shared Mem",
        "Dynamic Shared Memory Per Block", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput")


def main():
    rep = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value",
                                                "Metric Unit"))
    for r in rows[1:]:
        if filt in r[ki] and r[si] in SECTIONS and r[mi] in KEEP:
            print(f"{r[ki][:28]:28s} | {r[mi]:36s} = {r[vi]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, u = rr[0], rr[1]
    for row in rr[2:]:
        name = row[h.index("Kernel Name")]
        if filt not in name:
            continue
        stalls = []
        for i, m in enumerate(h):
            if m.startswith("smsp__average_warp_latency_issue_stalled_") or (
                    m.startswith("smsp__warp_issue_stalled_") and m.endswith("_per_warp_active.pct")):
                try:
                    stalls.append((float(row[i]), m))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print(name[:60], "top stalls:")
        for v, m in stalls[:8]:
            print(f"   {v:8.2f}  {m}")
        for i, m in enumerate(h):
            if m.startswith("sm__inst_executed_pipe_") and m.endswith("pct_of_peak_sustained_active"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v > 1:
                    print(f"   pipe {m[23:]:60s} {v:6.1f}")


if __name__ == "__main__":
    main()
