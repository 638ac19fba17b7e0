#!/usr/bin/env python
"""Summarise ncu outputs (read here, on the CPU box) into a markdown file for profiles/.

  python tools/ncu_summary.py --launches gpurun_out/launches_TAG.csv \
      --rep gpurun_out/prof_TAG.ncu-rep --out profiles/r01_TAG.md --title "..."
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess

KEY_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__grid_size",
    "launch__block_size",
    "sm__maximum_warps_per_active_cycle_pct",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
]


def launch_table(path):
    """Per-kernel launches, device time (gpu__time_duration.sum) and, when the CSV
    carries them, DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum)."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        metric = r[mi] if mi is not None else "gpu__time_duration.sum"
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        if metric == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += v * tscale.get(r[ui], 1e-3)
        elif metric.startswith("dram__bytes"):
            agg[name][2] += v * bscale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    has_b = any(v[2] > 0 for v in agg.values())
    if has_b:
        lines = ["| kernel | launches | total us | share | DRAM MB per launch | DRAM GB/s |", "|---|---|---|---|---|---|"]
    else:
        lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        row = f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / tot:.3f} |"
        if has_b:
            row += f" {v[2] / max(v[0], 1) / 1e6:.1f} | {v[2] / 1e3 / v[1] if v[1] > 0 else 0:.0f} |"
        lines.append(row)
    return "\n".join(lines), tot


def rep_metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return "(no data)"
    h, units = rows[0], rows[1]
    lines = []
    for rr in rows[2:]:
        name = rr[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        lines.append(f"**{name[:120]}**\n")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m in KEY_METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"| `{m}` | {rr[i]} | {units[i]} |")
        lines.append("")
    return "\n".join(lines)


def rep_traffic(path):
    """{short kernel name: dram__bytes_read.sum + dram__bytes_write.sum} in bytes"""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for rr in rows[2:]:
        name = rr[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += float(rr[i].replace(",", "")) * scale.get(units[i], 1.0)
        res[name] = tot
    return res


def rep_pipes(path):
    """{short kernel name: {pipe: % of peak sustained active}} for the ALU, FMA and XU
    pipes and the issue slots (what binds a kernel that is not HBM-bound)"""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h = rows[0]
    ms = {"alu": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "fma": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "xu": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active"}
    res = {}
    for rr in rows[2:]:
        name = rr[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        res[name] = {k: round(float(rr[h.index(m)].replace(",", "")), 1) for k, m in ms.items() if m in h}
    return res


def level0_traffic(path):
    """Mean DRAM bytes (read + write) per level-0 message-update launch -- the fused
    two-iteration launches (k_update_pair with u8 costs) and the one-iteration updates
    with u8 costs except MODE 3 (the WTA-only pass) -- from a launch-list CSV."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iu = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[1:]:
        k = r[ik].replace("void ", "")
        is_l0 = k.startswith("vsbp::k_update_pair<unsigned char,") or (
            k.startswith("vsbp::k_update_fast<unsigned char,") and not k.startswith("vsbp::k_update_fast<unsigned char, 3,"))
        if not is_l0 or r[im] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        key = (r[h.index("ID")] if "ID" in h else len(per))
        per[key] = per.get(key, 0.0) + float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    if not per:
        return None
    return {"bytes_per_launch": sum(per.values()) / len(per), "launches": len(per)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--traffic-json", help="write {kernel: dram bytes per launch} for bench.py's roofline.traffic")
    ap.add_argument("--batch", type=int, default=0, help="pairs per launch of the captured run")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--notes", default="")
    a = ap.parse_args()
    parts = [f"# {a.title}\n"]
    if a.notes:
        parts.append(a.notes + "\n")
    if a.launches:
        t, tot = launch_table(a.launches)
        parts.append("## Launch list (ncu `gpu__time_duration.sum`, cold-cache, serialised)\n")
        parts.append(f"Total device time of the captured launches: {tot:.1f} us\n")
        parts.append(t + "\n")
    traffic, pipes = {}, {}
    for rep in a.rep:
        parts.append("## `--set full` capture\n")
        parts.append(rep_metrics(rep) + "\n")
        traffic.update(rep_traffic(rep))
        pipes.update(rep_pipes(rep))
    if a.traffic_json:
        import json
        level0 = level0_traffic(a.launches) if a.launches else None
        with open(a.traffic_json, "w") as f:
            # bench.py reports the level-0 message updates' traffic (its roofline kernels):
            # the mean DRAM bytes per level-0 update launch over the launch list
            json.dump({"batch": a.batch, "source": a.out, "dram_bytes_per_launch": traffic,
                       "pipes_pct": pipes, "level0_update": level0}, f, indent=1)
    with open(a.out, "w") as f:
        f.write("\n".join(parts))
    print(open(a.out).read())


if __name__ == "__main__":
    main()
