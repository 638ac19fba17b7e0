#!/usr/bin/env python
"""A/B timing of the JBU launch (a6) at the bench's C5 shape: 128 pairs, 676x380
labels -> 2704x1520, s=4, r=2, sigma_s=3.75, sigma_r=15, guide = frames of the
synthetic video, labels = a smooth field with steps.  CUDA events on the launching
stream after warm-up; prints one JSON line per mode (upsample only, and the
pipeline's jbu_compact = JBU + counts + scan + packed write).
Run with VSBP_LIB=<other build> to compare kernel variants on one box.

  python tools/time_jbu.py [--batch 128] [--reps 10] [--tag name]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_09733_b200 as P  # noqa: E402
import synthgen  # noqa: E402
from synthgen import video  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--tag", default=os.environ.get("VSBP_LIB", "in-tree"))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    B = a.batch
    guide = torch.empty((B, 1520, 2704, 3), dtype=torch.uint8, device=dev)
    video.frames_device(video.VideoScene(1902), 0, guide)
    _, _, d_lo = synthgen.stereo_pair_rgb(3)
    lo = torch.from_numpy(d_lo).to(dev).to(torch.int32).expand(B, -1, -1).contiguous()
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    hi = torch.empty((B, 1520, 2704), dtype=torch.float32, device=dev)
    comp = P.CloudCompactor(2704, 1520, B, device=dev)
    xyz = torch.empty((B * 1520 * 2704, 3), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    modes = {
        "upsample": lambda: P.jbu_upsample(lo, guide, 4, 3.75, 15.0, 2, out=hi),
        "jbu_compact": lambda: P.jbu_compact(lo, guide, 4, 3.75, 15.0, 2, Q, 1.0, comp, disp_hi=hi, xyz=xyz),
    }
    for name, run in modes.items():
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            run()
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.reps
        print(json.dumps({"tag": a.tag, "mode": name, "batch": B, "us_per_launch": us, "us_per_pair": us / B}),
              flush=True)


if __name__ == "__main__":
    main()
