#!/usr/bin/env python
"""A/B timing of the fused JBU + reprojection launch (a6+a7) at the bench's C5
shape: 32 pairs, 676x380 labels -> 2704x1520, s=4, r=2, sigma_s=3.75, sigma_r=15.
CUDA events on the launching stream after warm-up; prints one JSON line.
Run twice with VSBP_LIB=<other build> to compare kernel variants on one box.

  python tools/time_jbu.py [--batch 32] [--reps 20] [--tag name]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tag", default=os.environ.get("VSBP_LIB", "in-tree"))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    pool = [synthgen.stereo_pair_rgb(100 + i) for i in range(4)]
    guide = torch.stack([torch.from_numpy(pool[i % 4][0]) for i in range(a.batch)]).to(dev)
    lo = torch.stack([torch.from_numpy(pool[i % 4][2]).to(torch.int32) for i in range(a.batch)]).to(dev)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    out = P.jbu_reproject(lo, guide, 4, 3.75, 15.0, 2, Q)
    st = torch.cuda.current_stream()

    def run():
        P.jbu_reproject(lo, guide, 4, 3.75, 15.0, 2, Q, disp_hi=out[0], xyz=out[1], n_valid=out[2])

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
    print(json.dumps({"tag": a.tag, "batch": a.batch, "us_per_launch": us, "us_per_pair": us / a.batch}))


if __name__ == "__main__":
    main()
