#!/usr/bin/env python
"""Single-core seconds per pair of the CPU oracle for BASELINE configs C1-C4
("Single-core seconds per pair for C1-C4").  One pair per config,
one thread, inputs from synthgen (C1: the 64x48 shifted texture; C2-C4: a pair of
the synthetic video).  Prints one JSON line; bench.py's cpu_baseline is the
all-core C5 rate.

  python tools/oracle_times.py [--out profiles/r02_oracle_single_core.json]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synthgen  # noqa: E402
from synthgen.video import VideoScene  # noqa: E402


def frames(scene, k):
    try:
        import torch
        if torch.cuda.is_available():
            from synthgen import video
            out = torch.empty((2, scene.H, scene.W, 3), dtype=torch.uint8, device="cuda")
            video.frames_device(scene, k, out)
            return out.cpu().numpy()
    except ImportError:
        pass
    return np.stack([scene.frame(k), scene.frame(k + 1)])


def timed(fn):
    t0 = time.perf_counter()
    r = fn()
    return time.perf_counter() - t0, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    oracle.build()
    I = synthgen.INTRINSICS
    Q = oracle.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    res = {"kind": "oracle (plain scalar C, gcc -O2), one thread, one pair", "host": platform.processor() or
           platform.machine(), "cpu_count": os.cpu_count()}
    l, r = synthgen.shifted_pair(1, 64, 48, 5)
    res["C1_bp_s"], _ = timed(lambda: oracle.bp_disparity(l, r, 16, 1, 5))
    f = frames(VideoScene(1902, 2704, 1520, 4, 8, 48), 100)
    gl, gr = oracle.prep(f[0], 4), oracle.prep(f[1], 4)
    res["C2_bp_s"], disp = timed(lambda: oracle.bp_disparity(gl, gr, 64, 5, 5))
    t_jbu, hi = timed(lambda: oracle.jbu(disp, f[0], 4, 3.75, 15.0, 2))
    t_pts, _ = timed(lambda: oracle.compact_cloud(hi, Q, 1.0))
    res["C3_pair_s"] = res["C2_bp_s"] + t_jbu + t_pts
    res["C3_jbu_s"], res["C3_cloud_s"] = t_jbu, t_pts
    f = frames(VideoScene(1902, 2704, 1520, 2, 16, 96), 100)
    gl, gr = oracle.prep(f[0], 2), oracle.prep(f[1], 2)
    res["C4_bp_s"], disp = timed(lambda: oracle.bp_disparity(gl, gr, 128, 6, 8))
    t_jbu, hi = timed(lambda: oracle.jbu(disp, f[0], 2, 7.5, 15.0, 3))
    t_pts, _ = timed(lambda: oracle.compact_cloud(hi, Q, 1.0))
    res["C4_pair_s"] = res["C4_bp_s"] + t_jbu + t_pts
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
