#!/usr/bin/env python
"""Timing of row f4 (icp_register) on the low-res Eq.3 cloud of one synthetic pair:
the 676x380 ground-truth disparity reprojected on the GPU (P.reproject), registered
against itself moved by a small rigid motion (0.3 deg about z, (5, 2, -3) cm).
CUDA events on the launching stream after warm-up; one JSON line.

  python tools/time_icp.py [--reps 5] [--stride 4] [--max-iter 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_09733_b200 as P  # noqa: E402
import synthgen  # noqa: E402


def lowres_cloud_pair(dev, seed=2):
    """(src, tgt) float32 [N,3] on dev: Eq.3 cloud of the low-res ground truth and its moved copy."""
    _, _, d_lo = synthgen.stereo_pair_rgb(seed)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"] / 4, I["f_dv"] / 4, (I["u0"] + 0.5) / 4 - 0.5, (I["v0"] + 0.5) / 4 - 0.5, I["B"])
    xyz, _ = P.reproject(torch.from_numpy(d_lo.astype(np.float32)).to(dev), Q, 1.0)
    src = xyz.reshape(-1, 3)
    th = np.deg2rad(0.3)
    Rm = torch.tensor([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]], dtype=torch.float64,
                      device=dev)
    tgt = (src.double() @ Rm.T + torch.tensor([0.05, 0.02, -0.03], dtype=torch.float64, device=dev)).float()
    return src.contiguous(), tgt.contiguous()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--stride", type=int, default=4)
    ap.add_argument("--max-iter", type=int, default=20)
    ap.add_argument("--max-dist", type=float, default=0.25)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    S, T = lowres_cloud_pair(dev)

    def run():
        return P.icp_register(S, T, max_iter=a.max_iter, max_dist=a.max_dist, eps=1e-7, stride=a.stride)

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        o = run()
    e1.record(st)
    torch.cuda.synchronize()
    o = o.cpu().numpy()
    print(json.dumps({"ms_per_registration": e0.elapsed_time(e1) / a.reps,
                      "points": int(torch.sum(~torch.isnan(S[:, 0])).item()), "stride": a.stride,
                      "max_dist_m": a.max_dist, "iterations": int(o[13]), "pairs": int(o[15]), "rms_m": float(o[12]),
                      "converged": int(o[14])}))


if __name__ == "__main__":
    main()
