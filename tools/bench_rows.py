#!/usr/bin/env python
"""Per-row device timings of the widened rows (f1-f4) on one B200, CUDA events on
the launching stream after warm-up.  bench.py remains the contract benchmark (the
a0-a8 path); this script measures the "next" rows at their natural units.

  python tools/bench_rows.py [--out profiles/r01_rows.json]
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


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch", type=int, default=16)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    B = a.batch
    res = {"gpu": torch.cuda.get_device_name(0), "batch": B}
    left, right, _ = synthgen.stereo_pair_rgb(0)
    L = torch.from_numpy(np.stack([left] * B)).to(dev)
    R = torch.from_numpy(np.stack([right] * B)).to(dev)

    # f1: undistortion + grey/box downsample of B raw 2.7K frames (left: with the rectified guide)
    cam = (1400.0, 1400.0, 1351.5, 759.5, -0.25, 0.08, -0.01)
    rect = torch.empty_like(L)
    gray = torch.empty((B, 380, 676), dtype=torch.uint8, device=dev)
    ms = timed(lambda: P.rectify_prep(L, cam, 4, gray=gray, rect=rect))
    res["f1_rectify_prep_with_rgb_out"] = {"ms_per_frame": ms / B, "GB_per_s": B * 2 * 2704 * 1520 * 3 / (ms / 1e3) / 1e9}
    ms = timed(lambda: P.rectify_prep(L, cam, 4, gray=gray))
    res["f1_rectify_prep_grey_only"] = {"ms_per_frame": ms / B}

    # grey pairs for BP / features
    gl = P.prep_downsample(L, 4)
    gr = P.prep_downsample(R, 4)

    # full BP (a1-a5) for reference, then f2 constant-space BP
    bp = P.StereoBP(676, 380, 64, 5, 5, batch=B, device=dev)
    out = torch.empty((B, 380, 676), dtype=torch.int32, device=dev)
    res["a1_a5_full_bp"] = {"ms_per_pair": timed(lambda: bp.disparity(gl, gr, out=out)) / B}
    # C4 (BASELINE configs[3]): 1352x760 (2.7K/2), L=128, 6 levels x 8 iterations,
    # guided upsampling s=2 (r=3, sigma_s=7.5 low-res px) to 2.7K + reprojection
    B4 = max(1, B // 4)
    gl2 = P.prep_downsample(L[:B4], 2)
    gr2 = P.prep_downsample(R[:B4], 2)
    bp4 = P.StereoBP(1352, 760, 128, 6, 8, batch=B4, device=dev)
    out4 = torch.empty((B4, 760, 1352), dtype=torch.int32, device=dev)
    ms_bp4 = timed(lambda: bp4.disparity(gl2, gr2, out=out4), reps=5) / B4
    I = synthgen.INTRINSICS
    Q4 = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    o4 = P.jbu_reproject(out4, L[:B4], 2, 7.5, 15.0, 3, Q4)
    ms_jbu4 = timed(lambda: P.jbu_reproject(out4, L[:B4], 2, 7.5, 15.0, 3, Q4, disp_hi=o4[0], xyz=o4[1],
                                            n_valid=o4[2]), reps=5) / B4
    res["c4_bp_1352x760_L128_6x8"] = {"ms_per_pair": ms_bp4, "pairs_per_s": 1e3 / ms_bp4,
                                       "workspace_MB_per_pair": bp4.workspace.numel() / B4 / 1e6}
    res["c4_jbu_s2_r3_reproject"] = {"ms_per_pair": ms_jbu4}
    # f2 at C4, where constant-space BP should pay (12.6 GB/pair of full-BP message
    # traffic at u16; k_l = min(128, k0 2^l) <= 64 candidates -> k0 <= 2)
    for k0 in (1, 2):
        cs4 = P.ConstantSpaceBP(1352, 760, 128, 6, 8, k0, batch=B4, device=dev)
        res[f"f2_csbp_c4_k0_{k0}"] = {"ms_per_pair": timed(lambda: cs4.disparity(gl2, gr2, out=out4), reps=5) / B4,
                                      "workspace_MB_per_pair": cs4.workspace.numel() / B4 / 1e6}
        del cs4
    del bp4, out4, o4
    for k0 in (1, 2, 4):
        cs = P.ConstantSpaceBP(676, 380, 64, 5, 5, k0, batch=B, device=dev)
        res[f"f2_csbp_k0_{k0}"] = {"ms_per_pair": timed(lambda: cs.disparity(gl, gr, out=out)) / B,
                                  "workspace_MB_per_pair": cs.workspace.numel() / B / 1e6}
    res["a1_a5_full_bp"]["workspace_MB_per_pair"] = bp.workspace.numel() / B / 1e6

    # f3: Harris corners on the 30x30 grid + ZSSD matching into the right frame
    for sr in (16, 48):
        def feat():
            _, xy, _, _ = P.harris_corners(gl, 30, 30, 4, 10 ** 9)
            P.zssd_match(gl, gr, xy, 5, sr)
        res[f"f3_harris_zssd_sr{sr}"] = {"ms_per_pair": timed(feat) / B}
    res["f3_harris_only"] = {"ms_per_pair": timed(lambda: P.harris_corners(gl, 30, 30, 4, 10 ** 9)) / B}

    # f4: ICP of a low-res Eq.3 cloud against itself moved by a small rigid motion
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"] / 4, I["f_dv"] / 4, (I["u0"] + 0.5) / 4 - 0.5, (I["v0"] + 0.5) / 4 - 0.5, I["B"])
    xyz, _ = P.reproject(out[0].float().contiguous(), Q, 1.0)  # Eq.3 on the GPU (a7)
    S = xyz.reshape(-1, 3).contiguous()
    src = S.cpu().numpy()
    th = np.deg2rad(0.3)
    Rm = torch.tensor([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]], dtype=torch.float64,
                      device=dev)
    T = (S.double() @ Rm.T + torch.tensor([0.05, 0.02, -0.03], dtype=torch.float64, device=dev)).float().contiguous()
    ms = timed(lambda: P.icp_register(S, T, max_iter=20, max_dist=0.25, eps=1e-7, stride=4), reps=5)
    o = P.icp_register(S, T, max_iter=20, max_dist=0.25, eps=1e-7, stride=4).cpu().numpy()
    res["f4_icp_lowres_cloud"] = {"ms_per_registration": ms, "points": int(np.sum(~np.isnan(src[:, 0]))),
                                  "stride": 4, "max_dist_m": 0.25, "iterations": int(o[13]), "pairs": int(o[15]), "rms_m": float(o[12])}
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
