#!/usr/bin/env python
"""CUDA-event timing of bp_disparity_batch for one configuration (default C4:
1352x760, L=128, 6 levels x 8 iterations, 8 pairs) with per-level update times;
A/B knobs through the environment (VSBP_PAIR, VSBP_PAIR_MINPX, VSBP_PAIR_BAND).
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_09733_b200 as P  # noqa: E402
import synthgen  # noqa: E402

W, H, L, LV, IT, B = (int(v) for v in os.environ.get("BP_CFG", "1352,760,128,6,8,8").split(","))
s = 2704 // W
left, right, _ = synthgen.stereo_pair_rgb(0, s=s, dmin=16 if L == 128 else 8, dmax=96 if L == 128 else 48)
Lt = torch.from_numpy(left).cuda().expand(B, -1, -1, -1).contiguous()
Rt = torch.from_numpy(right).cuda().expand(B, -1, -1, -1).contiguous()
gl, gr = P.prep_downsample(Lt, s), P.prep_downsample(Rt, s)
bp = P.StereoBP(W, H, L, LV, IT, batch=B, device="cuda")
bp.timing(True)
out = torch.empty((B, H, W), dtype=torch.int32, device="cuda")
for _ in range(3):
    bp.disparity(gl, gr, out=out)
torch.cuda.synchronize()
bp.timing_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    bp.disparity(gl, gr, out=out)
e1.record()
torch.cuda.synchronize()
lv = bp.timing_read()
print(json.dumps({"cfg": [W, H, L, LV, IT, B], "env": {k: v for k, v in os.environ.items() if k.startswith("VSBP_")},
                  "ms_per_pair": e0.elapsed_time(e1) / reps / B,
                  "level_ms_per_pair": [round(x["ms"] / reps / B, 4) for x in lv]}))
