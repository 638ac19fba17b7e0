#!/usr/bin/env python
"""CUDA-event timing of compact_cloud_batch at the bench's batch (128 pairs of
2704 x 1520, ~99 % valid) -- A/B experiments on the a8 kernel.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_09733_b200 as P  # noqa: E402

B, W, H = int(os.environ.get("B", "128")), 2704, 1520
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
disp = torch.rand((B, H, W), generator=g, device=dev) * 200.0
disp[torch.rand((B, H, W), generator=g, device=dev) < 0.01] = 0.0
Q = P.q_matrix(1400.0, 1400.0, 1351.5, 759.5, 0.5)
comp = P.CloudCompactor(W, H, B, device=dev)
xyz = torch.empty((B * H * W, 3), dtype=torch.float32, device=dev)
for _ in range(3):
    comp(disp, Q, 1.0, xyz=xyz)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    _, off, nv = comp(disp, Q, 1.0, xyz=xyz)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
pts = int(off[-1])
byts = B * H * W * 4 + pts * 12
print(json.dumps({"ms": ms, "points": pts, "GB": byts / 1e9, "GBs": byts / 1e9 / (ms / 1e3)}))
