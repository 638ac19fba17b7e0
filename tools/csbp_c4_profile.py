#!/usr/bin/env python
"""A few C4 constant-space BP runs (1352x760, L=128, 6 levels x 8 iterations, k0 from
argv, 4 pairs) -- the command ncu captures for the f2 per-kernel roofline."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_09733_b200 as P  # noqa: E402
import synthgen  # noqa: E402

k0 = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = 4
left, right, _ = synthgen.stereo_pair_rgb(0, s=2, dmin=16, dmax=96)
L = torch.from_numpy(left).cuda().expand(B, -1, -1, -1).contiguous()
R = torch.from_numpy(right).cuda().expand(B, -1, -1, -1).contiguous()
gl, gr = P.prep_downsample(L, 2), P.prep_downsample(R, 2)
cs = P.ConstantSpaceBP(1352, 760, 128, 6, 8, k0, batch=B, device="cuda")
for _ in range(2):
    cs.disparity(gl, gr)
torch.cuda.synchronize()
print("ok")
