#!/usr/bin/env python
"""Experiment: the C5 step (B pairs of the video stream, a0-a8) as one pipeline on
one stream vs K pipelines of B/K pairs on K streams (the ALU-bound fused BP of one
sub-batch can overlap the EX2-bound JBU or the HBM-bound compaction of another).
CUDA events; prints one JSON line per variant."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1902_09733_b200 as P  # noqa: E402
from synthgen import video  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    B = int(os.environ.get("TS_BATCH", "128"))
    I = bench.q_intrinsics()
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    frames = torch.empty((B + 1, bench.H_HI, bench.W_HI, 3), dtype=torch.uint8, device=dev)
    video.frames_device(bench.video_scene(1902), 0, frames)
    for K in [int(k) for k in os.environ.get("TS_K", "1,2,4").split(",")]:
        n = B // K
        pipes = [P.StereoPipeline(bench.W_HI, bench.H_HI, bench.S_DOWN, bench.NDISP, bench.LEVELS, bench.ITERS,
                                  batch=n, Q=Q, device=dev) for _ in range(K)]
        streams = [torch.cuda.Stream(dev) for _ in range(K)]
        main_s = torch.cuda.current_stream(dev)

        def step():
            ev = torch.cuda.Event()
            ev.record(main_s)
            for k in range(K):
                streams[k].wait_event(ev)
                with torch.cuda.stream(streams[k]):
                    pipes[k].run_frames(frames[k * n:(k + 1) * n + 1], first_pair_id=k * n)
            for k in range(K):
                e = torch.cuda.Event()
                e.record(streams[k])
                main_s.wait_event(e)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 20
        e0.record(main_s)
        for _ in range(steps):
            step()
        e1.record(main_s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print(json.dumps({"batch": B, "streams": K, "pairs_per_stream": n, "ms_per_step": ms,
                          "pairs_per_s": B / (ms / 1e3)}), flush=True)
        del pipes
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
