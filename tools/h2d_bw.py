#!/usr/bin/env python
"""Host -> device copy bandwidth from pinned memory (the link that binds bench.py's
e2e): one stream vs two / four streams, chunk sizes of one and several 2.7K frames.
CUDA events; prints one JSON line per variant."""
import json

import torch


def main():
    dev = torch.device("cuda:0")
    frame = 2704 * 1520 * 3
    total = 64 * frame
    host = torch.empty(total, dtype=torch.uint8).pin_memory()
    dst = torch.empty(total, dtype=torch.uint8, device=dev)
    for nstreams in (1, 2, 4):
        for chunk_frames in (1, 8):
            chunk = chunk_frames * frame
            streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
            main_s = torch.cuda.current_stream(dev)

            def run():
                ev = torch.cuda.Event()
                ev.record(main_s)
                for s in streams:
                    s.wait_event(ev)
                for i, off in enumerate(range(0, total, chunk)):
                    s = streams[i % nstreams]
                    with torch.cuda.stream(s):
                        dst[off:off + chunk].copy_(host[off:off + chunk], non_blocking=True)
                for s in streams:
                    e = torch.cuda.Event()
                    e.record(s)
                    main_s.wait_event(e)

            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            for _ in range(5):
                run()
            e1.record(main_s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(json.dumps({"streams": nstreams, "chunk_MB": chunk / 1e6, "GB_per_s": total / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
