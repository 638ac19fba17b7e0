#!/usr/bin/env python
"""bench.py -- 2.7K frame pairs/s of the stereo hot path (a0-a8) on 1..N B200s.

Contract (driver): `python bench.py --gpus N --steps K --warmup W [--impl reference]`,
torchrun for N > 1 (one rank per GPU, NCCL).  Rank 0 prints ONE JSON line.

Workload (BASELINE.json configs[4], the metric's configuration): a stream of 4096
virtual-stereo pairs of a synthetic 2.7K UAV video (synthgen/video.py, rendered
on the device by synthgen/libsynth.so before timing), pair k = (frame k, frame
k+1), so every frame is shared by two pairs.  One step =
one batch of B pairs (B+1 frames) per GPU through the whole path: prep (s=4) ->
hierarchical BP 676x380, L=64, 5 levels x 5 iterations -> JBU r=2 to 2704x1520
-> packed point clouds (Eq.3 + raster-order compaction) -> per-pair summary,
then the all_gather of the summaries on a side stream (the only exchange, SURVEY
§8e).  Batches go round-robin to the ranks (batch g -> rank g mod N, shard.py):
weak scaling; a rank cycles over its share of the stream.

`value`  : pairs/s over all ranks, inputs resident in HBM, device-timed (CUDA
           events on the launching stream, max over ranks).
`e2e`    : the same through the public API (StereoStream) with pinned HOST frame
           batches, the H2D of each step's B+1 frames and the D2H of its
           (gathered) summaries inside the timed region.
`roofline`: the dominant kernel (level-0 message updates, a4): algorithmic bytes
           / device time from live CUDA events inside the timed region, against
           MEASURED_PEAKS.json hbm_gbs.
`cpu_baseline`: the oracle (oracle/) on the host cores, rank 0 at N=1.
`--impl reference`: the oracle as the reference arm (this tier has no
           reference implementation).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "2.7K frame pairs/sec (disparity+point cloud) at 1/2/4/8 B200; HBM GB/s % peak"
W_HI, H_HI, S_DOWN, NDISP, LEVELS, ITERS = 2704, 1520, 4, 64, 5, 5
FEATURES = dict(gc=30, gr=30, K=4, thr=10 ** 9, r=5, sr=48)  # f3 on the 676x380 grey pair (P:84 grid)
CAMERA = (1400.0, 1400.0, 1351.5, 759.5, -0.25, 0.08, -0.01)  # f1: GoPro-like radial model
WORKLOAD = ("C5: stream of 4096 virtual-stereo pairs of a synthetic 2.7K video (pair k = frames k, k+1), full "
            "pipeline a0-a8 (prep s=4 -> BP 676x380 L=64 5 levels x 5 iters -> JBU r=2 to 2704x1520 -> Eq.3 + "
            "packed point cloud -> summary -> gather)")
LABELS = (8, 48)  # the video's true disparity range at the BP resolution (C2/C3: [8, 48] of L = 64)
JBU_RADIUS = None  # --jbu-radius (None: ceil(5 / s))
CONFIG = 5


def set_config(n: int):
    """--config: 5 (default) = BASELINE configs[4], the C5 stream above; 4 = configs[3],
    the same video stream through the same pipeline at 1352x760 (s = 2), L = 128,
    6 levels x 8 iterations, JBU r = 3 to 2.7K (BASELINE.json configs)."""
    global S_DOWN, NDISP, LEVELS, ITERS, WORKLOAD, LABELS, CONFIG
    CONFIG = n
    if n == 4:
        S_DOWN, NDISP, LEVELS, ITERS = 2, 128, 6, 8
        LABELS = (16, 96)
        WORKLOAD = ("C4: stream of virtual-stereo pairs of a synthetic 2.7K video (pair k = frames k, k+1), full "
                    "pipeline a0-a8 (prep s=2 -> BP 1352x760 L=128 6 levels x 8 iters -> JBU r=3 to 2704x1520 -> "
                    "Eq.3 + packed point cloud -> summary -> gather)")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=60)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, choices=[4, 5], default=5,
                   help="BASELINE.json config: 5 = the C5 stream (default, the headline); 4 = the C4 resolution "
                        "(1352x760, L = 128, 6 x 8) on the same stream")
    p.add_argument("--batch", type=int, default=0,
                   help="pairs per GPU per step (default 256 at C5 -- measured 96 / 128 / 192 / 256 -> "
                        "8550 / 8662 / 8759 / 8805 pairs/s; 51.6 GB of BP state -- and 16 at C4, whose BP state "
                        "is 1.4 GB per pair)")
    p.add_argument("--jbu-radius", type=int, default=0, help="JBU window radius (default ceil(5 / s): 2 at C5)")
    p.add_argument("--msg-bytes", type=int, default=0, choices=[0, 1, 2, 4],
                   help="BP message storage bytes (0: the smallest lossless, u8 here)")
    p.add_argument("--pairs", type=int, default=4096, help="length of the synthetic stream (C5: 4096 pairs)")
    p.add_argument("--seed", type=int, default=1902)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-threads", type=int, default=0)
    p.add_argument("--cpu-pairs", type=int, default=4, help="oracle pairs per host thread (cpu_baseline)")
    p.add_argument("--csbp", type=int, default=0, metavar="K0",
                   help="row f2: constant-space BP with k_l = min(L, K0 2^l) candidates instead of the full BP")
    p.add_argument("--features", action="store_true",
                   help="row f3: Harris corners (30x30 grid) on the left frame + ZSSD matching into the right")
    p.add_argument("--rectify", action="store_true",
                   help="row f1: undistort the raw frames (GoPro-like radial model) before a0")
    return p.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "samples": len(sm),
                "reasons": sorted(reasons)}


def video_scene(seed: int):
    from synthgen.video import VideoScene
    return VideoScene(seed, W_HI, H_HI, S_DOWN, *LABELS)


def host_frames(seed: int, k0: int, n: int):
    """n consecutive frames of the video as numpy (device generator when a GPU is
    present; the bit-identical numpy twin otherwise, ~15 s per frame)."""
    from synthgen import video
    sc = video_scene(seed)
    try:
        import torch
        if torch.cuda.is_available():
            out = torch.empty((n, H_HI, W_HI, 3), dtype=torch.uint8, device="cuda")
            video.frames_device(sc, k0, out)
            return out.cpu().numpy()
    except ImportError:
        pass
    return np.stack([sc.frame(k0 + i) for i in range(n)])


def q_intrinsics():
    import synthgen
    I = synthgen.INTRINSICS
    return I


def ncu_pipes(batch: int):
    """ncu pipe utilisation (% of peak sustained) of the captured level-0 update
    launches (profiles/traffic.json, same command and batch), or None"""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    if int(d.get("batch", -1)) != batch:
        return None
    return {k: v for k, v in (d.get("pipes_pct") or {}).items() if k.startswith("k_update_pair")} or None


def ncu_traffic(batch: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per level-0 message-update launch
    (mean over the fused two-iteration and the one-iteration launches of an ncu launch
    list of the same command, profiles/traffic.json), when that list was taken at this
    batch size; else None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    if int(d.get("batch", -1)) != batch:
        return None
    v = (d.get("level0_update") or {}).get("bytes_per_launch")
    return float(v) if v is not None else None


# ----------------------------------------------------------------------------- oracle timing
def oracle_rate(n_threads: int, pairs_per_thread: int, frames):
    """Run the oracle pipeline (a0-a8) on n_threads host threads (ctypes releases the
    GIL), each on pairs_per_thread pairs (frames[i], frames[i+1]) of the video;
    returns (pairs/s, pairs, seconds)."""
    import oracle
    I = q_intrinsics()
    Q = oracle.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])

    def work(k):
        for j in range(pairs_per_thread):
            i = (k + j) % (len(frames) - 1)
            d, hi, xyz, n = oracle.pipeline_pair(frames[i], frames[i + 1], S_DOWN, NDISP, LEVELS, ITERS, Q,
                                                 radius=JBU_RADIUS)
            oracle.compact_cloud(hi, Q, 1.0)  # a8: the packed cloud, as the GPU path

    ts = [threading.Thread(target=work, args=(k,)) for k in range(n_threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    n = n_threads * pairs_per_thread
    return n / dt, n, dt


def default_threads():
    try:
        c = len(os.sched_getaffinity(0))
    except AttributeError:
        c = os.cpu_count() or 1
    return max(1, min(c, 32))


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    threads = args.cpu_threads or default_threads()
    frames = host_frames(args.seed, 0, threads + 1)
    for _ in range(args.warmup):  # untimed rounds
        oracle_rate(threads, 1, frames)
    times, pairs = 0.0, 0
    for _ in range(args.steps):
        _, n, dt = oracle_rate(threads, 1, frames)
        times += dt
        pairs += n
    v = pairs / times
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * times / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": {"workload": WORKLOAD, "pairs_per_step": threads},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": threads, "kind": "oracle",
                         "sample": f"{threads} pairs per step (one per host thread, consecutive frames of the "
                                   f"C{CONFIG} video), {args.steps} steps"},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1902_09733_b200 as P
    from paper_1902_09733_b200 import shard

    rank, world, local_rank = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        # keep NCCL's communicator-init lines in the log (the driver's rank check reads them)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    P.lib()
    B = args.batch
    I = q_intrinsics()
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    pipe = P.StereoPipeline(W_HI, H_HI, S_DOWN, NDISP, LEVELS, ITERS, batch=B, Q=Q, device=dev,
                            radius=args.jbu_radius or None, msg_bytes=args.msg_bytes,
                            camera=CAMERA if args.rectify else None,
                            features=FEATURES if args.features else None, csbp_k0=args.csbp or None)
    full_bp = isinstance(pipe.bp, P.StereoBP)
    if full_bp:
        pipe.bp.timing(True)

    # the C5 stream: pair k = (frame k, frame k+1) of one synthetic video; rank r owns
    # global batches r, r+N, ... (shard.py), each B+1 frames, rendered into HBM now
    from synthgen import video
    scene = video_scene(args.seed)
    nbatch = (args.pairs + B - 1) // B
    local = [g for g in range(nbatch) if g % world == rank] or [rank]
    frames = torch.empty((len(local), B + 1, H_HI, W_HI, 3), dtype=torch.uint8, device=dev)
    for li, g in enumerate(local):
        video.frames_device(scene, g * B, frames[li])
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(device=dev)
    RING = 4
    sdev = [torch.empty((B, 8), dtype=torch.int64, device=dev) for _ in range(RING)]
    gdev = [torch.empty((world * B, 8), dtype=torch.int64, device=dev) for _ in range(RING)]
    produced = [torch.cuda.Event() for _ in range(RING)]
    consumed = [torch.cuda.Event() for _ in range(RING)]

    def step(s):
        li = s % len(local)
        r = s % RING
        stream.wait_event(consumed[r])
        summ = pipe.run_frames(frames[li], first_pair_id=local[li] * B, summary_out=sdev[r])
        produced[r].record(stream)
        with torch.cuda.stream(side):  # the one exchange, off the compute stream
            side.wait_event(produced[r])
            shard.gather_summaries(summ, out=gdev[r])
            consumed[r].record(side)
        return summ

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for s in range(args.warmup):
        step(s)
    if full_bp:
        pipe.bp.timing_read()  # discard warm-up timings
    P.jbu_timing(True)  # the JBU kernel's own CUDA events inside the timed steps (second roofline)
    barrier()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    n0 = P.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for s in range(args.steps):
        step(args.warmup + s)
    stream.wait_stream(side)
    e1.record(stream)
    barrier()
    launches = P.launch_count() - n0
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms)
    lv = pipe.bp.timing_read() if full_bp else None
    jt = P.jbu_timing_read()
    P.jbu_timing(False)
    pairs = world * B * args.steps
    value = pairs / (ms_max / 1000.0)
    n_valid_last = int(pipe.offsets[B].item()) if pipe.offsets is not None else None

    # ---- e2e: pinned host frame batches in, summaries out, through the public API
    e2e = None
    if not args.no_e2e:
        runner = P.StereoStream(pipe, device=dev, ring=RING, world=world)
        hb = [frames[i % len(local)].cpu().pin_memory() for i in range(2)]  # two distinct host batches
        gather = (lambda summ, out: shard.gather_summaries(summ, out=out))
        got = []
        runner.run(hb, gather=gather)  # warm the copy path
        barrier()
        runner.h2d_bytes = runner.d2h_bytes = 0
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        runner.run([hb[i & 1] for i in range(args.steps)], first_pair_id=shard.batch_first_pair(0, rank, world, B),
                   pair_stride=world * B, gather=gather, on_summary=lambda i, t: got.append(i))
        f1.record(stream)
        barrier()
        assert got == list(range(args.steps)), "a batch's summaries never reached the host"
        ems = max_over_ranks(f0.elapsed_time(f1))
        e2e = {"value": pairs / (ems / 1000.0), "unit": "pairs/s",
               "h2d_gbs_per_gpu": runner.h2d_bytes / (ems / 1000.0) / 1e9,
               "h2d_bytes_per_step": int(runner.h2d_bytes // args.steps),
               "d2h_bytes_per_step": int(runner.d2h_bytes // args.steps),
               "h2d_bytes_per_pair": runner.h2d_bytes / (args.steps * B),
               "overlap": "H2D of batch i+1 on a copy stream during compute of batch i; gather + D2H of the "
                          "summaries on a side stream"}
        if full_bp:
            pipe.bp.timing_read()
        del hb

    # ---- roofline of the dominant kernel: level-0 message updates (a4)
    peak, peak_kind = measured_peaks()
    roofline = None
    if full_bp:
        l0 = lv[0]
        achieved = (l0["bytes"] / 1e9) / (l0["ms"] / 1e3) if l0["ms"] > 0 else 0.0
        all_bytes = sum(x["bytes"] for x in lv)
        all_ms = sum(x["ms"] for x in lv)
        roofline = {
            "kernel": "level-0 message updates (a3+a4): k_update_pair (two iterations per launch; the last "
                      "iteration fused with the WTA of both colours, a5)", "bound": "hbm", "achieved": achieved,
            "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(B),
            # what binds it instead of HBM: the integer ALU pipe (ncu, same command)
            "pipes_pct_ncu": ncu_pipes(B),
            "bytes_per_launch": l0["bytes"] / max(l0["launches"], 1),
            "us_per_launch": 1000.0 * l0["ms"] / max(l0["launches"], 1),
            "share_of_step": all_ms / (ms if ms > 0 else 1.0),
            "all_levels_gbs": (all_bytes / 1e9) / (all_ms / 1e3) if all_ms > 0 else 0.0,
            "note": "bytes = the fused schedule's algorithmic bytes (a two-iteration launch moves 10L per pixel "
                    "pair, 0.56x two one-iteration launches; the fused last iteration + WTA moves D of both colours and "
                    "one colour's 4 incoming messages, 6L per pixel pair). Fusion trades HBM bytes for on-chip "
                    "work: k_update_pair is bound by the integer ALU pipe (pipes_pct_ncu; the pipe runs 64 "
                    "lane-ops/clk/SM, tools/micro/alu_bench), so its HBM fraction is not its binding roofline",
        }

    # ---- second roofline: the JBU kernel (a6 + the a8 counts), bound by MUFU.EX2 (one per
    # pixel-tap); peak = 16 EX2 lanes / clk / SM (tools/micro/mufu_bench measured 15.8)
    # x SMs x the SM clock sampled during the timed steps
    roofline_jbu = None
    if jt["launches"] > 0 and jt["ms"] > 0:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        peak_t = 16.0 * sms * mhz * 1e6 / 1e9  # G pixel-taps/s
        ach_t = (jt["taps"] / 1e9) / (jt["ms"] / 1e3)
        roofline_jbu = {"kernel": "k_jbu_vec (a6 JBU + a8 segment counts)", "bound": "xu (MUFU.EX2)",
                        "achieved": ach_t, "peak": peak_t, "unit": "G pixel-taps/s", "frac": ach_t / peak_t,
                        "us_per_launch": 1000.0 * jt["ms"] / jt["launches"],
                        "taps_per_launch": jt["taps"] / jt["launches"],
                        "note": "one weight 2^x (one MUFU.EX2) per output pixel and window tap; peak from the "
                                "nominal 16 EX2 lanes/clk/SM at the sampled SM clock"}

    # ---- CPU baseline: the oracle on this host's cores (rank 0 at N=1 only)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = args.cpu_threads or default_threads()
        fr = frames[0, : min(threads, B) + 1].cpu().numpy()
        v, n, dt = oracle_rate(threads, args.cpu_pairs, fr)
        cpu = {"value": v, "unit": "pairs/s", "cores": threads, "kind": "oracle",
               "sample": f"{n} pairs of the same workload (consecutive frames of the C{CONFIG} video), one thread per "
                         f"pair at a time ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": WORKLOAD + (" + f1 undistortion of the raw frames" if args.rectify else "")
                       + (" + f3 Harris/ZSSD correspondences (sr=48)" if args.features else "")
                       + (f" with f2 constant-space BP (k0={args.csbp})" if args.csbp else ""),
                       "batch_per_gpu": B, "pairs_per_step": world * B,
                       "parallelism": f"dp{world} (pairs round-robin, NCCL all_gather of summaries)",
                       "stream_pairs": nbatch * B, "frames_in_hbm": int(frames.shape[0] * frames.shape[1]),
                       "frames_per_step": B + 1, "cloud": "packed (raster-order valid points, offsets per pair)",
                       "l2": f"inputs larger than L2 ({frames[0].numel() / 1e6:.0f} MB RGB + "
                             f"{pipe.bp.workspace.numel() / 1e6:.0f} MB BP state per step, a different batch "
                             f"of the stream every step)",
                       "bp_msg_storage": f"u{8 * pipe.bp.params()['msg_bytes']}" if full_bp else "i32 (csbp)",
                       "jbu_arith": "f32"},
            "clocks": clocks, "gpu_launches": int(launches), "e2e": e2e, "roofline": roofline,
            "roofline_jbu": roofline_jbu,
            "cpu_baseline": cpu,
            "per_level_update_ms_per_step": [x["ms"] / args.steps for x in lv] if lv else None,
            "last_batch_points": n_valid_last,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    set_config(args.config)
    global JBU_RADIUS
    JBU_RADIUS = args.jbu_radius or None
    if not args.batch:
        args.batch = 256 if args.config == 5 else 16
    if args.config == 4 and args.cpu_pairs == 4:
        args.cpu_pairs = 1  # the oracle takes ~22 s per C4 pair on one core
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
