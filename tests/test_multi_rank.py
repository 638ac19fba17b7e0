"""N>1 path on CPU (gloo, world_size 2): the pair sharding and the one exchange step
(all_gather of per-pair summaries, reassembled in pair order on rank 0) that
bench.py and the multi-GPU stream use (paper_1902_09733_b200/shard.py).

Each rank computes its shard's summaries with the oracle on small synthetic pairs
(the per-pair work is independent); rank 0 checks the gathered, reassembled
stream against a serial run over every pair."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1902_09733_b200 import shard

N_PAIRS, BATCH, WORLD = 11, 2, 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pair_summary_row(pair: int) -> list[int]:
    """The a8 summary of pair `pair` computed by the oracle (tiny BP problem)."""
    import oracle
    import synthgen
    left, right = synthgen.shifted_pair(500 + pair, 24, 12, 1 + pair % 5)
    disp = oracle.bp_disparity(left, right, 8, 2, 4)
    label_sum, label_hash = oracle.disp_summary(disp)
    h = label_hash if label_hash < 2 ** 63 else label_hash - 2 ** 64
    return [int(np.sum(disp >= 1)), label_sum, h, pair, 0, 0, 0, 0]


def _worker(rank: int, port: int, out_path: str):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        rows = []
        for step in range(shard.steps_for(N_PAIRS, WORLD, BATCH)):
            first = shard.batch_first_pair(step, rank, WORLD, BATCH)
            summ = torch.full((BATCH, shard.SUMMARY_WORDS), -1, dtype=torch.int64)
            for j in range(BATCH):
                if first + j < N_PAIRS:
                    summ[j] = torch.tensor(_pair_summary_row(first + j), dtype=torch.int64)
            rows.append(shard.gather_summaries(summ))
        if rank == 0:
            full = shard.assemble(torch.cat(rows), n_pairs=N_PAIRS)
            torch.save(full, out_path)
    finally:
        dist.destroy_process_group()


def test_sharding_covers_every_pair_once():
    for world in (1, 2, 3, 8):
        for batch in (1, 4, 16):
            seen = []
            for r in range(world):
                seen += shard.local_pairs(100, r, world, batch)
            assert sorted(seen) == list(range(100))
            for r in range(world):  # a rank's batches are global batches r, r+N, ...
                ids = shard.local_pairs(100, r, world, batch)
                firsts = [shard.batch_first_pair(s, r, world, batch) for s in range(shard.steps_for(100, world, batch))]
                assert ids == [f + j for f in firsts for j in range(batch) if f + j < 100]


def test_assemble_rejects_duplicates_and_gaps():
    rows = torch.zeros((4, 8), dtype=torch.int64)
    rows[:, shard.PAIR_ID] = torch.tensor([2, 0, 1, 2])
    with pytest.raises(RuntimeError):
        shard.assemble(rows)
    rows[:, shard.PAIR_ID] = torch.tensor([3, 0, 1, -1])
    with pytest.raises(RuntimeError):
        shard.assemble(rows, n_pairs=3)
    rows[:, shard.PAIR_ID] = torch.tensor([2, 0, 1, -1])
    assert shard.assemble(rows, n_pairs=3)[:, shard.PAIR_ID].tolist() == [0, 1, 2]


def test_world2_gloo_gather_matches_serial():
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "full.pt")
        mp.spawn(_worker, args=(port, out), nprocs=WORLD, join=True)
        full = torch.load(out)
    serial = torch.tensor([_pair_summary_row(p) for p in range(N_PAIRS)], dtype=torch.int64)
    assert torch.equal(full, serial)


# ----------------------------------------------------------------------------- the stream driver on 2 ranks
S_PAIRS, S_BATCH, S_H, S_W = 17, 3, 2, 5


def _frame(k: int) -> torch.Tensor:
    """a tiny frame whose first two bytes encode its index in the video"""
    f = torch.zeros((S_H, S_W, 3), dtype=torch.uint8)
    f[0, 0, 0], f[0, 0, 1] = k % 256, k // 256
    return f


class _FramePipe:
    """CPU stand-in for StereoPipeline.run_frames: the summary row of pair j records
    which frames it was given (left, right) and its pair id -- the host logic of
    StereoStream (frame routing, pair numbering, ring, gather, delivery) is what is
    under test, not the method's arithmetic."""

    def __init__(self):
        self.B, self.H_hi, self.W_hi = S_BATCH, S_H, S_W

    def run_frames(self, frames, first_pair_id=0, stream=None, summary_out=None):
        ids = frames[:, 0, 0, 0].to(torch.int64) + 256 * frames[:, 0, 0, 1].to(torch.int64)
        n = frames.shape[0] - 1
        summary_out.zero_()
        summary_out[:, 0] = ids[:n]
        summary_out[:, 1] = ids[1:n + 1]
        summary_out[:, shard.PAIR_ID] = first_pair_id + torch.arange(n)
        return summary_out


def _stream_worker(rank: int, port: int, out_path: str):
    import paper_1902_09733_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        runner = P.StereoStream(_FramePipe(), device="cpu", ring=2, world=WORLD)
        batches = []
        for step in range(shard.steps_for(S_PAIRS, WORLD, S_BATCH)):
            first, count = shard.batch_frames(step, rank, WORLD, S_BATCH, S_PAIRS)
            batches.append(torch.stack([_frame(first + i) for i in range(count)]) if count else None)
        got = []
        n = runner.run(batches, first_pair_id=shard.batch_first_pair(0, rank, WORLD, S_BATCH),
                       pair_stride=WORLD * S_BATCH,
                       gather=lambda summ, out: shard.gather_summaries(summ, out=out),
                       on_summary=lambda i, t: got.append((i, t)))
        assert n == len(batches) and [i for i, _ in got] == list(range(n)), "every batch delivered, in order"
        if rank == 0:
            full = shard.assemble(torch.cat([t for _, t in got]), n_pairs=S_PAIRS)
            torch.save(full, out_path)
    finally:
        dist.destroy_process_group()


def test_world2_stream_driver_routes_frames_and_numbers_pairs():
    """StereoStream.run(gather=..., pair_stride=world*B) on two
    gloo ranks over a shared-frame stream of 17 pairs in batches of 3 (the last batch
    of one rank short, the other rank's last step empty): after the all_gather and
    shard.assemble every pair p appears once, built from frames (p, p+1)."""
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "stream.pt")
        mp.spawn(_stream_worker, args=(port, out), nprocs=WORLD, join=True)
        full = torch.load(out)
    p = torch.arange(S_PAIRS)
    assert torch.equal(full[:, shard.PAIR_ID], p)
    assert torch.equal(full[:, 0], p) and torch.equal(full[:, 1], p + 1)


def test_stream_driver_single_process_delivers_every_batch():
    """every batch's summaries reach on_summary (ring smaller than the
    number of batches), with no gather."""
    import paper_1902_09733_b200 as P
    runner = P.StereoStream(_FramePipe(), device="cpu", ring=2, world=1)
    batches = [torch.stack([_frame(3 * i + j) for j in range(4)]) for i in range(5)]
    got = []
    runner.run(batches, on_summary=lambda i, t: got.append((i, t)))
    assert [i for i, _ in got] == list(range(5))
    for i, t in got:
        assert t[:, shard.PAIR_ID].tolist() == [3 * i + j for j in range(3)]
        assert t[:, 0].tolist() == [3 * i + j for j in range(3)] and t[:, 1].tolist() == [3 * i + j + 1 for j in range(3)]
