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
