"""Multi-GPU plumbing of the stereo stream: pure host
logic, no arithmetic of the method.

Virtual-stereo pairs are independent units ("each pair is processed
independently"; BASELINE.json "independent frame pairs ... sharded across the 8
GPUs"), so the stream is sharded with no data-path collective:

* batch k of the global stream (pairs k*B .. k*B+B-1) belongs to rank k mod N
  (round-robin over batches -- every rank gets the same number of pairs, and a
  rank's s-th batch is global batch s*N + rank);
* the only exchange is one all_gather per step of the per-pair 64-byte summaries
  (a8: n_valid, label sum, label hash, pair id), which rank 0 reassembles in pair
  order.

Everything here runs on CPU tensors with the gloo backend as well as on device
tensors with NCCL; the tests exercise it with world_size 2 on gloo.
"""
from __future__ import annotations

import torch

SUMMARY_WORDS = 8   # int64 words per pair: n_valid, label_sum, label_hash, pair_id, 4 reserved
PAIR_ID = 3         # column of the pair id


def batch_first_pair(step: int, rank: int, world: int, batch: int) -> int:
    """Global id of the first pair of rank `rank`'s `step`-th batch."""
    if not (0 <= rank < world) or batch < 1 or step < 0:
        raise ValueError("bad shard arguments")
    return (step * world + rank) * batch


def batch_frames(step: int, rank: int, world: int, batch: int, n_pairs: int) -> tuple[int, int]:
    """Frames (first, count) of rank `rank`'s `step`-th batch of a video stream of
    n_pairs pairs, pair k = (frame k, frame k+1): frames first .. first+count-1,
    count = pairs + 1 (0 when the rank has no pair left)."""
    first = batch_first_pair(step, rank, world, batch)
    pairs = max(0, min(batch, n_pairs - first))
    return first, pairs + 1 if pairs else 0


def rank_of_pair(pair: int, world: int, batch: int) -> int:
    return (pair // batch) % world


def local_pairs(n_pairs: int, rank: int, world: int, batch: int) -> list[int]:
    """Global pair ids rank `rank` processes out of a stream of n_pairs."""
    return [p for p in range(n_pairs) if rank_of_pair(p, world, batch) == rank]


def steps_for(n_pairs: int, world: int, batch: int) -> int:
    """Steps (batches per rank) needed to cover n_pairs; the last may be partial."""
    per_step = world * batch
    return (n_pairs + per_step - 1) // per_step


def gather_summaries(summary: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """all_gather of every rank's [B, 8] int64 summary block into [world*B, 8]
    (rank-major).  The one collective of the path; on the same stream as the
    producer when NCCL is the backend."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if out is None:
        out = torch.empty((world * summary.shape[0], summary.shape[1]), dtype=summary.dtype, device=summary.device)
    if world == 1:
        out.copy_(summary)
    else:
        dist.all_gather_into_tensor(out, summary.contiguous(), group=group)
    return out


def assemble(gathered: torch.Tensor, n_pairs: int | None = None) -> torch.Tensor:
    """Rank-major gathered summaries -> rows in global pair order.  Checks that
    every pair id appears exactly once (and, with n_pairs, that the ids are
    exactly a contiguous window of n_pairs); padding rows (pair id < 0) of a
    partial last step are dropped."""
    g = gathered.cpu()
    keep = g[:, PAIR_ID] >= 0
    g = g[keep]
    order = torch.argsort(g[:, PAIR_ID], stable=True)
    g = g[order]
    ids = g[:, PAIR_ID]
    if ids.numel() and torch.any(ids[1:] == ids[:-1]):
        raise RuntimeError("a pair id was processed twice")
    if n_pairs is not None:
        if ids.numel() != n_pairs or (n_pairs and int(ids[-1] - ids[0]) != n_pairs - 1):
            raise RuntimeError(f"expected {n_pairs} contiguous pair ids, got {ids.numel()}")
    return g
