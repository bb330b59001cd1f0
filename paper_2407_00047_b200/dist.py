"""Data-parallel sharding of candidates and the cross-rank min-loc (a8, a12).

Candidates are independent units: rank r of W scores the contiguous global
index range shard_range(N, r, W) (weak scaling when every rank takes its own
N).  The only exchange is the argmin: every rank all-gathers the W 16-byte
best records (one NCCL call over NVLink) and reduces them with the
lexicographic (key, index) rule -- on the GPU with qlm_reduce_records.  MC
counts are summed with one all_reduce.  torch.distributed is plumbing only.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def attach_comm(est, group=None, unique_id=None):
    """Attach the library's own NCCL communicator to `est` (include/qlm.h
    qlm_comm_*): rank 0 creates the 128-byte unique id, torch.distributed
    broadcasts it (the only thing it carries), and every rank attaches.  From
    then on the library's argmin records are global and its MC counts are
    summed over ranks inside the C ABI; global_best / sum_counts pass through.
    """
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    make = unique_id if unique_id is not None else type(est).comm_unique_id
    on_gpu = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(make()), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    est.comm_attach(bytes(buf.cpu().numpy().tobytes()), rank, world)
    return est


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [first, first+count) of `total` candidates for `rank`."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_records(rec: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather each rank's int64[2] record -> int64[world*2] (same device).

    One NCCL all-gather of 16 B per rank over NVLink on the GPU path; the
    list form is used for backends without all_gather_into_tensor (gloo).
    """
    world = dist.get_world_size(group)
    rec = rec.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * 2, dtype=rec.dtype, device=rec.device)
        dist.all_gather_into_tensor(out, rec, group=group)
        return out
    parts = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(parts, rec, group=group)
    return torch.cat(parts)


def global_best(rec: torch.Tensor, reduce, group=None, est=None) -> torch.Tensor:
    """Global min-loc: gather all ranks' records, then `reduce(records)`.

    `reduce` is RwtEstimator.reduce_records on the GPU path.  When `est` has
    the library's communicator attached (attach_comm) its records are already
    global and this is the identity.
    """
    if est is not None and getattr(est, "comm_attached", False):
        return rec
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return rec
    return reduce(gather_records(rec, group))


def sum_counts(counts: torch.Tensor, group=None, est=None) -> torch.Tensor:
    if est is not None and getattr(est, "comm_attached", False):
        return counts                                   # summed inside the C ABI
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def local_search(est, row, moves: int = 2, per_iter: int = 1 << 16, iters: int = 16, seed: int = 1,
                 group=None):
    """Sharded iterated best-of-N over NEIGHBOR candidates (DESIGN R18).

    Iteration it's candidates [it*per_iter, (it+1)*per_iter) are split over
    the ranks with shard_range; each rank scores its slice, the iteration's
    winner is the global min-loc (global_best: one 16-B all-gather + reduce),
    and every rank adopts it with the same device-side rule, so the
    incumbent row stays identical on all ranks.  Equal to est.local_search on
    one rank.  Returns (row buffer, incumbent record).
    """
    if getattr(est, "comm_attached", False):          # the library shards and exchanges itself
        return est.local_search(row, moves, per_iter, iters, seed)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, n = shard_range(per_iter, rank, world)
    buf = est.row_buffer(row)
    inc = est.best_ordering_async(est.explicit(buf.view(1, -1)))
    inc[1:].fill_(-1)                                 # index -1: the start row is the incumbent
    for it in range(iters):
        cand = est.neighbor(buf, it * per_iter + lo, n, seed, moves)
        rec = est.best_ordering_async(cand)
        best = global_best(rec, est.reduce_records, group)
        est.adopt_best(cand, best, inc)
    return buf, inc
