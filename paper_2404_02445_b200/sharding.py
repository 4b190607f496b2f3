"""Data-parallel sharding of the (window, channel) series across ranks
(SURVEY.md §8(e)): every series is independent, so windows are split into
contiguous balanced ranges with no exchange on the hot path.  The only
collective is the final all-reduce of the fp64 error sums that form MSE/MAE
(PAPER.md:22 accuracy metric)."""
from __future__ import annotations


def shard_windows(B: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of rank's contiguous window range: the first B % world
    ranks take one extra window; start_k = k*floor(B/P) + min(k, B mod P)."""
    if world < 1 or not 0 <= rank < world or B < 0:
        raise ValueError(f"bad shard request B={B} world={world} rank={rank}")
    q, rem = divmod(B, world)
    start = rank * q + min(rank, rem)
    return start, q + (1 if rank < rem else 0)


def all_reduce_error_sums(sums, group=None):
    """In-place SUM all-reduce of a 3-element fp64 tensor {SSE, SAE, count}
    (NCCL on GPU tensors, gloo on CPU tensors); returns (MSE, MAE)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    s = sums.detach().cpu().tolist()
    return s[0] / s[2], s[1] / s[2]
