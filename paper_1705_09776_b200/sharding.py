"""Frame sharding across GPUs: frames are independent, so
each rank (one process per GPU) encodes a contiguous frame range with its own
context and stream; no collective touches the data path. The host-side gather
of bitstreams in frame order is the only cross-rank step and happens once per
job, off the hot path."""
from __future__ import annotations

from typing import List, Sequence, Tuple


def shard_range(n_frames: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [begin, end) frame range of `rank`; ranges tile [0, n) in
    rank order and differ in size by at most one frame."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_frames, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_containers(local: Sequence[bytes], rank: int, world: int, group=None) -> List[bytes]:
    """Concatenates every rank's containers in frame order on all ranks
    (torch.distributed object gather over the host backend)."""
    if world == 1:
        return list(local)
    import torch.distributed as dist

    parts: List[object] = [None] * world
    dist.all_gather_object(parts, list(local), group=group)
    out: List[bytes] = []
    for p in parts:
        out.extend(p)  # rank order == frame order (shard_range is monotone)
    return out
