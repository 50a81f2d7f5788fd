"""CPU: frame sharding across ranks (gloo, world size 2) — the multi-GPU
layout of bench.py --gpus N and of any multi-GPU deployment: contiguous
frame ranges, no data-path collective, bitstreams gathered in frame order."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_09776_b200.sharding import gather_containers, shard_range


def test_shard_ranges_tile_the_batch():
    for n in (0, 1, 7, 1024, 65536, 65537):
        for world in (1, 2, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(n, rank, world)
    # Stand-in encoder: a deterministic per-frame "container".
    local = [b"CDVZ1" + i.to_bytes(4, "little") for i in range(b, e)]
    allc = gather_containers(local, rank, world)
    out_q.put((rank, [int.from_bytes(c[5:9], "little") for c in allc]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 64])
def test_gloo_world2_gather_preserves_frame_order(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == list(range(n)) and results[1] == list(range(n))
