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


def _worker(rank, world, port, n, out_q, real):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(n, rank, world)
    if real:
        # The real per-frame encoder on this CPU-only box: the oracle (the
        # reference's algorithm, the checker the GPU is compared with), on
        # this rank's contiguous shard of seeded frames.
        import oracle_lib

        text = oracle_lib.bundle_text("b8")
        frames = oracle_lib.synth_frames(500, n, 160, 120)
        local = [oracle_lib.encode(text, frames[i], 3) for i in range(b, e)]
    else:
        local = [b"CDVZ1" + i.to_bytes(4, "little") for i in range(b, e)]
    allc = gather_containers(local, rank, world)
    out_q.put((rank, allc if real else [int.from_bytes(c[5:9], "little") for c in allc]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 64])
def test_gloo_world2_gather_preserves_frame_order(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q, False)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == list(range(n)) and results[1] == list(range(n))


def test_gloo_world2_real_containers_equal_one_process():
    """Two gloo ranks encode their shards of 5 frames with the real encoder
    (the CPU oracle here; the GPU multi-device path is covered by
    tests/test_gpu_boundary.py) and gather: both ranks hold every container,
    in frame order, identical to a single-process encode."""
    import oracle_lib

    n = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    text = oracle_lib.bundle_text("b8")
    frames = oracle_lib.synth_frames(500, n, 160, 120)
    want = [oracle_lib.encode(text, frames[i], 3) for i in range(n)]
    assert results[0] == want and results[1] == want
