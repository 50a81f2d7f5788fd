"""Retrieval benchmark: the reference's retrieve
(proj/src/eval.cpp:76-124) for a batch of queries over an index of CDVZ1
containers, on one B200, next to the CPU oracle on the host cores.

  python bench_retrieval.py [--index 65536 --queries 256 --depth 50]

The containers are the extractor's own output (4K mode, B8 bundle) for
synthetic VGA frames generated on the device (seeds 1000 + i*golden for the
index; queries are index members and unseen frames, half each). Timed with the
host clock around the synchronous C ABI calls, so host->device copies of the
query containers and the device->host copy of every ranked list are inside.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--index", type=int, default=65536)
    ap.add_argument("--queries", type=int, default=256)
    ap.add_argument("--depth", type=int, default=50)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--cpu-queries", type=int, default=4)
    args = ap.parse_args()
    import oracle_lib
    import paper_1705_09776_b200 as cg

    bundle = oracle_lib.bundle_text("b8")
    ex = cg.Extractor(bundle, max_batch=512)
    mode = cg.mode_by_name("4K")
    slot = cg.container_slot(mode)

    def encode(seed, count):
        out = []
        d_frames = ex.synth_frames_device(seed, count, 640, 480)
        d_out = ex.device_buffer(count * slot)
        d_len = ex.device_buffer(count * 4)
        ex.encode_device(d_frames, count, 640, 480, mode, d_out, d_len)
        raw = d_out.to_host(count * slot).tobytes()
        lens = np.frombuffer(d_len.to_host(count * 4).tobytes(), dtype=np.uint32)
        for i in range(count):
            out.append(raw[i * slot:i * slot + int(lens[i])])
        for b in (d_frames, d_out, d_len):
            b.free()
        return out

    t0 = time.perf_counter()
    index = []
    for base in range(0, args.index, 4096):
        index += encode(1000 + base, min(4096, args.index - base))
    t_encode = time.perf_counter() - t0
    unseen = encode(9_000_000, args.queries - args.queries // 2)
    queries = index[: args.queries // 2] + unseen

    t0 = time.perf_counter()
    idx = cg.Index(index)
    t_build = time.perf_counter() - t0
    info = idx.info()
    idx.retrieve_batch(queries[:8], 0.85, args.depth, max_results=0)  # warm-up
    # The ranked lists (queries x index entries) land in pinned host buffers.
    nq, n = len(queries), info["count"]
    pin_i, pin_s = ex.pinned_buffer(4 * nq * n), ex.pinned_buffer(8 * nq * n)
    out = (pin_i.array.view(np.int32).reshape(nq, n), pin_s.array.view(np.float64).reshape(nq, n))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        items, scores = idx.retrieve_batch(queries, 0.85, args.depth, max_results=0, out=out)
        times.append(time.perf_counter() - t0)
    best = min(times)
    med = sorted(times)[len(times) // 2]
    self_first = float(np.mean(items[: args.queries // 2, 0] == np.arange(args.queries // 2)))

    # CPU oracle on a bounded sample: retrieve over the same index for a few
    # queries, minus the oracle's index parse (timed with zero queries).
    cpu = None
    if args.cpu_queries > 0:
        sample = queries[: args.cpu_queries]
        t0 = time.perf_counter()
        oi, os_ = oracle_lib.retrieve(index, sample, 0.85, args.depth)
        t_all = time.perf_counter() - t0
        gi, gs = idx.retrieve_batch(sample, 0.85, args.depth)
        cpu = {"queries_per_s": len(sample) / t_all, "cores": 1, "kind": "port",
               "sample": f"{len(sample)} queries over the same {len(index)}-container index, single-threaded oracle "
                         "(reference's retrieve restated; includes its parse of the index once)",
               "parity": bool(np.array_equal(gi, oi) and np.array_equal(gs, os_))}
    idx.close()
    ex.close()
    line = {
        "metric": "retrieval queries/s (retrieve, 4K mode containers, rerank depth 50)", "value": args.queries / med,
        "unit": "queries/s", "best_value": args.queries / best, "n_gpus": 1, "steps": args.steps,
        "config": {"index_containers": len(index), "queries": args.queries, "rerank_depth": args.depth,
                   "ratio_test": 0.85, "components": info["components"], "index_codes": info["total_codes"],
                   "data": "synthetic VGA frames encoded by the extractor on the device"},
        "index_build_s": t_build, "index_build_containers_per_s": len(index) / t_build,
        "encode_s": t_encode, "self_retrieved_first": self_first,
        "output": f"{args.queries} x {len(index)} ranked (item, score) pairs copied to pinned host buffers per step",
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
