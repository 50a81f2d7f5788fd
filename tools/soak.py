"""Soak test: streams randomly sized batches (sizes, modes, bundles, grey /
PPM / f64 input, device-resident calls, submit / wait with two in flight)
through long-lived extractors for a fixed time, checking every container
against the same frame's container from a fresh context (the encode is pure
per frame) and a sample against the oracle; reports device memory before /
after (a leak shows up as growth).
   python tools/soak.py [minutes]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle_lib  # noqa: E402
import paper_1705_09776_b200 as cg  # noqa: E402

minutes = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
rng = np.random.default_rng(20261017)
texts = {"b8": oracle_lib.bundle_text("b8"), "b512": oracle_lib.bundle_text("b512")}
exs = {k: cg.Extractor(v, max_batch=64) for k, v in texts.items()}
# Streamed calls get their own extractors: a context refuses a synchronous
# call while one of its submitted batches is in flight.
streams = {k: cg.Extractor(v, max_batch=64) for k, v in texts.items()}


def mem_used():
    out = os.popen("nvidia-smi --query-gpu=memory.used --format=csv,noheader,nounits").read().strip().splitlines()
    return int(out[0]) if out else -1


start_mem = None
t_end = time.time() + 60 * minutes
calls = frames_done = mism = oracle_checked = 0
pending = []
while time.time() < t_end:
    bundle = "b512" if rng.random() < 0.25 else "b8"
    ex = exs[bundle]
    w, h = int(rng.integers(64, 1300)), int(rng.integers(64, 900))
    n = int(rng.integers(1, 40))
    mode = int(rng.integers(0, 6))
    kind = rng.choice(["grey", "grey", "stream", "rgb", "f64"])
    seed = int(rng.integers(1, 1 << 30))
    if kind == "rgb":
        frames = oracle_lib.synth_rgb(seed, n, w, h)
    else:
        frames = oracle_lib.synth_frames(seed, n, w, h)
    if kind == "stream":
        pending.append((streams[bundle].encode_batch_submit(frames, mode), frames, bundle, mode, kind))
        if len(pending) > 2:
            pb, fr, bd, md, kd = pending.pop(0)
            got, st = pb.wait()
        else:
            continue
    elif kind == "f64":
        fr, bd, md, kd = frames, bundle, mode, kind
        got, st = ex.encode_batch(frames.astype(np.float64) * (1.0 / 255.0), mode)
    else:
        fr, bd, md, kd = frames, bundle, mode, kind
        got, st = ex.encode_batch(frames, mode)
    if start_mem is None:
        start_mem = mem_used()
    calls += 1
    frames_done += len(got)
    # Re-encode one frame on a fresh context: the encode is pure per frame.
    k = int(rng.integers(0, len(got)))
    fresh = cg.Extractor(texts[bd], max_batch=4)
    if kd == "f64":
        want, _ = fresh.encode_batch(fr[k:k + 1].astype(np.float64) * (1.0 / 255.0), md)
    else:
        want, _ = fresh.encode_batch(fr[k:k + 1], md)
    fresh.close()
    ok = bool((st == 0).all()) and got[k] == want[0]
    if calls % 10 == 0 and kd in ("grey", "stream"):
        ok = ok and got[k] == oracle_lib.encode(texts[bd], fr[k], md)
        oracle_checked += 1
    if not ok:
        mism += 1
        print("MISMATCH", calls, bd, w, h, n, md, kd, flush=True)
    if calls % 50 == 0:
        print(f"{calls} calls, {frames_done} frames, {mism} mismatches, GPU memory {mem_used()} MiB", flush=True)
for pb, *_ in pending:
    pb.wait()
end_mem = mem_used()
print(f"soak: {calls} calls, {frames_done} frames in {minutes} min, {mism} mismatches, "
      f"{oracle_checked} oracle checks, GPU memory {start_mem} -> {end_mem} MiB")
