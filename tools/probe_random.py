"""One-off: many seeded random configurations (size, aspect, mode, bundle,
max_side, grey or PPM colour input), GPU containers vs the oracle's.
python tools/probe_random.py [cases]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle_lib  # noqa: E402
import paper_1705_09776_b200 as cg  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(424242)
texts = {"b8": oracle_lib.bundle_text("b8"), "b512": oracle_lib.bundle_text("b512")}
exs = {k: cg.Extractor(v, max_batch=8) for k, v in texts.items()}
bad = 0
for c in range(cases):
    w, h = int(rng.integers(8, 1400)), int(rng.integers(8, 1000))
    mode = int(rng.integers(0, 6))
    max_side = int(rng.choice([640, 640, 480, 1024, 2048]))
    bundle = "b512" if c % 4 == 3 else "b8"
    colour = c % 5 == 4
    seed = int(rng.integers(1, 1 << 30))
    if colour:
        frames = oracle_lib.synth_rgb(seed, 2, w, h)
        got, st = exs[bundle].encode_batch(frames, mode, max_side=max_side)
        want = [oracle_lib.encode_rgb(texts[bundle], frames[i], mode, max_side=max_side) for i in range(2)]
    else:
        frames = oracle_lib.synth_frames(seed, 2, w, h)
        got, st = exs[bundle].encode_batch(frames, mode, max_side=max_side)
        want = oracle_lib.encode_batch(texts[bundle], frames, mode, max_side=max_side)
    ok = bool((st == 0).all()) and got == want
    bad += not ok
    print(c, w, h, mode, max_side, bundle, "rgb" if colour else "grey", "OK" if ok else "MISMATCH", flush=True)
print(f"{cases - bad}/{cases} configurations byte-identical")
