"""One-off validation that the extrema pre-screen is conservative: per-octave
survivor lists and containers with the screen equal those of the exact test
on every pixel, over many frames and sizes.  python tools/probe_screen.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle_lib  # noqa: E402
import paper_1705_09776_b200 as cg  # noqa: E402

b = oracle_lib.bundle_text("b8")
rng = np.random.default_rng(7)
sizes = [(640, 480)] * 4 + [(1920, 1080), (1280, 720), (333, 257), (800, 600), (3840, 2160)]
total = 0
for k, (w, h) in enumerate(sizes):
    n = 2 if w * h > 2e6 else 24
    a = cg.Extractor(b, max_batch=n)
    x = cg.Extractor(b, max_batch=n)
    a.set_debug(True)
    x.set_debug(True, exact_only=True)
    frames = a.synth_frames(int(rng.integers(1, 1 << 30)), n, w, h)
    ca, _ = a.encode_batch(frames, "16K", max_side=4096)
    cx, _ = x.encode_batch(frames, "16K", max_side=4096)
    assert ca == cx, (w, h)
    for f in range(n):
        for o in range(4):
            assert np.array_equal(a.debug_get(f"refined:{o}", f), x.debug_get(f"refined:{o}", f)), (w, h, f, o)
    total += n
    a.close()
    x.close()
    print(f"{w}x{h}: {n} frames identical", flush=True)
print(f"screen conservative on {total} frames")
