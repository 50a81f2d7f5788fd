import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, oracle_lib, paper_1705_09776_b200 as cg
b = oracle_lib.bundle_text("b8")
ex = cg.Extractor(b, max_batch=8)
for (w, h) in [(3840, 2160), (1920, 1080)]:
    fr = ex.synth_frames(11, 2, w, h)
    got, st = ex.encode_batch(fr, "16K", max_side=4096)
    print(w, h, st.tolist(), [len(g) for g in got])
    ex.set_debug(True)
    got, st = ex.encode_batch(fr[:1], "16K", max_side=4096)
    n = [ex.debug_get(f"refined:{o}", 0).size // 8 for o in range(4)]
    print("refined per octave", n)
    ex.set_debug(False)
if len(sys.argv) > 1 and sys.argv[1] == "oracle":
    import time
    fr = ex.synth_frames(11, 1, 3840, 2160)
    got, st = ex.encode_batch(fr, "16K", max_side=4096)
    t = time.time()
    want = oracle_lib.encode(b, fr[0], 5, max_side=4096)
    print("4K native vs oracle:", got[0] == want, len(got[0]), len(want), f"oracle {time.time() - t:.1f} s")
