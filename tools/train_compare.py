"""GPU train_model vs the reference's (the committed bundles are its output,
tests/golden/make_bundles.py): per-section identity / max relative difference
and wall times.  python tools/train_compare.py [out.json]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib  # noqa: E402  (checker only)
import paper_1705_09776_b200 as cg  # noqa: E402
from test_gpu_train import numbers, sections  # noqa: E402

GOLDEN = 0x9E3779B97F4A7C15
rows = []
corpus = np.stack([oracle_lib.synth_f64((401 + i * GOLDEN) % (1 << 64), 256, 256) for i in range(20)])
for name, gmm in (("b8", 8), ("b512", 512)):
    want = oracle_lib.bundle_text(name)
    t = time.perf_counter()
    got = cg.train_model(corpus, seed=11, gmm_components=gmm, em_iterations=15)
    gpu_s = time.perf_counter() - t
    row = {"bundle": name, "gmm_components": gmm, "gpu_train_s": round(gpu_s, 3), "identical_text": got == want}
    sg, sw = sections(got), sections(want)
    for sec in sw:
        if sg[sec] == sw[sec]:
            row[sec] = "identical"
        else:
            a, b = numbers(sg[sec]), numbers(sw[sec])
            rel = float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.shape == b.shape else None
            row[sec] = {"max_rel_diff": rel, "identical_lines": int(sum(x == y for x, y in zip(sg[sec], sw[sec]))),
                        "lines": len(sw[sec])}
    try:
        import ref_lib
        if ref_lib.available():
            t = time.perf_counter()
            ref = ref_lib.train_bundle(401, 20, 256, 256, 11, gmm, 15, workers=os.cpu_count() or 8)
            row["reference_train_s"] = round(time.perf_counter() - t, 3)
            row["reference_cores"] = os.cpu_count()
            row["reference_equals_committed"] = ref == want
    except Exception as e:  # noqa: BLE001
        row["reference_error"] = str(e)
    print(json.dumps(row), flush=True)
    rows.append(row)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
