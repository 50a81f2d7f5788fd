"""Stage-by-stage GPU vs oracle comparison on a few frames (diagnostic)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib  # noqa: E402
import paper_1705_09776_b200 as cg  # noqa: E402


def main(nframes=4, w=640, h=480, mode=3, bundle="b8", seed=1000):
    text = oracle_lib.bundle_text(bundle)
    frames = oracle_lib.synth_frames(seed, nframes, w, h)
    ex = cg.Extractor(text, max_batch=max(nframes, 1))
    ex.set_debug(True)
    res, status = ex.encode_batch(frames, mode)
    print("status", status.tolist(), "crc", hex(ex.model_crc), "oracle crc", hex(oracle_lib.bundle_crc(text)[0]))
    print("stage ms", ex.stage_times(), ex.kernel_stats())
    same = 0
    for f in range(nframes):
        tr = oracle_lib.Trace(text, frames[f], mode)
        ref = tr.get("container").astype(np.uint8).tobytes()
        ok = ref == res[f]
        same += ok
        line = [f"frame {f}: container {'IDENTICAL' if ok else 'DIFF'} ({len(res[f])} vs {len(ref)} B)"]
        dims = tr.get("dims")
        for o in range(int(dims[2])):
            for k in range(4):
                a, b = ex.debug_get(f"gauss:{o}:{k}", f), tr.get(f"gauss:{o}:{k}")
                if a.size != b.size or not np.array_equal(a, b):
                    line.append(f"  gauss {o}:{k} mismatch size {a.size}/{b.size} maxdiff {np.max(np.abs(a - b)) if a.size == b.size else -1}")
            a, b = ex.debug_get(f"refined:{o}", f), tr.get(f"refined:{o}")
            if not np.array_equal(a, b):
                line.append(f"  refined {o}: gpu {a.size // 8} oracle {b.size // 8} equal={np.array_equal(a, b)}")
        for name in ("keypoints", "selected", "oriented", "descriptors", "x", "gamma", "gm"):
            a, b = ex.debug_get(name, f), tr.get(name)
            if a.size != b.size:
                line.append(f"  {name}: size gpu {a.size} oracle {b.size}")
            elif not np.array_equal(a, b):
                d = np.max(np.abs(a - b))
                line.append(f"  {name}: max abs diff {d:.3e} ({np.count_nonzero(a != b)} / {a.size} differ)")
        print("\n".join(line))
    print(f"{same}/{nframes} containers identical")


if __name__ == "__main__":
    main(*[int(a) if a.isdigit() else a for a in sys.argv[1:]])
