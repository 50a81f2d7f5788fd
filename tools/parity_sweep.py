"""Large-scale parity evidence: the bench workload and other configurations
encoded on the GPU, by the CPU oracle and by the REFERENCE ITSELF (oracle/_ref,
its sources built against the Eigen-subset), both frame-parallel on the host
cores; counts byte-identical containers against each.
python tools/parity_sweep.py [out.json]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib  # noqa: E402
import ref_lib  # noqa: E402
import paper_1705_09776_b200 as cg  # noqa: E402


def sweep(name, bundle, frames, mode, max_side=640):
    text = oracle_lib.bundle_text(bundle)
    ex = cg.Extractor(text, max_batch=512)
    got, status = ex.encode_batch(frames, mode, max_side=max_side)
    ex.close()
    t = time.time()
    want = oracle_lib.encode_batch(text, frames, cg.mode_by_name(mode).id if isinstance(mode, str) else mode,
                                   max_side=max_side, threads=os.cpu_count() or 8)
    same = sum(int(a == b) for a, b in zip(got, want))
    oracle_s = round(time.time() - t, 1)
    t = time.time()
    mid = cg.mode_by_name(mode).id if isinstance(mode, str) else mode
    ref = ref_lib.encode_batch(text, frames, mid, threads=os.cpu_count() or 8, workers=1, max_side=max_side)
    same_ref = sum(int(a == b) for a, b in zip(got, ref))
    row = {"case": name, "bundle": bundle, "mode": mode, "frames": len(frames), "size": list(frames.shape[1:3][::-1]),
           "gpu_ok": int((status == 0).sum()), "byte_identical": same, "byte_identical_vs_reference": same_ref,
           "oracle_s": oracle_s, "reference_s": round(time.time() - t, 1)}
    print(json.dumps(row), flush=True)
    return row


def main(out):
    rows = []
    vga = oracle_lib.synth_frames(1000, 1024, 640, 480)  # the bench frames (BASELINE configs[1], base seed 1000)
    rows.append(sweep("configs[1]: 1024 VGA frames, 4K", "b8", vga, "4K"))
    rows.append(sweep("configs[1] with the 512-component bundle (DMMA posteriors)", "b512", vga, "4K"))
    rows.append(sweep("512-component bundle, 16K (variance planes)", "b512", vga[:256], "16K"))
    rows.append(sweep("512B mode, VGA", "b8", vga[256:448], "512B"))
    rows.append(sweep("8K mode (variance planes)", "b8", vga[448:576], "8K"))
    hd = oracle_lib.synth_frames(4000, 64, 1920, 1080)
    rows.append(sweep("configs[2]: 1080p -> 640x360, 16K", "b8", hd, "16K"))
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)
    total = sum(r["frames"] for r in rows)
    same = sum(r["byte_identical"] for r in rows)
    same_ref = sum(r["byte_identical_vs_reference"] for r in rows)
    print(f"{same}/{total} containers byte-identical to the oracle, {same_ref}/{total} to the reference")


def main_extended(out):
    """Unseen content: 8192 more VGA frames (other seeds) in 4K and 16K with the
    8-component bundle and 2048 with the 512-component one, 1024 at 1280x720
    resized, against the oracle and the reference."""
    rows = []
    for k, (seed, mode) in enumerate([(200000, "4K"), (300000, "16K"), (400000, "1K"), (500000, "2K")]):
        for part in range(2):
            vga = oracle_lib.synth_frames(seed + 1024 * part, 1024, 640, 480)
            rows.append(sweep(f"VGA seeds {seed + 1024 * part}+, {mode}", "b8", vga, mode))
    for part in range(2):
        vga = oracle_lib.synth_frames(600000 + 1024 * part, 1024, 640, 480)
        rows.append(sweep(f"VGA seeds {600000 + 1024 * part}+, 4K, 512 components", "b512", vga, "4K"))
    hd = oracle_lib.synth_frames(700000, 1024, 1280, 720)
    rows.append(sweep("1280x720 -> 640x360, 8K", "b8", hd, "8K"))
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)
    total = sum(r["frames"] for r in rows)
    same = sum(r["byte_identical"] for r in rows)
    same_ref = sum(r["byte_identical_vs_reference"] for r in rows)
    print(f"{same}/{total} containers byte-identical to the oracle, {same_ref}/{total} to the reference")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "extended":
        main_extended(sys.argv[1])
        sys.exit(0)
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_sweep.json")
