"""N1 measurement: SCFV posteriors on the FP64 tensor cores
(DMMA, k_posterior<true>) against the default FP64 SIMT kernel
(k_posterior<false>, the reference's separately rounded products), with the
paper's 512-component bundle on the 1024 bench frames (4K mode).

  python tools/posterior_dmma.py [out.json]          # containers + timing
  python tools/posterior_dmma.py --ncu-once dmma|simt  # one small run for ncu

Reports the aggregation-stage time of both (serial mode: kernels do not
overlap), and how many containers the DMMA rounding changes (the SIMT
containers equal the oracle's, checked on a sample here and on every frame by
tests/tools/parity_sweep.py)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle_lib  # noqa: E402  (the checker only)
import paper_1705_09776_b200 as cg  # noqa: E402

N = 1024


def run(ex, d_frames, n, dmma, steps=5):
    slot = cg.container_slot("4K")
    dout, dlen = ex.device_buffer(n * slot), ex.device_buffer(4 * n)
    ex.set_debug(False, serial=True, post_simt=not dmma)
    ex.encode_device(d_frames, n, 640, 480, "4K", dout, dlen)
    ex.sync()
    agg = 0.0
    for _ in range(steps):
        ex.encode_device(d_frames, n, 640, 480, "4K", dout, dlen)
        ex.sync()
        agg += ex.stage_times()["aggregation"]
    lens = np.frombuffer(dlen.to_host(), dtype=np.uint32)
    raw = dout.to_host()
    outs = [raw[i * slot:i * slot + int(lens[i])].tobytes() for i in range(n)]
    return outs, agg / steps


def main():
    b512 = oracle_lib.bundle_text("b512")
    if len(sys.argv) > 2 and sys.argv[1] == "--ncu-once":
        ex = cg.Extractor(b512, max_batch=64)
        d = ex.synth_frames_device(1000, 64, 640, 480)
        run(ex, d, 64, sys.argv[2] == "dmma", steps=0)
        ex.close()
        return
    ex = cg.Extractor(b512, max_batch=512)
    d = ex.synth_frames_device(1000, N, 640, 480)
    simt, t_simt = run(ex, d, N, False)
    dmma, t_dmma = run(ex, d, N, True)
    frames = np.frombuffer(d.to_host(), dtype=np.uint8).reshape(N, 480, 640)
    sample = list(range(0, N, 64))
    oracle_ok = sum(simt[i] == oracle_lib.encode(b512, frames[i], 3) for i in sample)
    diff = [i for i in range(N) if simt[i] != dmma[i]]
    # where a container differs: which section (global SCFV or local codes)
    glob = 0
    for i in diff:
        a, b = simt[i], dmma[i]
        k = next(j for j in range(min(len(a), len(b))) if a[j] != b[j]) if a[:min(len(a), len(b))] != b[:min(len(a), len(b))] else min(len(a), len(b))
        glob += 1 if k < len(a) - 4 else 0
    res = {
        "bundle": "b512 (512 components)", "mode": "4K", "frames": N,
        "aggregation_ms_per_1024_frames": {"simt_fp64": t_simt, "dmma_tensor": t_dmma},
        "containers_changed_by_dmma": len(diff), "changed_frames_first": diff[:16],
        "simt_equals_oracle_on_sample": f"{oracle_ok}/{len(sample)}",
    }
    print(json.dumps(res))
    if len(sys.argv) > 1:
        json.dump(res, open(sys.argv[1], "w"), indent=1)
    ex.close()


if __name__ == "__main__":
    main()
