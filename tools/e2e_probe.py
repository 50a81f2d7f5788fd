"""Where the end-to-end time goes: device-resident steps vs streamed host
steps (submit / wait wall times), and the raw H2D rate of one step's frames.
python tools/e2e_probe.py"""
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib  # noqa: E402
import paper_1705_09776_b200 as cg  # noqa: E402

W, H, N, STEPS = 640, 480, 1024, 8
ex = cg.Extractor(oracle_lib.bundle_text("b8"), max_batch=512)
d = ex.synth_frames_device(1000, N, W, H)
slot = cg.container_slot("4K")
dout, dlen = ex.device_buffer(N * slot), ex.device_buffer(4 * N)
for _ in range(3):
    ex.encode_device(d, N, W, H, "4K", dout, dlen)
ex.sync()
t = time.perf_counter()
for _ in range(STEPS):
    ex.encode_device(d, N, W, H, "4K", dout, dlen)
ex.sync()
t_dev = (time.perf_counter() - t) / STEPS
print(f"device-resident: {t_dev * 1e3:.2f} ms/step  {N / t_dev:.0f} frames/s (wall)", ex.stage_times())

host = ex.pinned_buffer(N * W * H)
host.array[:] = d.to_host(N * W * H)
dd = ex.device_buffer(N * W * H)
lib = ex._lib
ex._check(lib.cdvz_gpu_copy(ex._ctx, dd.ptr, host.ptr, N * W * H, 1))
ex.sync()
t = time.perf_counter()
for _ in range(4):
    ex._check(lib.cdvz_gpu_copy(ex._ctx, dd.ptr, host.ptr, N * W * H, 1))
ex.sync()
t_h2d = (time.perf_counter() - t) / 4
print(f"H2D of one step ({N * W * H / 1e6:.0f} MB): {t_h2d * 1e3:.2f} ms  {N * W * H / t_h2d / 1e9:.1f} GB/s")

frames = host.array.reshape(N, H, W)
outs = [ex.pinned_buffer(N * slot) for _ in range(2)]
offs = [np.zeros(N + 1, dtype=np.uint64) for _ in range(2)]
sts = [np.zeros(N, dtype=np.int32) for _ in range(2)]


def submit(k):
    tk = ctypes.c_uint64()
    ex._check(lib.cdvz_gpu_encode_batch_submit(ex._ctx, frames.ctypes.data, W, H, W, N, 3, 640, outs[k].ptr, N * slot,
                                               offs[k].ctypes.data, sts[k].ctypes.data, ctypes.byref(tk)))
    return tk.value


def wait(tk):
    ex._check(lib.cdvz_gpu_encode_batch_wait(ex._ctx, tk))


for mode in ("sync", "stream"):
    wait(submit(0))
    ts, tw = [], []
    t = time.perf_counter()
    pend, k = None, 0
    for _ in range(STEPS):
        a = time.perf_counter()
        tk = submit(k)
        b = time.perf_counter()
        if mode == "sync":
            wait(tk)
        elif pend is not None:
            wait(pend)
        c = time.perf_counter()
        ts.append(b - a)
        tw.append(c - b)
        if mode == "stream":
            pend, k = tk, k ^ 1
    if mode == "stream":
        wait(pend)
    tot = (time.perf_counter() - t) / STEPS
    print(f"{mode}: {tot * 1e3:.2f} ms/step {N / tot:.0f} frames/s; submit ms {np.round(np.array(ts) * 1e3, 2).tolist()}"
          f" wait ms {np.round(np.array(tw) * 1e3, 2).tolist()}", ex.stage_times())
ex.close()
