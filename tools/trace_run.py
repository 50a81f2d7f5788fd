import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle_lib
import paper_1705_09776_b200 as cg
W, H, N = 640, 480, 1024
mode = sys.argv[1]
ex = cg.Extractor(oracle_lib.bundle_text("b8"), max_batch=512)
d = ex.synth_frames_device(1000, N, W, H)
slot = cg.container_slot("4K")
lib = ex._lib
if mode == "device":
    dout, dlen = ex.device_buffer(N * slot), ex.device_buffer(4 * N)
    for _ in range(4):
        ex.encode_device(d, N, W, H, "4K", dout, dlen)
    ex.sync(); ex.stage_times()
else:
    host = ex.pinned_buffer(N * W * H); host.array[:] = d.to_host(N * W * H)
    frames = host.array.reshape(N, H, W)
    outs = [ex.pinned_buffer(N * slot) for _ in range(2)]
    offs = [np.zeros(N + 1, dtype=np.uint64) for _ in range(2)]
    sts = [np.zeros(N, dtype=np.int32) for _ in range(2)]
    def submit(k):
        tk = ctypes.c_uint64()
        ex._check(lib.cdvz_gpu_encode_batch_submit(ex._ctx, frames.ctypes.data, W, H, W, N, 3, 640, outs[k].ptr, N * slot, offs[k].ctypes.data, sts[k].ctypes.data, ctypes.byref(tk)))
        return tk.value
    pend, k = None, 0
    for _ in range(4):
        tk = submit(k)
        if mode == "sync": ex._check(lib.cdvz_gpu_encode_batch_wait(ex._ctx, tk))
        else:
            if pend: ex._check(lib.cdvz_gpu_encode_batch_wait(ex._ctx, pend))
            pend, k = tk, k ^ 1
    if pend: ex._check(lib.cdvz_gpu_encode_batch_wait(ex._ctx, pend))
    ex.stage_times()
ex.close()
