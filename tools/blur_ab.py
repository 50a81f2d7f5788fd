import sys, os, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle_lib
import paper_1705_09776_b200 as cg
b8 = oracle_lib.bundle_text("b8")
frames = oracle_lib.synth_frames(900, 16, 640, 480)
outs = {}
for unrolled in (False, True):
    ex = cg.Extractor(b8, max_batch=16)
    ex.set_debug(False, blur_unrolled=unrolled)
    outs[unrolled] = ex.encode_batch(frames, "4K")[0]
    ex.close()
assert outs[False] == outs[True], "blur variants differ"
for i in range(4):
    assert outs[False][i] == oracle_lib.encode(b8, frames[i], 3)
print("blur variants identical")
# timing: pyramid_bench-like via bench-style device run
d = None
for unrolled in (False, True):
    ex = cg.Extractor(b8, max_batch=512)
    ex.set_debug(False, serial=True, blur_unrolled=unrolled)
    dfr = ex.synth_frames_device(1000, 1024, 640, 480)
    slot = cg.container_slot("4K")
    dout = ex.device_buffer(1024 * slot); dlen = ex.device_buffer(4 * 1024)
    for it in range(3):
        ex.encode_device(dfr, 1024, 640, 480, "4K", dout, dlen)
    ex.sync()
    ex.event_record(0)
    for it in range(5):
        ex.encode_device(dfr, 1024, 640, 480, "4K", dout, dlen)
    ex.event_record(1); ex.sync()
    st = ex.stage_times()
    print("unrolled" if unrolled else "rolled", "ms/step", ex.event_elapsed(0, 1) / 5, "stages(last call)", st, "kstats", ex.kernel_stats())
    ex.close()
