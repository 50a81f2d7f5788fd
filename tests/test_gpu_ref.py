"""GPU containers against the REFERENCE ITSELF (oracle/_ref/libref.so: the
reference's proj/src built against the Eigen-subset, tests/ref_lib.py), not
only against the oracle restatement: the bench frames, other modes, the
512-component bundle, 1080p -> 640x360 and f64 GrayImage input."""
import os

import numpy as np
import pytest

import oracle_lib
import ref_lib

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(ref_lib.LIB), reason="oracle/_ref/libref.so not built")]

cg = pytest.importorskip("paper_1705_09776_b200")
THREADS = os.cpu_count() or 8


def test_bench_frames_equal_the_reference(bundle_b8):
    frames = oracle_lib.synth_frames(1000, 64, 640, 480, threads=THREADS)  # the first bench frames
    ex = cg.Extractor(bundle_b8, max_batch=64)
    got, status = ex.encode_batch(frames, "4K")
    ex.close()
    assert (status == 0).all()
    want = ref_lib.encode_batch(bundle_b8, frames, 3, threads=THREADS, workers=1)
    assert sum(a == b for a, b in zip(got, want)) == len(frames)


@pytest.mark.parametrize("bundle,mode,size", [("b8", "512B", (640, 480)), ("b8", "8K", (640, 480)),
                                              ("b512", "4K", (640, 480)), ("b8", "16K", (1920, 1080))])
def test_modes_bundles_sizes_equal_the_reference(bundle, mode, size):
    text = oracle_lib.bundle_text(bundle)
    frames = oracle_lib.synth_frames(7100, 8, size[0], size[1], threads=THREADS)
    ex = cg.Extractor(text, max_batch=8)
    got, status = ex.encode_batch(frames, mode)
    ex.close()
    assert (status == 0).all()
    want = ref_lib.encode_batch(text, frames, cg.mode_by_name(mode).id, threads=THREADS, workers=1)
    assert got == want


def test_f64_grayimage_equals_the_reference(bundle_b8):
    imgs = np.stack([ref_lib.synth_f64(8100 + i, 640, 480) for i in range(3)])
    ex = cg.Extractor(bundle_b8, max_batch=4)
    got, status = ex.encode_batch(imgs, "4K")
    ex.close()
    assert (status == 0).all()
    for i in range(3):
        assert got[i] == ref_lib.encode_f64(bundle_b8, imgs[i], 3)[0]
