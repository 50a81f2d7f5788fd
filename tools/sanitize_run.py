"""Small workload for compute-sanitizer (tests/test_gpu_sanitizer.py): every
kernel of the product path on a handful of frames, no torch.

  python tools/sanitize_run.py [all|encode|match]

* encode: 2 frames of 320x240 (SAN_W / SAN_H / SAN_N override) in 4K mode (u8 path: k_blur<.., 0>, k_detect_walk,
  merge, select, orient, expand, geometry, sample, describe, PCA,
  posterior-small, Fisher, SCFV, pack), the same frames with the 512-component
  bundle (k_posterior on the FP64 tensor cores), one f64 frame at three times the size (resized) (k_validate, f64 k_resize,
  k_blur<.., 1>), one odd-width RGB frame (k_grey_rgb, unaligned u8 rows),
  on-device synthesis, streamed submit / wait batches (one context and a
  two-shard multi-device context), an f64 frame with -0.0 pixels, a
  selection budget above the rank-sort limit, the register-bin describe
  variant, and the debug paths (exact-only extrema, the TMA tile kernel and its plain-load
  variant, tiny capacities -> the capacity retry);
* match: an 8-container index, retrieve + match_pairs (k_match.cu);
* train: cdvz_gpu_train_model on a 20-image corpus (train.cu).
Exit 0 when every container equals the oracle's (sanity: the sanitizer run
must not change results).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib  # noqa: E402  (the checker only)
import paper_1705_09776_b200 as cg  # noqa: E402


def encode_part():
    b8, b512 = oracle_lib.bundle_text("b8"), oracle_lib.bundle_text("b512")
    w, h, n = int(os.environ.get("SAN_W", 320)), int(os.environ.get("SAN_H", 240)), int(os.environ.get("SAN_N", 2))
    frames = np.stack([oracle_lib.synth_u8(1000 + i, w, h) for i in range(n)])
    ex = cg.Extractor(b8, max_batch=4)
    got, st = ex.encode_batch(frames, "4K")
    assert st.tolist() == [0] * n
    for i in range(n):
        assert got[i] == oracle_lib.encode(b8, frames[i], 3), f"u8 frame {i}"
    f64 = oracle_lib.synth_f64(77, 3 * w, 3 * h)[None]
    got, st = ex.encode_batch(f64, "8K")
    assert st.tolist() == [0] and got[0] == oracle_lib.encode_f64(b8, f64[0], 4)[0]
    rgb = np.random.default_rng(5).integers(0, 256, (1, 121, 163, 3), dtype=np.uint8)
    got, st = ex.encode_batch(rgb, "512B")
    assert st.tolist() == [0]
    d = ex.synth_frames_device(1000, 2, 320, 240)
    d.free()
    want0 = oracle_lib.encode(b8, frames[0], 3)
    for flags in (dict(exact_only=True), dict(tile_detect=True), dict(tile_detect=True, no_tma=True),
                  dict(tiny_caps=True)):
        ex.set_debug(True, **flags)
        got, st = ex.encode_batch(frames[:1], "4K")
        assert got[0] == want0, flags
    ex.set_debug(False)
    # streamed submit / wait (two batches in flight) and the describe variant with register bins
    p0 = ex.encode_batch_submit(frames, "4K")
    p1 = ex.encode_batch_submit(frames[:1], "8K")
    assert p0.wait()[0][0] == want0 and p1.wait()[1].tolist() == [0]
    ex.set_debug(False, desc_registers=True)
    got, st = ex.encode_batch(frames[:1], "4K")
    assert got[0] == want0
    ex.set_debug(False)
    # an f64 frame with a -0.0 band (the f64-base blur's zero canonicalisation)
    negz = oracle_lib.synth_f64(78, w, h)
    negz[:, w // 3:w // 2] = -0.0
    got, st = ex.encode_batch(negz[None], "4K")
    assert st.tolist() == [0] and got[0] == oracle_lib.encode_f64(b8, negz, 3)[0]
    ex.close()
    # a multi-device context (two shards on one GPU), streamed
    mx = cg.Extractor(b8, max_batch=4, devices=[0, 0])
    q0 = mx.encode_batch_submit(frames, "4K")
    q1 = mx.encode_batch_submit(frames, "4K")
    assert q0.wait()[0][0] == want0 and q1.wait()[0][0] == want0
    mx.close()
    # a selection budget above the rank-sort limit (k_select's bitonic network)
    import zlib
    lines = b8.split("\n")
    k = lines.index(next(ln for ln in lines if ln.startswith("section selector")))
    _, name, nl, _ = lines[k].split()
    body = lines[k + 1:k + 1 + int(nl)]
    body[0] = "n = 3000"
    lines[k] = f"section {name} {nl} %08x" % zlib.crc32(("\n".join(body) + "\n").encode())
    lines[k + 1:k + 1 + int(nl)] = body
    big = "\n".join(lines)
    bx = cg.Extractor(big, max_batch=4)
    got, st = bx.encode_batch(frames[:1], "4K")
    assert st.tolist() == [0] and got[0] == oracle_lib.encode(big, frames[0], 3)
    bx.close()
    ex = cg.Extractor(b512, max_batch=4)
    got, st = ex.encode_batch(frames[:2], "4K")
    for i in range(2):
        assert got[i] == oracle_lib.encode(b512, frames[i], 3), f"b512 frame {i}"
    ex.set_debug(False, post_simt=True)  # the SIMT posterior kernel too
    got2, st = ex.encode_batch(frames[:2], "4K")
    assert got2 == got
    ex.close()


def match_part():
    b8 = oracle_lib.bundle_text("b8")
    frames = np.stack([oracle_lib.synth_u8(2000 + i, 160, 120) for i in range(8)])
    ex = cg.Extractor(b8, max_batch=8)
    conts, st = ex.encode_batch(frames, "4K")
    ex.close()
    idx = cg.Index(conts)
    items, _ = idx.retrieve_batch(conts[:3])
    assert items[:, 0].tolist() == [0, 1, 2], "self retrieval"
    idx.match_pairs(conts[:2], [(0, 1), (1, 0)])
    idx.close()


def train_part():
    """cdvz_gpu_train_model on a 20-image corpus (the training kernels)."""
    golden = 0x9E3779B97F4A7C15
    corpus = np.stack([oracle_lib.synth_f64((401 + i * golden) % (1 << 64), 256, 256) for i in range(20)])
    text = cg.train_model(corpus, seed=11, gmm_components=8, em_iterations=3)
    cg.bundle_check(text)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "encode"):
        encode_part()
    if what in ("all", "match"):
        match_part()
    if what in ("all", "train"):
        train_part()
    print("sanitize_run ok")
