"""GPU tests of the drop-in boundary beyond the 8-bit batch path:

* the reference's own input type — an f64 GrayImage (image.hpp:11-18) straight
  from synth_image, no 8-bit quantisation — through cdvz_gpu_encode_batch_f64,
  with validate() (image.cpp:46-51) per frame;
* the EncodedImage struct out (container.hpp:19-25) through the C++ shim's
  reference-signature encode_image, incl. SCFVDescriptor::norms;
* the multi-device context (cdvz_gpu_create_multi): frame-sharded host batches
  gathered in frame order, byte-identical to one context;
* the capacity retry of the host path (frames whose lists overflow are
  re-encoded with the maximal capacities) and adversarial frames.

Every container is compared with the CPU oracle's.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle_lib

pytestmark = pytest.mark.gpu

cg = pytest.importorskip("paper_1705_09776_b200")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ex(bundle_b8):
    e = cg.Extractor(bundle_b8, max_batch=16)
    yield e
    e.close()


def test_f64_grayimage_matches_oracle(ex, bundle_b8):
    """Unquantised synth_image doubles: containers and SCFV norms equal the
    oracle's, at the prepared size and through resize_max_side (960x720)."""
    for (w, h, mode) in [(640, 480, 3), (960, 720, 5), (320, 240, 0)]:
        frames = np.stack([oracle_lib.synth_f64(3000 + 7 * i + w, w, h) for i in range(3)])
        got, status = ex.encode_batch(frames, mode)
        assert status.tolist() == [0, 0, 0]
        for i in range(3):
            want, norms = oracle_lib.encode_f64(bundle_b8, frames[i], mode)
            assert got[i] == want, f"{w}x{h} frame {i}"
        # norms of the last frame of the batch (debug arrays hold the last chunk);
        # libdevice exp (the softmax) vs glibc moves the last ulps of gm only.
        ex.encode_batch(frames[2:3], mode)
        got_n, want_n = ex.debug_get("norms", 0), oracle_lib.encode_f64(bundle_b8, frames[2], mode)[1]
        assert got_n.shape == want_n.shape and np.allclose(got_n, want_n, rtol=1e-12, atol=0)


def test_f64_negative_zero_pixels_match_oracle(ex, bundle_b8):
    """-0.0 passes validate() (-0.0 >= 0.0). The reference's blur sums start
    from 0.0, so its pyramid never holds -0.0; the GPU's f64-base blur maps an
    all -0.0 sum to +0.0 the same way, so zero signs downstream (the bilinear
    taps, atan2's +-pi) match. Bands and a +-0 checkerboard next to textured
    regions, in a batch with an ordinary frame, against the oracle; and the
    pyramid levels of a -0.0 frame hold no -0.0."""
    frames = np.stack([oracle_lib.synth_f64(5200 + i, 320, 240) for i in range(3)])
    frames[0, :, 100:160] = -0.0
    frames[0, 60:120, :] = 0.0
    frames[1, 40:200, 40:200] = np.where((np.indices((160, 160)).sum(0) % 2) == 0, -0.0, 0.0)
    frames[1, 90:110, :] = -0.0
    assert np.signbit(frames[0]).any() and np.signbit(frames[1]).any() and not np.signbit(frames[2]).any()
    for mode in (3, 5):
        got, status = ex.encode_batch(frames, mode)
        assert status.tolist() == [0, 0, 0]
        for i in range(3):
            assert got[i] == oracle_lib.encode_f64(bundle_b8, frames[i], mode)[0], f"mode {mode} frame {i}"
    ex.encode_batch(frames[0:1], 3)
    for lvl in range(4):
        g = ex.debug_get(f"gauss:0:{lvl}", 0)
        assert g.size > 0 and (g == 0.0).any() and not (np.signbit(g) & (g == 0.0)).any(), lvl


def test_f64_validate_per_frame(ex, bundle_b8):
    """validate(): a NaN, an inf or a value outside [0, 1] fails that frame
    alone with a DataError status; the neighbours are unaffected."""
    base = np.stack([oracle_lib.synth_f64(4100 + i, 320, 240) for i in range(5)])
    bad = base.copy()
    bad[1, 10, 10] = np.nan
    bad[2, 0, 0] = 1.0000000000000002
    bad[3, 239, 319] = -np.inf
    got, status = ex.encode_batch(bad, "2K")
    assert status.tolist() == [0, 2, 2, 2, 0]
    assert got[1] == got[2] == got[3] == b""
    assert got[0] == oracle_lib.encode_f64(bundle_b8, base[0], 2)[0]
    assert got[4] == oracle_lib.encode_f64(bundle_b8, base[4], 2)[0]
    with pytest.raises(cg.DataError, match="finite and in"):
        ex.encode_image(bad[1], "2K")


def test_multi_device_context_is_byte_identical(bundle_b8):
    """cdvz_gpu_create_multi over [0, 0, 0] (three contexts on this GPU, one
    host thread each): 37 distinct frames (uneven shards) in u8 and f64 give the
    single-device containers in frame order."""
    frames = oracle_lib.synth_frames(5000, 37, 320, 240)
    single = cg.Extractor(bundle_b8, max_batch=16)
    multi = cg.Extractor(bundle_b8, max_batch=8, devices=[0, 0, 0])
    assert multi.devices == [0, 0, 0] and single.devices == [0]
    a, sa = single.encode_batch(frames, "4K")
    b, sb = multi.encode_batch(frames, "4K")
    assert sa.tolist() == sb.tolist() == [0] * 37
    assert a == b
    assert a[5] == oracle_lib.encode(bundle_b8, frames[5], 3)
    f64 = frames[:7].astype(np.float64) * (1.0 / 255.0)  # load_image reads a PGM byte as b * (1/255)
    c, sc = multi.encode_batch(f64, "4K")
    assert sc.tolist() == [0] * 7 and c == a[:7]
    st = multi.stage_times()
    assert st["detection"] > 0 and st["description"] > 0
    with pytest.raises(cg.UsageError):
        multi.device_buffer(16)
    multi.close()
    single.close()


def test_capacity_retry_reencodes_overflowing_frames(bundle_b8):
    """With tiny list capacities every frame overflows; the host path re-encodes
    each on its own with the maximal capacities and splices it in frame order,
    so the containers still equal the oracle's."""
    frames = oracle_lib.synth_frames(6000, 6, 320, 240)
    e = cg.Extractor(bundle_b8, max_batch=4)
    e.set_debug(False, tiny_caps=True)
    got, status = e.encode_batch(frames, "4K")
    assert status.tolist() == [0] * 6
    for i in range(6):
        assert got[i] == oracle_lib.encode(bundle_b8, frames[i], 3), f"frame {i}"
    e.close()


def test_adversarial_frames_match_oracle(ex, bundle_b8):
    """White noise, a dense sine grid (14k octave-0 keypoints, ~4 orientations
    per selected point), a flat plateau and a checkerboard: no status failures
    and the oracle's containers (capacity retries included)."""
    rng = np.random.default_rng(5)
    yy, xx = np.mgrid[0:480, 0:640].astype(float)
    frames = np.stack([
        rng.integers(0, 256, (480, 640), dtype=np.uint8),
        np.clip(np.round(127.5 + 127.5 * np.sin(xx * 0.7 + 0.3) * np.sin(yy * 0.7 + 0.7)), 0, 255).astype(np.uint8),
        np.full((480, 640), 128, dtype=np.uint8),
        ((((yy // 3) % 2).astype(int) ^ ((xx // 3) % 2).astype(int)) * 255).astype(np.uint8),
    ])
    got, status = ex.encode_batch(frames, "4K")
    assert status.tolist() == [0, 0, 0, 0]
    for i in range(len(frames)):
        assert got[i] == oracle_lib.encode(bundle_b8, frames[i], 3), f"frame {i}"


def test_cpp_reference_signature_struct_out(tmp_path, bundle_b8):
    """examples/encode_gray.cpp: cdvz::gpu::encode_image(GrayImage, ModelBundle,
    ModeSpec, Engine, StageTimings*, EncodeOptions) -> EncodedImage, then
    serialize_container: bytes equal the oracle's, the struct's fields equal
    the container's decode, norms equal the oracle's; the multi-device batch
    through the shim is byte-identical to one device."""
    lib_dir = os.path.join(ROOT, "paper_1705_09776_b200")
    exe = str(tmp_path / "encode_gray")
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "examples", "encode_gray.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    bundle = tmp_path / "bundle.txt"
    bundle.write_text(bundle_b8)
    img = oracle_lib.synth_f64(4242, 640, 480)
    raw = tmp_path / "in.f64"
    raw.write_bytes(img.tobytes())
    out, txt = tmp_path / "out.cdvz", tmp_path / "out.txt"
    r = subprocess.run([exe, str(bundle), "8K", "640", "480", str(raw), str(out), str(txt), "0,0"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    want, norms = oracle_lib.encode_f64(bundle_b8, img, 4)
    assert out.read_bytes() == want
    fields = {}
    codes = []
    for line in txt.read_text().splitlines():
        parts = line.split()
        if parts and parts[0] in ("mode", "size", "model_crc", "components", "mask", "mean", "var", "norms", "codes"):
            fields[parts[0]] = parts[1:]
        elif parts and parts[0] != "stage":
            codes.append([int(v) for v in parts])
    hdr = cg.parse_container_header(want)
    assert int(fields["mode"][0]) == 4 and [int(v) for v in fields["size"]] == [640, 480]
    assert int(fields["model_crc"][0]) == hdr["model_crc"]
    got_norms = np.array([float(v) for v in fields["norms"]])
    assert got_norms.shape == norms.shape and np.allclose(got_norms, norms, rtol=1e-12, atol=0)
    assert len(codes) == int(fields["codes"][0]) > 0
    assert all(len(c) == 5 + 103 and c[4] == 4 for c in codes)
    assert "stage detection" in txt.read_text()


def test_multi_device_submit_wait_streams_batches(bundle_b8):
    """A multi-device context (two shards here, on one GPU) streams batches
    too: submit enqueues every shard's share and returns, wait gathers in
    frame order; a third submit completes the oldest; results equal a
    single-device context's and the oracle's."""
    single = cg.Extractor(bundle_b8, max_batch=16)
    multi = cg.Extractor(bundle_b8, max_batch=16, devices=[0, 0])
    batches = [oracle_lib.synth_frames(6000 + 100 * k, 7, 320, 240) for k in range(3)]
    pend = [multi.encode_batch_submit(b, "4K") for b in batches]
    assert all(p.ticket != 0 for p in pend)
    got = {2: pend[2].wait(), 0: pend[0].wait(), 1: pend[1].wait()}
    for k, b in enumerate(batches):
        want, st = single.encode_batch(b, "4K")
        assert got[k][0] == want and got[k][1].tolist() == [0] * 7
    assert got[0][0][0] == oracle_lib.encode(bundle_b8, batches[0][0], 3)
    with pytest.raises(cg.UsageError):
        multi._check(multi._lib.cdvz_gpu_encode_batch_wait(multi._ctx, pend[1].ticket))
    multi.close()
    single.close()


def test_submit_wait_streams_batches(bundle_b8):
    """cdvz_gpu_encode_batch_submit / _wait: three batches submitted before
    any wait (the third submit completes the first), waited out of order —
    every batch's containers equal encode_batch's and the oracle's."""
    ex = cg.Extractor(bundle_b8, max_batch=16)
    batches = [oracle_lib.synth_frames(5000 + 100 * k, 6, 320, 240) for k in range(3)]
    pend = [ex.encode_batch_submit(b, "4K") for b in batches]
    got = [pend[2].wait(), pend[0].wait(), pend[1].wait()]
    got = [got[1], got[2], got[0]]
    for k, b in enumerate(batches):
        want, st = ex.encode_batch(b, "4K")
        assert got[k][0] == want and got[k][1].tolist() == [0] * 6
        assert want[0] == oracle_lib.encode(bundle_b8, b[0], 3)
    with pytest.raises(cg.UsageError):
        pend[0].ex._check(pend[0].ex._lib.cdvz_gpu_encode_batch_wait(ex._ctx, pend[0].ticket))
    ex.close()


def test_cpp_stream_example_matches_encode_batch(bundle_b8, tmp_path):
    """examples/stream.cpp streams a raw frame file through the shim's
    submit_batch / PendingBatch::wait (batch k + 1 submitted before batch k
    is waited for); its containers equal encode_batch's."""
    import os
    import struct
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    frames = oracle_lib.synth_frames(4200, 10, 320, 240)
    (tmp_path / "frames.u8").write_bytes(frames.tobytes())
    (tmp_path / "bundle.txt").write_text(bundle_b8)
    exe = tmp_path / "stream"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(root, "examples", "stream.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = tmp_path / "out.bin"
    p = subprocess.run([str(exe), str(tmp_path / "bundle.txt"), "4K", "320", "240", str(tmp_path / "frames.u8"), "4",
                        str(out)], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    blob, got = out.read_bytes(), []
    while blob:
        (n,) = struct.unpack("<I", blob[:4])
        got.append(blob[4:4 + n])
        blob = blob[4 + n:]
    ex = cg.Extractor(bundle_b8, max_batch=16)
    want, st = ex.encode_batch(frames, "4K")
    ex.close()
    assert got == want
