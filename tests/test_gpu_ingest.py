"""GPU PPM ingest: cdvz_gpu_encode_batch_rgb (grey conversion on the device,
then resize_max_side on the grey plane) byte-identical to the oracle's
encode_image(load_image(P6)) (proj/src/image.cpp:53-92, pipeline.cpp:54-97)."""
import numpy as np
import pytest

import oracle_lib
import paper_1705_09776_b200 as cg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex(bundle_b8):
    e = cg.Extractor(bundle_b8, max_batch=4)
    yield e
    e.close()


@pytest.mark.parametrize("w,h,mode", [(640, 480, 3), (333, 257, 1), (1280, 720, 5)])
def test_rgb_containers_match_oracle(ex, bundle_b8, w, h, mode):
    frames = oracle_lib.synth_rgb(900 + w, 3, w, h)
    got, status = ex.encode_batch(frames, mode)
    assert (status == 0).all()
    for i in range(3):
        assert got[i] == oracle_lib.encode_rgb(bundle_b8, frames[i], mode), (w, h, i)


def test_grey_rgb_keeps_the_ppm_arithmetic(ex):
    """r = g = b = v: load_image's P6 grey ((0.299 v + 0.587 v) + 0.114 v) / 255
    is not always v / 255 bit for bit, so the RGB path must not shortcut to
    the PGM path; the containers follow the P6 arithmetic."""
    g = oracle_lib.synth_frames(31, 2, 320, 240)
    rgb = np.repeat(g[..., None], 3, axis=-1)
    v = np.arange(256, dtype=np.float64)
    assert not np.array_equal(((0.299 * v + 0.587 * v) + 0.114 * v) * (1.0 / 255.0), v * (1.0 / 255.0))
    got, status = ex.encode_batch(rgb, "4K")
    assert (status == 0).all()
    assert got[0] == oracle_lib.encode_rgb(oracle_lib.bundle_text("b8"), rgb[0], 3)


def test_encode_pnm_files(ex, bundle_b8):
    grey = oracle_lib.synth_frames(77, 1, 160, 120)[0]
    pgm = b"P5\n# synthetic\n160 120\n255\n" + grey.tobytes()
    assert ex.encode_pnm(pgm, "2K") == oracle_lib.encode(bundle_b8, grey, 2)
    rgb = oracle_lib.synth_rgb(78, 1, 160, 120)[0]
    ppm = b"P6 160 120 255\n" + rgb.tobytes()
    assert ex.encode_pnm(ppm, "2K") == oracle_lib.encode_rgb(bundle_b8, rgb, 2)
    with pytest.raises(cg.DataError):
        ex.encode_pnm(b"P6 160 120 255\n" + rgb.tobytes()[:-1], "2K")


def test_cpp_example_extracts_pgm_and_ppm_files(tmp_path, bundle_b8):
    """examples/extract.cpp (the reference CLI's extract flow over the shim's
    load_pnm + encode_image) writes the oracle's container for a PGM and a
    PPM file; a truncated file is a data error (exit code 2)."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.join(root, "paper_1705_09776_b200")
    exe = str(tmp_path / "extract")
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(root, "examples", "extract.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    bundle = tmp_path / "bundle.txt"
    bundle.write_text(bundle_b8)
    grey = oracle_lib.synth_frames(91, 1, 320, 240)[0]
    rgb = oracle_lib.synth_rgb(92, 1, 320, 240)[0]
    cases = [(b"P5\n320 240\n255\n" + grey.tobytes(), oracle_lib.encode(bundle_b8, grey, 3)),
             (b"P6\n320 240\n255\n" + rgb.tobytes(), oracle_lib.encode_rgb(bundle_b8, rgb, 3))]
    for k, (data, want) in enumerate(cases):
        src, dst = tmp_path / f"in{k}.pnm", tmp_path / f"out{k}.cdvz"
        src.write_bytes(data)
        subprocess.run([exe, str(bundle), "4K", str(src), str(dst)], check=True, capture_output=True)
        assert dst.read_bytes() == want
    bad = tmp_path / "bad.ppm"
    bad.write_bytes(cases[1][0][:-10])
    r = subprocess.run([exe, str(bundle), "4K", str(bad), str(tmp_path / "x.cdvz")], capture_output=True)
    assert r.returncode == 2
    # --timings: the reference's StageTimings CSV (stage,calls,total_ms,percent), five labels in order.
    csv_path = tmp_path / "t.csv"
    subprocess.run([exe, str(bundle), "4K", str(tmp_path / "in0.pnm"), str(tmp_path / "o.cdvz"), str(csv_path)],
                   check=True, capture_output=True)
    lines = csv_path.read_text().splitlines()
    assert lines[0] == "stage,calls,total_ms,percent"
    assert [ln.split(",")[0] for ln in lines[1:]] == ["detection", "selection", "description", "compression",
                                                     "aggregation"]
    assert abs(sum(float(ln.split(",")[3]) for ln in lines[1:]) - 100.0) < 0.03  # five values rounded to 0.001
