"""GPU training (cdvz_gpu_train_model): train_model (proj/src/pipeline.cpp:
99-166) with pass 1, the partner detection, the PCA covariance / projection,
the EM iterations and the descriptor transform on the device.

Checked against the committed B8 bundle, which is the reference's own
train_model(synth_corpus(401, 20, 256, 256), seed 11, GMM 8, EM 15)
(tests/golden/make_bundles.py, oracle/_ref):
* the detector, selector (relevance tables from the labelled partner pairs)
  and transform sections are byte-identical: pass 1, apply_transform, the
  partner detection and the labelling reproduce the reference bit for bit;
* the quantizer, PCA and GMM sections agree numerically: they go through
  libm (descriptor atan2 / exp / hypot, EM exp / log) and an eigensolver,
  whose last bits differ between libdevice / this Jacobi and glibc / the
  reference build;
* the GPU-trained bundle is a working bundle: the extractor's containers with
  it equal the oracle's with it.
"""
import numpy as np
import pytest

import oracle_lib

pytestmark = pytest.mark.gpu

cg = pytest.importorskip("paper_1705_09776_b200")

GOLDEN = 0x9E3779B97F4A7C15


def sections(text):
    out, lines, i = {}, text.split("\n"), 1
    while i < len(lines) and lines[i].startswith("section "):
        _, name, n, _crc = lines[i].split()
        out[name] = lines[i + 1:i + 1 + int(n)]
        i += 1 + int(n)
    return out


def numbers(lines):
    vals = []
    for ln in lines:
        for tok in ln.replace("=", " ").split():
            try:
                vals.append(float(tok))
            except ValueError:
                pass
    return np.array(vals)


@pytest.fixture(scope="module")
def trained():
    corpus = np.stack([oracle_lib.synth_f64((401 + i * GOLDEN) % (1 << 64), 256, 256) for i in range(20)])
    return cg.train_model(corpus, seed=11, gmm_components=8, em_iterations=15)


def test_trained_sections_against_the_reference(trained, bundle_b8):
    got, want = sections(trained), sections(bundle_b8)
    assert list(got) == list(want) == ["detector", "selector", "transforms", "quantizer", "pca", "gmm"]
    for name in ("detector", "selector", "transforms"):
        assert got[name] == want[name], name
    q_got, q_want = got["quantizer"], want["quantizer"]
    assert np.allclose(numbers(q_got[:2]), numbers(q_want[:2]), rtol=1e-9, atol=1e-12)
    assert q_got[2:] == q_want[2:]  # priority order and degenerate flags
    g, w = numbers(got["pca"]), numbers(want["pca"])
    assert g.shape == w.shape and np.allclose(g, w, rtol=1e-6, atol=1e-9)
    g, w = numbers(got["gmm"]), numbers(want["gmm"])
    assert g.shape == w.shape and np.allclose(g, w, rtol=1e-5, atol=1e-8)


def test_trained_bundle_encodes_like_the_oracle(trained):
    cg.bundle_check(trained)
    frames = oracle_lib.synth_frames(7000, 3, 640, 480)
    ex = cg.Extractor(trained, max_batch=4)
    got, st = ex.encode_batch(frames, "4K")
    ex.close()
    assert st.tolist() == [0, 0, 0]
    for i in range(3):
        assert got[i] == oracle_lib.encode(trained, frames[i], 3)


def test_train_model_argument_errors():
    small = np.zeros((5, 64, 64))
    with pytest.raises(cg.DataError):
        cg.train_model(small)


def test_cpp_train_cli_matches_the_python_binding(tmp_path):
    """examples/train.cpp (run_train over the shim: PGM files, load_image's
    v / 255, train_model, save_model) writes the bundle the ctypes binding
    trains from the same rasters."""
    import os
    import subprocess

    rasters = [np.round(oracle_lib.synth_f64((401 + i * GOLDEN) % (1 << 64), 128, 128) * 255.0).astype(np.uint8)
               for i in range(20)]
    corpus = tmp_path / "corpus"
    corpus.mkdir()
    for i, r in enumerate(rasters):
        (corpus / f"img{i:02d}.pgm").write_bytes(b"P5\n128 128\n255\n" + r.tobytes())
    exe = tmp_path / "train"
    lib_dir = os.path.dirname(cg.library_path())
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(root, "examples", "train.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = tmp_path / "bundle.txt"
    p = subprocess.run([str(exe), str(corpus), str(out), "5", "4", "6", "120"], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    want = cg.train_model(np.stack([r.astype(np.float64) * (1.0 / 255.0) for r in rasters]), seed=5,
                          gmm_components=4, em_iterations=6, select_n=120)
    assert out.read_text() == want
    assert f"crc {cg.bundle_check(want)[0]:08x}" in p.stdout
