"""Pins the oracle to the REFERENCE ITSELF (CPU, no GPU needed).

oracle/refbuild/Makefile compiles /root/reference/proj/src/*.cpp and its
doctest suites against an Eigen-subset and a doctest-subset header (Eigen3 and
doctest are absent from this image); tests/ref_lib.py drives the result. Here:

* the reference's own unit suites run, and the only failures are the seven
  known-answer tests the oracle documents as expected failures
  (oracle/selftest.cpp) — so those fail in the reference too;
* the oracle's outputs equal the reference's: containers byte for byte over
  modes, bundles, sizes, f64 input, adversarial frames; keypoints, selection and
  orientations bit for bit; descriptors to 1e-12 (glibc libm on both sides);
* beta (FullPivLU), model_crc and synth_image agree bit for bit;
* the reference's train_model reproduces the committed B8 bundle's detector,
  relevance, transform and quantizer sections exactly (PCA/GMM hang on the
  eigen-solver, which the Eigen-subset cannot pin).
"""
import ctypes

import numpy as np
import pytest

import oracle_lib
import ref_lib

pytestmark = pytest.mark.skipif(not ref_lib.available(), reason="oracle/_ref not built and /root/reference absent")

# The reference's KATs that fail under its own code (with the Eigen-subset);
# oracle/selftest.cpp keeps the same seven as expected failures.
KNOWN_REFERENCE_FAILURES = {
    "refinement is exact against the closed-form quadratic vertex",
    "detection is translation covariant for interior points",
    "two equal orthogonal edge populations emit two orientations",
    "a constant image describes to all zeros",
    "descriptor norm and clamp contract",
    "delta statistics",
    "two well-separated clusters train to even weights",
}


@pytest.fixture(scope="module")
def b8():
    return oracle_lib.bundle_text("b8")


@pytest.fixture(scope="module")
def b512():
    return oracle_lib.bundle_text("b512")


def test_reference_unit_suites_fail_only_the_known_seven():
    res = ref_lib.run_doctests()
    failed = {name.split("] ", 1)[1] for name in res["failed"]}
    assert len(res["passed"]) >= 130
    assert failed == KNOWN_REFERENCE_FAILURES, res["failed"]


def test_beta_crc_and_synth_match_the_reference(b8, b512):
    for text in (b8, b512):
        assert oracle_lib.bundle_crc(text) == ref_lib.bundle_crc(text)
    raw = b8.encode()
    a, b = np.zeros(16), np.zeros(16)
    assert ref_lib.lib().ref_bundle_beta(raw, ctypes.c_size_t(len(raw)), a.ctypes.data_as(ctypes.c_void_p)) == 0
    L = oracle_lib.lib()
    assert L.orc_bundle_beta(raw, ctypes.c_size_t(len(raw)), b.ctypes.data_as(ctypes.c_void_p)) == 0
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    for seed, (w, h) in [(1000, (640, 480)), (77, (97, 61))]:
        assert np.array_equal(oracle_lib.synth_u8(seed, w, h), ref_lib.synth_u8(seed, w, h))
        assert np.array_equal(oracle_lib.synth_f64(seed, w, h), ref_lib.synth_f64(seed, w, h))


def test_containers_match_the_reference(b8, b512):
    frames = oracle_lib.synth_frames(1000, 4, 640, 480)
    for i, f in enumerate(frames):
        for mode in (0, 3, 5):
            assert oracle_lib.encode(b8, f, mode) == ref_lib.encode(b8, f, mode), f"frame {i} mode {mode}"
    assert oracle_lib.encode(b512, frames[0], 3) == ref_lib.encode(b512, frames[0], 3)
    assert oracle_lib.encode(b512, frames[1], 4) == ref_lib.encode(b512, frames[1], 4)
    big = oracle_lib.synth_frames(2000, 1, 1920, 1080)[0]  # resize_max_side -> 640x360
    assert oracle_lib.encode(b8, big, 5) == ref_lib.encode(b8, big, 5)
    rng = np.random.default_rng(5)
    noise = rng.integers(0, 256, (480, 640), dtype=np.uint8)
    assert oracle_lib.encode(b8, noise, 3) == ref_lib.encode(b8, noise, 3)
    flat = np.full((240, 320), 128, dtype=np.uint8)  # no keypoints: the n = 0 SCFV edge case
    assert oracle_lib.encode(b8, flat, 3) == ref_lib.encode(b8, flat, 3)


def test_f64_input_and_norms_match_the_reference(b8):
    img = oracle_lib.synth_f64(4242, 640, 480)
    c0, n0 = oracle_lib.encode_f64(b8, img, 4)
    c1, n1 = ref_lib.encode_f64(b8, img, 4)
    assert c0 == c1
    assert np.array_equal(n0, n1)


def test_stage_outputs_match_the_reference(b8):
    frame = oracle_lib.synth_frames(1000, 1, 640, 480)[0]
    tr = oracle_lib.Trace(b8, frame, 3)
    for name in ("keypoints", "selected", "oriented"):
        assert np.array_equal(tr.get(name), ref_lib.stages(b8, frame, name)), name
    d0, d1 = tr.get("descriptors"), ref_lib.stages(b8, frame, "descriptors")
    assert d0.shape == d1.shape
    assert np.array_equal(d0, d1)


def test_engine_workers_do_not_change_the_reference_output(b8):
    """parallel.hpp:16-18 on the reference itself: Engine{1} == Engine{4}, and
    the CPU baseline's mode A (intra-frame workers) == mode B (frame threads)."""
    frames = oracle_lib.synth_frames(1300, 3, 320, 240)
    a = ref_lib.encode_batch(b8, frames, 3, threads=1, workers=4)
    b = ref_lib.encode_batch(b8, frames, 3, threads=3, workers=1)
    assert a == b
    assert a[0] == oracle_lib.encode(b8, frames[0], 3)


def test_reference_training_reproduces_the_committed_bundle_sections(b8):
    """train_model(synth_corpus(401, 20, 256, 256), seed 11, GMM 8, EM 15) in the
    reference (acceptance.cpp:509-514): every section before the PCA is
    identical to the committed B8 bundle; PCA and GMM depend on the eigen
    solver (Eigen's SelfAdjointEigenSolver vs a Jacobi restatement)."""
    got = ref_lib.train_bundle(401, 20, 256, 256, 11, 8, 15, workers=8)
    head = lambda t: t[: t.index("section pca")]
    assert head(got) == head(b8)
