"""ctypes access to the REFERENCE ITSELF (oracle/_ref/libref.so) — TEST INFRASTRUCTURE.

oracle/refbuild/Makefile compiles /root/reference/proj/src/*.cpp (where they lie,
never copied) against the Eigen-subset and doctest-subset headers in
oracle/refbuild/include, plus oracle/refbuild/ref_capi.cpp (flat C entry points).
The built files live in oracle/_ref/ (git-ignored, shipped to the GPU box with
the snapshot). Only tests/, bench.py's reference leg and tools/ use this
module; the product never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFBUILD = os.path.join(ROOT, "oracle", "refbuild")
REF_DIR = os.path.join(ROOT, "oracle", "_ref")
LIB = os.path.join(REF_DIR, "libref.so")
TESTS_BIN = os.path.join(REF_DIR, "cdvz_tests")
REFERENCE_SRC = "/root/reference/proj"

_lib = None


def available() -> bool:
    """True when the reference library is built (or buildable here)."""
    if os.path.exists(LIB):
        return True
    return os.path.isdir(REFERENCE_SRC)


def build() -> None:
    """Builds oracle/_ref from /root/reference (only where the reference
    exists; the GPU box uses the prebuilt files)."""
    if os.path.isdir(REFERENCE_SRC):
        subprocess.run(["make", "-s", "-j16"], cwd=REFBUILD, check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        P, S, I, U64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_synth_f64.argtypes = [U64, I, I, P]
        L.ref_synth_u8.argtypes = [U64, I, I, P]
        L.ref_bundle_crc.argtypes = [ctypes.c_char_p, S, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(I)]
        L.ref_bundle_canonical.argtypes = [ctypes.c_char_p, S, P, S, ctypes.POINTER(S)]
        L.ref_train_bundle.argtypes = [U64, I, I, I, U64, I, I, I, P, S, ctypes.POINTER(S)]
        L.ref_encode_u8.argtypes = [ctypes.c_char_p, S, P, I, I, S, I, I, I, P, S, ctypes.POINTER(S), P]
        L.ref_encode_f64.argtypes = [ctypes.c_char_p, S, P, I, I, I, I, P, S, ctypes.POINTER(S), P, S, ctypes.POINTER(S)]
        L.ref_encode_batch_u8.argtypes = [ctypes.c_char_p, S, P, I, I, I, I, I, I, I, P, S, P]
        L.ref_stages_u8.argtypes = [ctypes.c_char_p, S, P, I, I, I, ctypes.c_char_p, P, S, ctypes.POINTER(S)]
        _lib = L
    return _lib


def _check(code: int) -> None:
    if code:
        raise RuntimeError(f"reference error {code}: {lib().ref_last_error().decode()}")


def synth_u8(seed: int, w: int, h: int) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    _check(lib().ref_synth_u8(seed, w, h, out.ctypes.data))
    return out


def synth_f64(seed: int, w: int, h: int) -> np.ndarray:
    out = np.empty((h, w), dtype=np.float64)
    _check(lib().ref_synth_f64(seed, w, h, out.ctypes.data))
    return out


def bundle_crc(text: str) -> tuple:
    crc, nc = ctypes.c_uint32(), ctypes.c_int()
    raw = text.encode()
    _check(lib().ref_bundle_crc(raw, len(raw), ctypes.byref(crc), ctypes.byref(nc)))
    return crc.value, nc.value


def train_bundle(corpus_base: int, count: int, w: int, h: int, seed: int, gmm: int, em: int, workers: int = 0) -> str:
    n = ctypes.c_size_t()
    _check(lib().ref_train_bundle(corpus_base, count, w, h, seed, gmm, em, workers, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _check(lib().ref_train_bundle(corpus_base, count, w, h, seed, gmm, em, workers, buf, n.value, ctypes.byref(n)))
    return buf.raw[: n.value].decode()


def encode(text: str, frame: np.ndarray, mode_id: int, max_side: int = 640, workers: int = 1, stage_ms=None) -> bytes:
    """encode_image + serialize_container of the reference on one 8-bit frame."""
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w = frame.shape
    cap = 16384 + 64
    out = np.empty(cap, dtype=np.uint8)
    n = ctypes.c_size_t()
    raw = text.encode()
    _check(lib().ref_encode_u8(raw, len(raw), frame.ctypes.data, w, h, w, mode_id, max_side, workers, out.ctypes.data,
                               cap, ctypes.byref(n), stage_ms.ctypes.data if stage_ms is not None else None))
    return out[: n.value].tobytes()


def encode_f64(text: str, img: np.ndarray, mode_id: int, max_side: int = 640):
    img = np.ascontiguousarray(img, dtype=np.float64)
    h, w = img.shape
    cap = 16384 + 64
    out = np.empty(cap, dtype=np.uint8)
    norms = np.empty(4096, dtype=np.float64)
    n, nn = ctypes.c_size_t(), ctypes.c_size_t()
    raw = text.encode()
    _check(lib().ref_encode_f64(raw, len(raw), img.ctypes.data, w, h, mode_id, max_side, out.ctypes.data, cap,
                                ctypes.byref(n), norms.ctypes.data, norms.size, ctypes.byref(nn)))
    return out[: n.value].tobytes(), norms[: nn.value].copy()


def encode_batch(text: str, frames: np.ndarray, mode_id: int, threads: int, workers: int, max_side: int = 640) -> list:
    """The reference on a batch: `threads` frames in flight, each with
    Engine{workers} (BASELINE.md CPU mode A = (1, nproc), mode B = (nproc, 1))."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    n, h, w = frames.shape
    slot = 16384 + 64
    out = np.empty(n * slot, dtype=np.uint8)
    lens = np.zeros(n, dtype=np.uint64)
    raw = text.encode()
    _check(lib().ref_encode_batch_u8(raw, len(raw), frames.ctypes.data, n, w, h, mode_id, max_side, threads, workers,
                                     out.ctypes.data, slot, lens.ctypes.data))
    return [out[i * slot: i * slot + int(lens[i])].tobytes() for i in range(n)]


def stages(text: str, frame: np.ndarray, name: str, max_side: int = 640) -> np.ndarray:
    """Stage outputs of the reference's extract path: "keypoints", "selected",
    "oriented" (8 or 9 doubles per point) or "descriptors" (128 per point)."""
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w = frame.shape
    raw = text.encode()
    n = ctypes.c_size_t()
    _check(lib().ref_stages_u8(raw, len(raw), frame.ctypes.data, w, h, max_side, name.encode(), None, 0, ctypes.byref(n)))
    out = np.empty(n.value, dtype=np.float64)
    _check(lib().ref_stages_u8(raw, len(raw), frame.ctypes.data, w, h, max_side, name.encode(), out.ctypes.data,
                               out.size, ctypes.byref(n)))
    return out


def run_doctests(suite: str = "") -> dict:
    """Runs the reference's own doctest suites (oracle/_ref/cdvz_tests) ->
    {"passed": [...], "failed": {name: [messages]}}."""
    if not os.path.exists(TESTS_BIN):
        build()
    args = [TESTS_BIN] + ([f"-ts={suite}"] if suite else [])
    r = subprocess.run(args, capture_output=True, text=True, cwd=REF_DIR, timeout=600)
    passed, failed, cur = [], {}, None
    for line in r.stdout.splitlines():
        if line.startswith("PASS "):
            passed.append(line[5:].rsplit(" (", 1)[0])
            cur = None
        elif line.startswith("FAIL "):
            cur = line[5:].rsplit(" (", 1)[0]
            failed[cur] = []
        elif line.startswith("    ") and cur:
            failed[cur].append(line.strip())
    return {"passed": passed, "failed": failed, "returncode": r.returncode}
