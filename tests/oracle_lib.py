"""ctypes access to the CPU oracle (oracle/liborc.so) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs use this module; the product package never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "liborc.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-j8"], cwd=ORACLE_DIR, check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        P, S, I, U64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_synth_u8.argtypes = [U64, I, I, P]
        L.orc_synth_frames_u8.argtypes = [U64, I, I, I, I, P]
        L.orc_bundle_crc.argtypes = [ctypes.c_char_p, S, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(I)]
        L.orc_encode_u8.argtypes = [ctypes.c_char_p, S, P, I, I, S, I, I, P, S, ctypes.POINTER(S), P]
        L.orc_encode_batch_u8.argtypes = [ctypes.c_char_p, S, P, I, I, I, I, I, I, P, S, P]
        L.orc_encode_rgb.argtypes = [ctypes.c_char_p, S, P, I, I, S, I, I, P, S, ctypes.POINTER(S)]
        L.orc_grey_rgb.argtypes = [P, I, I, S, P]
        L.orc_synth_f64.argtypes = [U64, I, I, P]
        L.orc_encode_f64.argtypes = [ctypes.c_char_p, S, P, I, I, I, I, P, S, ctypes.POINTER(S), P, S, ctypes.POINTER(S)]
        L.orc_trace_u8.argtypes = [ctypes.c_char_p, S, P, I, I, I, I, ctypes.POINTER(P)]
        L.orc_trace_free.argtypes = [P]
        L.orc_trace_get.argtypes = [P, ctypes.c_char_p, P, S, ctypes.POINTER(S)]
        L.orc_retrieve.argtypes = [P, P, I, P, P, I, ctypes.c_double, I, P, P]
        L.orc_match_pair.argtypes = [P, S, P, S, ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I)]
        _lib = L
    return _lib


def _check(code: int) -> None:
    if code:
        raise RuntimeError(f"oracle error {code}: {lib().orc_last_error().decode()}")


def bundle_text(name: str = "b8") -> str:
    with open(os.path.join(GOLDEN, f"bundle_{name}.txt")) as f:
        return f.read()


def synth_u8(seed: int, w: int, h: int) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    _check(lib().orc_synth_u8(seed, w, h, out.ctypes.data))
    return out


def synth_frames(base_seed: int, count: int, w: int, h: int, threads: int = 8) -> np.ndarray:
    out = np.empty((count, h, w), dtype=np.uint8)
    _check(lib().orc_synth_frames_u8(base_seed, count, w, h, threads, out.ctypes.data))
    return out


def bundle_crc(text: str) -> tuple:
    crc, nc = ctypes.c_uint32(), ctypes.c_int()
    raw = text.encode()
    _check(lib().orc_bundle_crc(raw, len(raw), ctypes.byref(crc), ctypes.byref(nc)))
    return crc.value, nc.value


def encode(text: str, frame: np.ndarray, mode_id: int, max_side: int = 640) -> bytes:
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w = frame.shape
    cap = 16384 + 64
    out = np.empty(cap, dtype=np.uint8)
    n = ctypes.c_size_t()
    raw = text.encode()
    _check(lib().orc_encode_u8(raw, len(raw), frame.ctypes.data, w, h, w, mode_id, max_side, out.ctypes.data, cap,
                               ctypes.byref(n), None))
    return out[: n.value].tobytes()


def stage_ms(text: str, frames: np.ndarray, mode_id: int, max_side: int = 640) -> dict:
    """Single-threaded encode of each frame with the reference's StageTimings
    labels (pipeline.cpp:19-94); mean ms per frame and label."""
    acc = np.zeros(5, dtype=np.float64)
    raw = text.encode()
    cap = 16384 + 64
    out = np.empty(cap, dtype=np.uint8)
    n = ctypes.c_size_t()
    for f in frames:
        f = np.ascontiguousarray(f, dtype=np.uint8)
        h, w = f.shape
        _check(lib().orc_encode_u8(raw, len(raw), f.ctypes.data, w, h, w, mode_id, max_side, out.ctypes.data, cap,
                                   ctypes.byref(n), acc.ctypes.data))
    labels = ("detection", "selection", "description", "compression", "aggregation")
    return {k: float(v) / max(1, len(frames)) for k, v in zip(labels, acc)}


def encode_rgb(text: str, frame: np.ndarray, mode_id: int, max_side: int = 640) -> bytes:
    """encode_image(load_image(P6 raster)) for one [H, W, 3] uint8 frame."""
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w, _ = frame.shape
    cap = 16384 + 64
    out = np.empty(cap, dtype=np.uint8)
    n = ctypes.c_size_t()
    raw = text.encode()
    _check(lib().orc_encode_rgb(raw, len(raw), frame.ctypes.data, w, h, 3 * w, mode_id, max_side, out.ctypes.data, cap,
                                ctypes.byref(n)))
    return out[: n.value].tobytes()


def synth_f64(seed: int, w: int, h: int) -> np.ndarray:
    """synth_image(seed, w, h) as the reference's f64 GrayImage (no quantisation)."""
    out = np.empty((h, w), dtype=np.float64)
    _check(lib().orc_synth_f64(seed, w, h, out.ctypes.data))
    return out


def encode_f64(text: str, img: np.ndarray, mode_id: int, max_side: int = 640):
    """encode_image on an f64 GrayImage -> (container bytes, SCFVDescriptor.norms)."""
    img = np.ascontiguousarray(img, dtype=np.float64)
    h, w = img.shape
    cap = 16384 + 64
    out = np.empty(cap, dtype=np.uint8)
    norms = np.empty(4096, dtype=np.float64)
    n, nn = ctypes.c_size_t(), ctypes.c_size_t()
    raw = text.encode()
    _check(lib().orc_encode_f64(raw, len(raw), img.ctypes.data, w, h, mode_id, max_side, out.ctypes.data, cap,
                                ctypes.byref(n), norms.ctypes.data, norms.size, ctypes.byref(nn)))
    return out[: n.value].tobytes(), norms[: nn.value].copy()


def grey_rgb(frame: np.ndarray) -> np.ndarray:
    """The grey plane load_image makes of a P6 raster ([H, W, 3] uint8)."""
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w, _ = frame.shape
    out = np.empty((h, w), dtype=np.float64)
    _check(lib().orc_grey_rgb(frame.ctypes.data, w, h, 3 * w, out.ctypes.data))
    return out


def synth_rgb(base_seed: int, count: int, w: int, h: int) -> np.ndarray:
    """[count, h, w, 3] colour frames whose channels are three synthetic grey
    frames (synth_corpus seeds base, base + count, base + 2 count)."""
    g = synth_frames(base_seed, 3 * count, w, h)
    return np.stack([g[:count], g[count:2 * count], g[2 * count:]], axis=-1)


def encode_batch(text: str, frames: np.ndarray, mode_id: int, max_side: int = 640, threads: int = 8) -> list:
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    n, h, w = frames.shape
    slot = 16384 + 64
    out = np.empty(n * slot, dtype=np.uint8)
    lens = np.zeros(n, dtype=np.uint64)
    raw = text.encode()
    _check(lib().orc_encode_batch_u8(raw, len(raw), frames.ctypes.data, n, w, h, mode_id, max_side, threads,
                                     out.ctypes.data, slot, lens.ctypes.data))
    return [out[i * slot: i * slot + int(lens[i])].tobytes() for i in range(n)]


class Trace:
    """encode_image with every intermediate retained (oracle orc_trace_u8)."""

    def __init__(self, text: str, frame: np.ndarray, mode_id: int, max_side: int = 640):
        frame = np.ascontiguousarray(frame, dtype=np.uint8)
        h, w = frame.shape
        self._h = ctypes.c_void_p()
        raw = text.encode()
        _check(lib().orc_trace_u8(raw, len(raw), frame.ctypes.data, w, h, mode_id, max_side, ctypes.byref(self._h)))

    def get(self, name: str) -> np.ndarray:
        n = ctypes.c_size_t()
        _check(lib().orc_trace_get(self._h, name.encode(), None, 0, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.float64)
        _check(lib().orc_trace_get(self._h, name.encode(), out.ctypes.data, out.size, ctypes.byref(n)))
        return out

    def __del__(self):
        try:
            lib().orc_trace_free(self._h)
        except Exception:
            pass


def _pack(containers):
    offs = np.zeros(len(containers) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(c) for c in containers], dtype=np.uint64)
    blob = np.frombuffer(b"".join(containers) or b"\0", dtype=np.uint8).copy()
    return blob, offs


def retrieve(index: list, queries: list, ratio: float = 0.85, depth: int = 50):
    """The oracle's retrieve (eval.cpp:76-124) for each query over `index`
    (ids in index order) -> (items int32 [nq, n], scores float64 [nq, n])."""
    ib, io = _pack(index)
    qb, qo = _pack(queries)
    n, nq = len(index), len(queries)
    items = np.empty((nq, n), dtype=np.int32)
    scores = np.empty((nq, n), dtype=np.float64)
    _check(lib().orc_retrieve(ib.ctypes.data, io.ctypes.data, n, qb.ctypes.data, qo.ctypes.data, nq, ratio, depth,
                              items.ctypes.data, scores.ctypes.data))
    return items, scores


def match_pair(a: bytes, b: bytes, ratio: float = 0.85):
    """The oracle's match_pair (eval.cpp:66-74) -> (global_similarity, local_match_count)."""
    sim, loc = ctypes.c_double(), ctypes.c_int()
    _check(lib().orc_match_pair(a, len(a), b, len(b), ratio, ctypes.byref(sim), ctypes.byref(loc)))
    return sim.value, loc.value
