"""B200-native CDVS-style extractor (arxiv 1705.09776 reference path).

Python host mirror of the reference's extraction API
(/root/reference/proj/include/cdvz/pipeline.hpp:18-20 ``encode_image``,
container.hpp:27 ``serialize_container``, model_io.hpp:30-33 ``load_model``,
transform_coding.hpp:22-24 ``mode_by_name``/``mode_by_id``) over the C ABI in
``include/cdvz_gpu.h``. All compute runs in ``libcdvz_gpu.so`` (sm_100a CUDA);
there is no CPU fallback: a missing library or device raises.

Errors mirror the reference's exception classes: ``UsageError`` (bad mode name,
bad arguments) and ``DataError`` (bad raster, bad bundle), plus
``InternalError`` for device failures (the CLI's exit code 3).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Iterable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libcdvz_gpu.so")


class UsageError(RuntimeError):
    """Reference UsageError (proj/include/cdvz/common.hpp:12-14)."""


class DataError(RuntimeError):
    """Reference DataError (proj/include/cdvz/common.hpp:15-17)."""


class InternalError(RuntimeError):
    """Device / runtime failure (CLI exit code 3, proj/tools/cdvz.cpp:308-317)."""


@dataclass(frozen=True)
class ModeSpec:
    """proj/include/cdvz/transform_coding.hpp:13-20."""

    id: int
    name: str
    budget_bytes: int
    elements: int
    scfv_fraction: float
    variance_planes: bool


MODES = (
    ModeSpec(0, "512B", 512, 20, 32.0 / 512.0, False),
    ModeSpec(1, "1K", 1024, 32, 64.0 / 512.0, False),
    ModeSpec(2, "2K", 2048, 64, 128.0 / 512.0, False),
    ModeSpec(3, "4K", 4096, 103, 256.0 / 512.0, False),
    ModeSpec(4, "8K", 8192, 103, 320.0 / 512.0, True),
    ModeSpec(5, "16K", 16384, 128, 512.0 / 512.0, True),
)


def mode_by_name(name: str) -> ModeSpec:
    """transform_coding.cpp:39-44 — UsageError on an unknown name."""
    for m in MODES:
        if m.name == name:
            return m
    raise UsageError(f"unknown mode '{name}' (expected 512B, 1K, 2K, 4K, 8K or 16K)")


def mode_by_id(mode_id: int) -> ModeSpec:
    """transform_coding.cpp:33-37 — DataError on an unknown id."""
    for m in MODES:
        if m.id == mode_id:
            return m
    raise DataError(f"unknown mode id {mode_id}")


_lib_handle: Optional[ctypes.CDLL] = None


def library_path() -> str:
    return _LIB_PATH


def _lib() -> ctypes.CDLL:
    global _lib_handle
    if _lib_handle is not None:
        return _lib_handle
    if not os.path.exists(_LIB_PATH):
        raise InternalError(f"{_LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    P, S, I, U32, U64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64
    sig = {
        "cdvz_gpu_create": (I, [ctypes.c_char_p, S, I, I, ctypes.POINTER(P)]),
        "cdvz_gpu_create_multi": (I, [ctypes.c_char_p, S, P, I, I, ctypes.POINTER(P)]),
        "cdvz_gpu_device_count": (I, [P, P, I]),
        "cdvz_gpu_visible_devices": (I, []),
        "cdvz_gpu_encode_batch_f64": (I, [P, P, I, I, S, I, I, I, P, S, P, P]),
        "cdvz_gpu_destroy": (None, [P]),
        "cdvz_gpu_last_error": (ctypes.c_char_p, [P]),
        "cdvz_gpu_bundle_check": (I, [ctypes.c_char_p, S, ctypes.POINTER(U32), ctypes.POINTER(I)]),
        "cdvz_gpu_bundle_info": (I, [P, ctypes.POINTER(U32), ctypes.POINTER(I), ctypes.POINTER(I)]),
        "cdvz_gpu_encode_batch": (I, [P, P, I, I, S, I, I, I, P, S, P, P]),
        "cdvz_gpu_encode_batch_rgb": (I, [P, P, I, I, S, I, I, I, P, S, P, P]),
        "cdvz_gpu_encode_batch_submit": (I, [P, P, I, I, S, I, I, I, P, S, P, P, ctypes.POINTER(U64)]),
        "cdvz_gpu_train_model": (I, [I, P, I, I, I, S, U64, I, I, I, I, I, P, S, ctypes.POINTER(S)]),
        "cdvz_gpu_encode_batch_wait": (I, [P, U64]),
        "cdvz_gpu_pnm_parse": (I, [P, S, ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(S)]),
        "cdvz_gpu_encode_device": (I, [P, P, I, I, S, I, I, I, P, P]),
        "cdvz_gpu_container_slot": (S, [I]),
        "cdvz_gpu_sync": (I, [P]),
        "cdvz_gpu_trim": (I, [P]),
        "cdvz_gpu_stage_times": (I, [P, P]),
        "cdvz_gpu_kernel_stats": (I, [P, ctypes.POINTER(I), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "cdvz_gpu_debug_get": (I, [P, ctypes.c_char_p, I, P, S, ctypes.POINTER(S)]),
        "cdvz_gpu_set_debug": (I, [P, I]),
        "cdvz_gpu_event_record": (I, [P, I]),
        "cdvz_gpu_event_elapsed": (I, [P, I, I, ctypes.POINTER(ctypes.c_double)]),
        "cdvz_gpu_synth_frames": (I, [P, U64, I, I, I, P]),
        "cdvz_gpu_device_alloc": (I, [P, S, ctypes.POINTER(P)]),
        "cdvz_gpu_device_free": (I, [P, P]),
        "cdvz_gpu_host_alloc": (I, [P, S, ctypes.POINTER(P)]),
        "cdvz_gpu_host_free": (I, [P, P]),
        "cdvz_gpu_copy": (I, [P, P, P, S, I]),
        "cdvz_gpu_pyramid_bench": (I, [P, P, I, I, I, I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "cdvz_gpu_index_create": (I, [I, P, P, I, P, ctypes.POINTER(P)]),
        "cdvz_gpu_index_destroy": (None, [P]),
        "cdvz_gpu_index_last_error": (ctypes.c_char_p, [P]),
        "cdvz_gpu_index_info": (I, [P, ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(U32), ctypes.POINTER(I),
                                    ctypes.POINTER(ctypes.c_longlong)]),
        "cdvz_gpu_retrieve": (I, [P, P, P, I, ctypes.c_double, I, I, P, P]),
        "cdvz_gpu_match_pairs": (I, [P, P, P, I, P, I, ctypes.c_double, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib_handle = lib
    return lib


def _raise(code: int, msg: str) -> None:
    if code == 0:
        return
    if code == 1:
        raise UsageError(msg)
    if code == 2:
        raise DataError(msg)
    raise InternalError(msg)


def device_count() -> int:
    """Number of visible CUDA devices (0 without a GPU)."""
    return int(_lib().cdvz_gpu_visible_devices())


def bundle_check(bundle_text: str) -> tuple:
    """Host-only parse/validate of a bundle; returns (model_crc, components)."""
    lib = _lib()
    raw = bundle_text.encode() if isinstance(bundle_text, str) else bytes(bundle_text)
    crc, nc = ctypes.c_uint32(), ctypes.c_int()
    code = lib.cdvz_gpu_bundle_check(raw, len(raw), ctypes.byref(crc), ctypes.byref(nc))
    _raise(code, lib.cdvz_gpu_last_error(None).decode())
    return crc.value, nc.value


class DeviceBuffer:
    """Device allocation owned by an Extractor's device (for the HBM-resident path)."""

    def __init__(self, ex: "Extractor", nbytes: int):
        self._ex = ex
        self.nbytes = nbytes
        ptr = ctypes.c_void_p()
        ex._check(ex._lib.cdvz_gpu_device_alloc(ex._ctx, nbytes, ctypes.byref(ptr)))
        self.ptr = ptr.value

    def to_host(self, nbytes: Optional[int] = None) -> np.ndarray:
        n = self.nbytes if nbytes is None else nbytes
        out = np.empty(n, dtype=np.uint8)
        self._ex._check(self._ex._lib.cdvz_gpu_copy(self._ex._ctx, out.ctypes.data, self.ptr, n, 2))
        return out

    def from_host(self, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr)
        self._ex._check(self._ex._lib.cdvz_gpu_copy(self._ex._ctx, self.ptr, arr.ctypes.data, arr.nbytes, 1))

    def free(self) -> None:
        if self.ptr:
            self._ex._lib.cdvz_gpu_device_free(self._ex._ctx, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host buffer (cudaMallocHost) exposed as a numpy array."""

    def __init__(self, ex: "Extractor", nbytes: int):
        self._ex = ex
        ptr = ctypes.c_void_p()
        ex._check(ex._lib.cdvz_gpu_host_alloc(ex._ctx, nbytes, ctypes.byref(ptr)))
        self.ptr = ptr.value
        self.array = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(self.ptr))

    def free(self) -> None:
        if self.ptr:
            self._ex._lib.cdvz_gpu_host_free(self._ex._ctx, self.ptr)
            self.ptr = None


def parse_pnm(data: bytes):
    """The header of a binary PGM/PPM held in memory, parsed like load_image
    (proj/src/image.cpp:53-77): returns (width, height, channels, raster_offset);
    raises DataError for a malformed file."""
    lib = _lib()
    buf = ctypes.create_string_buffer(bytes(data), len(data))
    w, h, ch, off = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
    code = lib.cdvz_gpu_pnm_parse(ctypes.addressof(buf), len(data), ctypes.byref(w), ctypes.byref(h), ctypes.byref(ch),
                                  ctypes.byref(off))
    _raise(code, lib.cdvz_gpu_last_error(None).decode())
    return w.value, h.value, ch.value, off.value


def train_model(corpus: np.ndarray, seed: int = 7, gmm_components: int = 8, em_iterations: int = 25,
                select_n: int = 300, max_side: int = 640, relevance_bins: int = 16, device: int = 0) -> str:
    """train_model (proj/src/pipeline.cpp:99-166) on the GPU (cdvz_gpu_train_model):
    ``corpus`` is float64 [N, H, W] (N >= 20 GrayImages in [0, 1]); returns the
    bundle text. Defaults are the reference's TrainOptions."""
    lib = _lib()
    c = np.ascontiguousarray(corpus, dtype=np.float64)
    if c.ndim != 3:
        raise UsageError("corpus must be float64 [N, H, W]")
    n, h, w = c.shape
    ln = ctypes.c_size_t()
    cap = (1 << 20) + 2048 * max(1, gmm_components)  # ~1.4 KB of text per component, plus the rest
    buf = ctypes.create_string_buffer(cap)
    rc = lib.cdvz_gpu_train_model(device, c.ctypes.data, n, w, h, w, seed, gmm_components, em_iterations, select_n,
                                  max_side, relevance_bins, buf, cap, ctypes.byref(ln))
    if rc:
        _raise(rc, lib.cdvz_gpu_last_error(None).decode())
    return buf.raw[:ln.value].decode()


class PendingBatch:
    """A submitted batch (Extractor.encode_batch_submit); holds its buffers."""

    def __init__(self, ex: "Extractor", frames: np.ndarray, n: int, slot: int):
        self.ex, self.frames, self.n = ex, frames, n
        self.out = np.empty(max(1, n * slot), dtype=np.uint8)
        self.offsets = np.zeros(n + 1, dtype=np.uint64)
        self.status = np.zeros(max(1, n), dtype=np.int32)
        self.ticket = 0
        self._done = None

    def wait(self):
        if self._done is None:
            self.ex._check(self.ex._lib.cdvz_gpu_encode_batch_wait(self.ex._ctx, self.ticket))
            res = [self.out[int(self.offsets[i]):int(self.offsets[i + 1])].tobytes() for i in range(self.n)]
            self._done = (res, self.status[:self.n].copy())
        return self._done


class Extractor:
    """One GPU context holding a model bundle: the reference's
    ``encode_image(img, bundle, mode)`` for batches of frames (8-bit grey or
    RGB rasters, or the reference's own f64 GrayImage values).

    ``devices``: a list of device indices makes a multi-device context
    (``cdvz_gpu_create_multi``): host batches are frame-sharded across the
    devices, one host thread each, and gathered in frame order."""

    def __init__(self, bundle_text: str, device: int = 0, max_batch: int = 256, devices: Optional[Sequence[int]] = None):
        self._lib = _lib()
        raw = bundle_text.encode() if isinstance(bundle_text, str) else bytes(bundle_text)
        ctx = ctypes.c_void_p()
        if devices is not None:
            devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
            code = self._lib.cdvz_gpu_create_multi(raw, len(raw), devs.ctypes.data, len(devs), max_batch, ctypes.byref(ctx))
            device = int(devs[0]) if len(devs) else device
        else:
            code = self._lib.cdvz_gpu_create(raw, len(raw), device, max_batch, ctypes.byref(ctx))
        _raise(code, self._lib.cdvz_gpu_last_error(None).decode())
        self._ctx = ctx.value
        crc, nc, sel = ctypes.c_uint32(), ctypes.c_int(), ctypes.c_int()
        self._lib.cdvz_gpu_bundle_info(self._ctx, ctypes.byref(crc), ctypes.byref(nc), ctypes.byref(sel))
        self.model_crc, self.components, self.select_n = crc.value, nc.value, sel.value
        self.device = device
        self.max_batch = max_batch
        devs = (ctypes.c_int * 64)()
        n = self._lib.cdvz_gpu_device_count(self._ctx, devs, 64)
        self.devices = [int(devs[i]) for i in range(min(n, 64))]

    # -- plumbing
    def _check(self, code: int) -> None:
        if code:
            _raise(code, self._lib.cdvz_gpu_last_error(self._ctx).decode())

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.cdvz_gpu_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- reference API
    def encode_batch(self, frames: np.ndarray, mode, max_side: int = 640):
        """Encodes ``frames`` and returns (containers, status):
        ``containers[i]`` is frame i's CDVZ1 byte string (b"" on failure).
        uint8 [N, H, W] grey (PGM bytes, read as b/255) or [N, H, W, 3] RGB (as
        in a PPM); float64 [N, H, W] grey values in [0, 1] (the reference's
        GrayImage, validated per frame like validate())."""
        m = mode if isinstance(mode, ModeSpec) else (mode_by_name(mode) if isinstance(mode, str) else mode_by_id(mode))
        f64 = np.asarray(frames).dtype == np.float64
        frames = np.ascontiguousarray(frames, dtype=np.float64 if f64 else np.uint8)
        if frames.ndim == 2:
            frames = frames[None]
        rgb = frames.ndim == 4
        if frames.ndim not in (3, 4) or (rgb and (frames.shape[-1] != 3 or f64)):
            raise UsageError("frames must be [N, H, W] or [N, H, W, 3] uint8, or [N, H, W] float64")
        n, h, w = frames.shape[:3]
        ch = 3 if rgb else 1
        slot = m.budget_bytes + 28
        out = np.empty(max(1, n * slot), dtype=np.uint8)
        offsets = np.zeros(n + 1, dtype=np.uint64)
        status = np.zeros(max(1, n), dtype=np.int32)
        if f64:
            fn, stride = self._lib.cdvz_gpu_encode_batch_f64, w
        else:
            fn, stride = (self._lib.cdvz_gpu_encode_batch_rgb if rgb else self._lib.cdvz_gpu_encode_batch), w * ch
        self._check(fn(self._ctx, frames.ctypes.data, w, h, stride, n, m.id, max_side, out.ctypes.data, out.nbytes,
                       offsets.ctypes.data, status.ctypes.data))
        res = [out[int(offsets[i]):int(offsets[i + 1])].tobytes() for i in range(n)]
        return res, status[:n].copy()

    def encode_batch_submit(self, frames: np.ndarray, mode, max_side: int = 640) -> "PendingBatch":
        """cdvz_gpu_encode_batch_submit for uint8 [N, H, W] grey frames: returns
        at once; ``.wait()`` gives (containers, status) like encode_batch.
        Up to two batches are in flight per extractor (the frames array is
        kept alive by the handle)."""
        m = mode if isinstance(mode, ModeSpec) else (mode_by_name(mode) if isinstance(mode, str) else mode_by_id(mode))
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        if frames.ndim == 2:
            frames = frames[None]
        if frames.ndim != 3:
            raise UsageError("frames must be [N, H, W] uint8")
        n, h, w = frames.shape
        slot = m.budget_bytes + 28
        pb = PendingBatch(self, frames, n, slot)
        t = ctypes.c_uint64()
        self._check(self._lib.cdvz_gpu_encode_batch_submit(self._ctx, frames.ctypes.data, w, h, w, n, m.id, max_side,
                                                           pb.out.ctypes.data, pb.out.nbytes, pb.offsets.ctypes.data,
                                                           pb.status.ctypes.data, ctypes.byref(t)))
        pb.ticket = t.value
        return pb

    def encode_pnm(self, data: bytes, mode, max_side: int = 640) -> bytes:
        """load_image + encode_image + serialize_container for one in-memory
        PGM/PPM file (proj/src/image.cpp:53-92)."""
        w, h, ch, off = parse_pnm(data)
        raster = np.frombuffer(data, dtype=np.uint8, count=w * h * ch, offset=off)
        frames = raster.reshape(1, h, w, 3) if ch == 3 else raster.reshape(1, h, w)
        res, status = self.encode_batch(frames, mode, max_side)
        if status[0] != 0:
            _raise(int(status[0]), self._lib.cdvz_gpu_last_error(self._ctx).decode() or "frame failed")
        return res[0]

    def encode_image(self, frame: np.ndarray, mode, max_side: int = 640) -> bytes:
        """encode_image + serialize_container for one frame; raises on failure."""
        res, status = self.encode_batch(np.asarray(frame)[None], mode, max_side)
        if status[0] == 2:
            raise DataError("image values must be finite and in [0, 1]")
        if status[0] != 0:
            _raise(int(status[0]), self._lib.cdvz_gpu_last_error(self._ctx).decode() or "frame failed")
        return res[0]

    def encode_device(self, d_frames: DeviceBuffer, count: int, width: int, height: int, mode, d_out: DeviceBuffer,
                      d_lengths: DeviceBuffer, max_side: int = 640) -> None:
        m = mode if isinstance(mode, ModeSpec) else (mode_by_name(mode) if isinstance(mode, str) else mode_by_id(mode))
        self._check(self._lib.cdvz_gpu_encode_device(self._ctx, d_frames.ptr, width, height, width, count, m.id,
                                                     max_side, d_out.ptr, d_lengths.ptr))

    def trim(self) -> None:
        """Free the per-batch device buffers (re-planned by the next encode)."""
        self._check(self._lib.cdvz_gpu_trim(self._ctx))

    def sync(self) -> None:
        self._check(self._lib.cdvz_gpu_sync(self._ctx))

    def stage_times(self) -> dict:
        """Device ms per reference stage label (parallel.hpp:117-134)."""
        arr = (ctypes.c_double * 5)()
        self._check(self._lib.cdvz_gpu_stage_times(self._ctx, arr))
        return dict(zip(("detection", "selection", "description", "compression", "aggregation"), list(arr)))

    def kernel_stats(self) -> dict:
        n, ms, by = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        self._check(self._lib.cdvz_gpu_kernel_stats(self._ctx, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by)))
        return {"launches": n.value, "pyramid_ms": ms.value, "pyramid_bytes": by.value}

    def set_debug(self, on: bool = True, exact_only: bool = False, serial: bool = False, no_tma: bool = False,
                  tile_detect: bool = False, tiny_caps: bool = False, blur_unrolled: bool = False,
                  post_simt: bool = False, desc_registers: bool = False) -> None:
        """on: keep per-octave lists; exact_only: bypass the FP32 extrema screen;
        serial: no kernel overlap (standalone per-kernel timing); tile_detect:
        the first-generation TMA tile extrema kernel instead of the column walk
        (a cross-check); no_tma: no TMA (the tile kernel with plain loads, the
        column walk with per-lane cp.async rows); tiny_caps: tiny list
        capacities, so frames take the capacity retry; blur_unrolled: k_blur's
        y pass unrolled by one accumulator period instead of the rolled loop;
        post_simt: SCFV posteriors of large mixtures on the FP64 SIMT kernel
        (gamma bit-identical to the reference's separately rounded products)
        instead of the FP64 tensor cores; desc_registers: the
        descriptor histograms with register bins (k_describe) instead of the
        shared-memory cell accumulators (k_describe_cells)."""
        flags = ((1 if on else 0) | (2 if exact_only else 0) | (4 if serial else 0) | (8 if no_tma else 0)
                 | (16 if tile_detect else 0) | (32 if tiny_caps else 0) | (64 if blur_unrolled else 0)
                 | (128 if post_simt else 0) | (256 if desc_registers else 0))
        self._check(self._lib.cdvz_gpu_set_debug(self._ctx, flags))

    def debug_get(self, name: str, frame: int) -> np.ndarray:
        n = ctypes.c_size_t()
        self._check(self._lib.cdvz_gpu_debug_get(self._ctx, name.encode(), frame, None, 0, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.float64)
        self._check(self._lib.cdvz_gpu_debug_get(self._ctx, name.encode(), frame, out.ctypes.data, out.size,
                                                 ctypes.byref(n)))
        return out

    def event_record(self, slot: int) -> None:
        self._check(self._lib.cdvz_gpu_event_record(self._ctx, slot))

    def event_elapsed(self, a: int, b: int) -> float:
        ms = ctypes.c_double()
        self._check(self._lib.cdvz_gpu_event_elapsed(self._ctx, a, b, ctypes.byref(ms)))
        return ms.value

    def device_buffer(self, nbytes: int) -> DeviceBuffer:
        return DeviceBuffer(self, nbytes)

    def pinned_buffer(self, nbytes: int) -> PinnedBuffer:
        return PinnedBuffer(self, nbytes)

    def synth_frames_device(self, base_seed: int, count: int, width: int, height: int) -> DeviceBuffer:
        """synth_corpus(base_seed, count, width, height) quantised to bytes, on the device."""
        buf = DeviceBuffer(self, max(1, count * width * height))
        self._check(self._lib.cdvz_gpu_synth_frames(self._ctx, base_seed, count, width, height, buf.ptr))
        return buf

    def pyramid_bench(self, d_frames: DeviceBuffer, count: int, width: int, height: int, iters: int = 5) -> tuple:
        """(ms per pass, algorithmic bytes per pass) of the octave kernel pair at native size."""
        ms, by = ctypes.c_double(), ctypes.c_double()
        self._check(self._lib.cdvz_gpu_pyramid_bench(self._ctx, d_frames.ptr, width, height, count, iters,
                                                     ctypes.byref(ms), ctypes.byref(by)))
        return ms.value, by.value

    def synth_frames(self, base_seed: int, count: int, width: int, height: int) -> np.ndarray:
        buf = self.synth_frames_device(base_seed, count, width, height)
        arr = buf.to_host(count * width * height).reshape(count, height, width)
        buf.free()
        return arr


def _pack(containers) -> tuple:
    """Concatenate container byte strings -> (uint8 blob, uint64 offsets[n+1])."""
    offs = np.zeros(len(containers) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(c) for c in containers], dtype=np.uint64)
    blob = np.frombuffer(b"".join(containers), dtype=np.uint8) if containers else np.zeros(1, np.uint8)
    if blob.size == 0:
        blob = np.zeros(1, np.uint8)
    return np.ascontiguousarray(blob), offs


class Index:
    """Compressed-domain retrieval index on one GPU: the
    reference's retrieve / match_pair (proj/src/eval.cpp:66-124) over CDVZ1
    containers decoded on the device (parse_container, container.cpp:60-93).

    ids: optional item ids; their ascending order is the tie-break of equal
    scores, as in the reference (default: index order)."""

    def __init__(self, containers, device: int = 0, ids=None):
        self._lib = _lib()
        self._idx = ctypes.c_void_p()
        self._blob, self._offs = _pack(list(containers))
        n = len(self._offs) - 1
        self.ids = list(ids) if ids is not None else None
        rank = None
        if ids is not None:
            if len(ids) != n:
                raise UsageError("one id per container")
            order = sorted(range(n), key=lambda i: ids[i])
            rank = np.empty(n, dtype=np.int32)
            rank[np.array(order, dtype=np.int64)] = np.arange(n, dtype=np.int32)
        code = self._lib.cdvz_gpu_index_create(device, self._blob.ctypes.data, self._offs.ctypes.data, n,
                                               rank.ctypes.data if rank is not None else None, ctypes.byref(self._idx))
        if code:
            _raise(code, (self._lib.cdvz_gpu_index_last_error(None) or b"").decode())
        self.count = n

    def _check(self, code: int) -> None:
        if code:
            _raise(code, (self._lib.cdvz_gpu_index_last_error(self._idx) or b"").decode())

    def info(self) -> dict:
        n, m, nc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        crc, tot = ctypes.c_uint32(), ctypes.c_longlong()
        self._check(self._lib.cdvz_gpu_index_info(self._idx, ctypes.byref(n), ctypes.byref(m), ctypes.byref(crc),
                                                  ctypes.byref(nc), ctypes.byref(tot)))
        return {"count": n.value, "mode_id": m.value, "model_crc": crc.value, "components": nc.value,
                "total_codes": tot.value}

    def retrieve_batch(self, queries, ratio_test: float = 0.85, rerank_depth: int = 50, max_results: int = 0,
                       out=None):
        """retrieve() for every query -> (items int32 [nq, k], scores float64 [nq, k]).
        out: optional preallocated (items, scores) of those shapes and dtypes —
        e.g. views of pinned buffers (Extractor.pinned_buffer), which the
        device-to-host copy of the ranked lists fills at full link speed."""
        blob, offs = _pack(list(queries))
        nq = len(offs) - 1
        k = self.count if max_results <= 0 else min(self.count, max_results)
        if out is None:
            items = np.empty((nq, k), dtype=np.int32)
            scores = np.empty((nq, k), dtype=np.float64)
        else:
            items, scores = out
            if (items.shape != (nq, k) or items.dtype != np.int32 or not items.flags.c_contiguous
                    or scores.shape != (nq, k) or scores.dtype != np.float64 or not scores.flags.c_contiguous):
                raise UsageError(f"out must be C-contiguous int32 and float64 arrays of shape {(nq, k)}")
        self._check(self._lib.cdvz_gpu_retrieve(self._idx, blob.ctypes.data, offs.ctypes.data, nq, ratio_test,
                                                rerank_depth, max_results, items.ctypes.data, scores.ctypes.data))
        return items, scores

    def retrieve(self, query: bytes, ratio_test: float = 0.85, rerank_depth: int = 50) -> list:
        """The reference's RankedList for one query: [(id, score), ...]."""
        items, scores = self.retrieve_batch([query], ratio_test, rerank_depth)
        ids = self.ids if self.ids is not None else list(range(self.count))
        return [(ids[int(i)], float(s)) for i, s in zip(items[0], scores[0])]

    def match_pairs(self, queries, pairs, ratio_test: float = 0.85):
        """match_pair(queries[q], index[i]) for (q, i) in pairs -> (global_sim, local_matches)."""
        blob, offs = _pack(list(queries))
        pr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        sim = np.empty(len(pr), dtype=np.float64)
        loc = np.empty(len(pr), dtype=np.int32)
        self._check(self._lib.cdvz_gpu_match_pairs(self._idx, blob.ctypes.data, offs.ctypes.data, len(offs) - 1,
                                                   pr.ctypes.data, len(pr), ratio_test, sim.ctypes.data, loc.ctypes.data))
        return sim, loc

    def close(self) -> None:
        if self._idx:
            self._lib.cdvz_gpu_index_destroy(self._idx)
            self._idx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def container_slot(mode) -> int:
    m = mode if isinstance(mode, ModeSpec) else (mode_by_name(mode) if isinstance(mode, str) else mode_by_id(mode))
    return m.budget_bytes + 28


def parse_container_header(data: bytes) -> dict:
    """Header fields of a CDVZ1 container (container.cpp:60-93)."""
    if len(data) < 28 or data[:5] != b"CDVZ1":
        raise DataError("container magic mismatch")
    le = int.from_bytes
    return {
        "mode_id": data[5], "width": le(data[6:8], "little"), "height": le(data[8:10], "little"),
        "components": le(data[10:12], "little"), "model_crc": le(data[12:16], "little"),
        "global_len": le(data[16:20], "little"), "local_len": le(data[20:24], "little"),
        "crc": le(data[-4:], "little"),
    }


__all__ = [
    "Extractor", "ModeSpec", "MODES", "mode_by_name", "mode_by_id", "UsageError", "DataError", "InternalError",
    "bundle_check", "container_slot", "device_count", "parse_container_header", "library_path", "Index",
]
