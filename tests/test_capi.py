"""CPU: the C ABI library loads, exports every entry point include/cdvz_gpu.h
declares, and refuses to run without a B200 (no CPU fallback)."""
import ctypes
import os
import re

import pytest

import paper_1705_09776_b200 as cg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "cdvz_gpu.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(cdvz_gpu_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("cdvz_gpu_create", "cdvz_gpu_encode_batch", "cdvz_gpu_encode_device", "cdvz_gpu_stage_times",
                 "cdvz_gpu_last_error", "cdvz_gpu_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(cg.library_path())
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", cg.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with open(os.path.join(ROOT, "tests", "golden", "bundle_b8.txt")) as f:
        text = f.read()
    with pytest.raises(cg.InternalError, match="CUDA device"):
        cg.Extractor(text)


def test_mode_table_and_errors():
    assert [m.budget_bytes for m in cg.MODES] == [512, 1024, 2048, 4096, 8192, 16384]
    assert cg.mode_by_name("4K").elements == 103 and cg.mode_by_name("16K").elements == 128
    with pytest.raises(cg.UsageError):
        cg.mode_by_name("3K")
    with pytest.raises(cg.DataError):
        cg.mode_by_id(99)
    assert cg.container_slot("4K") == 4124


def test_container_slot_from_the_library():
    lib = ctypes.CDLL(cg.library_path())
    lib.cdvz_gpu_container_slot.restype = ctypes.c_size_t
    assert [lib.cdvz_gpu_container_slot(i) for i in range(6)] == [540, 1052, 2076, 4124, 8220, 16412]
    assert lib.cdvz_gpu_container_slot(7) == 0


def test_cpp_shim_compiles_and_validates_bundles(tmp_path):
    """The reference-shaped C++ API over the ABI builds and links against the
    library; bundle validation works host-side (no GPU)."""
    import subprocess

    exe = tmp_path / "extract"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "examples", "extract.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    bad = tmp_path / "bad.txt"
    bad.write_text("CDVZ-MODEL 2\nend\n")
    p = subprocess.run([str(exe), str(bad), "4K", "x.pgm", "y.cdvz"], capture_output=True, text=True)
    assert p.returncode == 2 and "version" in p.stderr
    good = os.path.join(ROOT, "tests", "golden", "bundle_b8.txt")
    p = subprocess.run([str(exe), good, "3K", "x.pgm", "y.cdvz"], capture_output=True, text=True)
    assert p.returncode == 1 and "unknown mode" in p.stderr


def test_cpp_retrieval_shim_compiles_and_links(tmp_path):
    """examples/retrieve.cpp (the reference's run_retrieve over the shim)
    builds against the library; without arguments it is a usage error."""
    import subprocess

    exe = tmp_path / "retrieve"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "examples", "retrieve.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    p = subprocess.run([str(exe)], capture_output=True, text=True)
    assert p.returncode == 1 and "usage" in p.stderr


def test_cpp_train_shim_compiles_and_checks_the_corpus(tmp_path):
    """examples/train.cpp (the reference CLI's run_train over the shim) builds;
    list_images' and train_model's corpus errors surface before any device
    work: not a directory (usage), no images / fewer than 20 (data)."""
    import subprocess

    exe = tmp_path / "train"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "examples", "train.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    p = subprocess.run([str(exe), str(tmp_path / "missing"), "b.txt"], capture_output=True, text=True)
    assert p.returncode == 1 and "not a directory" in p.stderr
    corpus = tmp_path / "corpus"
    corpus.mkdir()
    p = subprocess.run([str(exe), str(corpus), "b.txt"], capture_output=True, text=True)
    assert p.returncode == 2 and "no .pgm/.ppm" in p.stderr
    for i in range(3):
        (corpus / f"{i}.pgm").write_bytes(b"P5\n16 16\n255\n" + bytes(256))
    p = subprocess.run([str(exe), str(corpus), "b.txt"], capture_output=True, text=True)
    assert p.returncode == 2 and "at least 20" in p.stderr


def test_cpp_stream_shim_compiles(tmp_path):
    """examples/stream.cpp (the shim's submit_batch / PendingBatch) builds;
    without arguments it is a usage error."""
    import subprocess

    exe = tmp_path / "stream"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "examples", "stream.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    p = subprocess.run([str(exe)], capture_output=True, text=True)
    assert p.returncode == 1 and "usage" in p.stderr


def test_cpp_match_shim_compiles(tmp_path):
    """examples/match.cpp (the reference CLI's match over the shim) builds;
    without arguments it is a usage error, a missing file a data error."""
    import subprocess

    exe = tmp_path / "match"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "examples", "match.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    p = subprocess.run([str(exe)], capture_output=True, text=True)
    assert p.returncode == 1 and "usage" in p.stderr
    p = subprocess.run([str(exe), str(tmp_path / "a.cdvz"), str(tmp_path / "b.cdvz")], capture_output=True, text=True)
    assert p.returncode == 2 and "cannot open" in p.stderr
