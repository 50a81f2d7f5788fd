"""GPU parity of compressed-domain matching and retrieval:
cdvz_gpu_retrieve / cdvz_gpu_match_pairs against the oracle's restatement of
retrieve / match_pair / count_local_matches (proj/src/eval.cpp:17-124), on
containers the extractor emits. Bar: identical ranked item order and
bit-identical scores (integer distances and the reference's double formulas)."""
import numpy as np
import pytest

import oracle_lib

pytestmark = pytest.mark.gpu

cg = pytest.importorskip("paper_1705_09776_b200")


def _containers(ex, seed, count, mode, w=640, h=480):
    frames = oracle_lib.synth_frames(seed, count, w, h)
    blobs, status = ex.encode_batch(frames, mode)
    assert all(s == 0 for s in status)
    return blobs


@pytest.fixture(scope="module")
def ex_b8(bundle_b8):
    ex = cg.Extractor(bundle_b8, max_batch=64)
    yield ex
    ex.close()


@pytest.fixture(scope="module")
def corpus_4k(ex_b8):
    return _containers(ex_b8, 7000, 40, "4K")


@pytest.mark.parametrize("depth,ratio", [(50, 0.85), (3, 0.85), (0, 0.85), (10, 0.7)])
def test_retrieve_matches_oracle(corpus_4k, depth, ratio):
    index = corpus_4k[:32]
    queries = corpus_4k[28:40]  # 4 indexed images, 8 unseen ones
    idx = cg.Index(index)
    got_i, got_s = idx.retrieve_batch(queries, ratio, depth)
    want_i, want_s = oracle_lib.retrieve(index, queries, ratio, depth)
    idx.close()
    assert np.array_equal(got_i, want_i)
    assert np.array_equal(got_s, want_s)


def test_retrieve_query_chunks_match_one_pass(corpus_4k, monkeypatch):
    """Query batches run in chunks (so queries x items never overflows the
    sort's int offsets); chunks of 5 queries give the single-pass result."""
    index, queries = corpus_4k[:32], corpus_4k[20:40]
    idx = cg.Index(index)
    want_i, want_s = idx.retrieve_batch(queries, 0.85, 10)
    monkeypatch.setenv("CDVZ_GPU_RETRIEVE_QCHUNK", "5")
    got_i, got_s = idx.retrieve_batch(queries, 0.85, 10)
    idx.close()
    assert np.array_equal(got_i, want_i) and np.array_equal(got_s, want_s)


def test_retrieve_into_pinned_buffers(corpus_4k, ex_b8):
    """retrieve_batch(out=...) fills caller-provided (pinned) arrays with the
    same ranked lists (here the whole index is re-ranked); bad
    shapes / dtypes are a UsageError."""
    index, queries = corpus_4k[:40], corpus_4k[30:40]
    idx = cg.Index(index)
    want_i, want_s = idx.retrieve_batch(queries, 0.85, 300)  # head = all 40 items
    nq, n = len(queries), len(index)
    pin_i, pin_s = ex_b8.pinned_buffer(4 * nq * n), ex_b8.pinned_buffer(8 * nq * n)
    out = (pin_i.array.view(np.int32).reshape(nq, n), pin_s.array.view(np.float64).reshape(nq, n))
    got_i, got_s = idx.retrieve_batch(queries, 0.85, 300, out=out)
    assert got_i is out[0] and got_s is out[1]
    assert np.array_equal(got_i, want_i) and np.array_equal(got_s, want_s)
    oracle_i, oracle_s = oracle_lib.retrieve(index, queries, 0.85, 300)
    assert np.array_equal(got_i, oracle_i) and np.array_equal(got_s, oracle_s)
    with pytest.raises(cg.UsageError):
        idx.retrieve_batch(queries, 0.85, 300, out=(out[0][:, :5], out[1]))
    idx.close()


def test_indexed_image_retrieves_itself_first(corpus_4k):
    """test_pipeline.cpp:164-170 on the GPU."""
    idx = cg.Index(corpus_4k[:16], ids=[f"img{i}" for i in range(16)])
    for i in range(16):
        ranked = idx.retrieve(corpus_4k[i])
        assert ranked[0][0] == f"img{i}"
        assert all(ranked[k][1] <= ranked[k - 1][1] for k in range(1, len(ranked)))
    idx.close()


def test_max_results_truncates_the_ranking(corpus_4k):
    idx = cg.Index(corpus_4k[:20])
    full_i, full_s = idx.retrieve_batch(corpus_4k[:3], rerank_depth=5)
    top_i, top_s = idx.retrieve_batch(corpus_4k[:3], rerank_depth=5, max_results=7)
    assert np.array_equal(top_i, full_i[:, :7]) and np.array_equal(top_s, full_s[:, :7])
    idx.close()


def test_ties_break_on_ids(corpus_4k):
    """Equal scores order by id ascending (eval.cpp:91-94, :107-112)."""
    dup = [corpus_4k[0], corpus_4k[0], corpus_4k[1]]
    ranked = cg.Index(dup, ids=["b", "a", "c"]).retrieve(corpus_4k[0], rerank_depth=0)
    assert [r[0] for r in ranked[:2]] == ["a", "b"]
    ranked = cg.Index(dup, ids=["a", "b", "c"]).retrieve(corpus_4k[0], rerank_depth=3)
    assert [r[0] for r in ranked[:2]] == ["a", "b"]


def test_match_pairs_match_oracle(corpus_4k):
    index = corpus_4k[:12]
    queries = corpus_4k[10:16]
    pairs = [(q, i) for q in range(len(queries)) for i in range(len(index))]
    idx = cg.Index(index)
    sim, loc = idx.match_pairs(queries, pairs)
    for k, (q, i) in enumerate(pairs):
        ws, wl = oracle_lib.match_pair(queries[q], index[i])
        assert sim[k] == ws and loc[k] == wl, (q, i)
    idx.close()


def test_self_match_kat(corpus_4k):
    """test_pipeline.cpp:110-117: global similarity 1, every code matched."""
    idx = cg.Index(corpus_4k[:1])
    sim, loc = idx.match_pairs(corpus_4k[:1], [(0, 0)])
    hdr = cg.parse_container_header(corpus_4k[0])
    local = corpus_4k[0][24 + hdr["global_len"]:24 + hdr["global_len"] + hdr["local_len"]]
    n_codes = local[2] | (local[3] << 8)
    assert sim[0] == 1.0 and loc[0] == n_codes and n_codes > 20
    idx.close()


@pytest.mark.parametrize("mode", ["16K", "512B"])
def test_retrieve_b512_and_other_modes(bundle_b512, mode):
    ex = cg.Extractor(bundle_b512, max_batch=32)
    blobs = _containers(ex, 7100, 20, mode, 480, 360)
    ex.close()
    idx = cg.Index(blobs[:16])
    got_i, got_s = idx.retrieve_batch(blobs[12:20], 0.85, 8)
    want_i, want_s = oracle_lib.retrieve(blobs[:16], blobs[12:20], 0.85, 8)
    idx.close()
    assert np.array_equal(got_i, want_i) and np.array_equal(got_s, want_s)


def test_decoder_rejects_what_parse_container_rejects(corpus_4k):
    good = corpus_4k[:4]
    with pytest.raises(cg.DataError):
        cg.Index([])
    bad_crc = bytearray(good[1])
    bad_crc[30] ^= 0x40
    with pytest.raises(cg.DataError, match="item 1: container checksum mismatch"):
        cg.Index([good[0], bytes(bad_crc)])
    with pytest.raises(cg.DataError, match="truncated"):
        cg.Index([good[0], good[1][:20]])
    bad_magic = b"CDVZ2" + good[2][5:]
    with pytest.raises(cg.DataError, match="magic"):
        cg.Index([bad_magic])


def test_bundle_and_mode_mismatches_are_rejected(ex_b8, bundle_b512, corpus_4k):
    idx = cg.Index(corpus_4k[:4])
    other_mode = _containers(ex_b8, 7200, 1, "1K")
    with pytest.raises(cg.DataError, match="mode"):
        idx.retrieve_batch(other_mode)
    ex = cg.Extractor(bundle_b512, max_batch=4)
    other_bundle = _containers(ex, 7201, 1, "4K")
    ex.close()
    with pytest.raises(cg.DataError, match="model bundle"):
        idx.match_pairs(other_bundle, [(0, 0)])
    with pytest.raises(cg.DataError, match="model bundle"):
        cg.Index(corpus_4k[:2] + other_bundle)
    idx.close()


def test_cpp_retrieval_example_matches_python(corpus_4k, tmp_path):
    """examples/retrieve.cpp ranks like Index.retrieve (ids = file paths)."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "retrieve"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(root, "examples", "retrieve.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    paths = []
    for i, blob in enumerate(corpus_4k[:6]):
        p = tmp_path / f"c{i}.cdvz"
        p.write_bytes(blob)
        paths.append(str(p))
    out = subprocess.run([str(exe), paths[2], "--"] + paths, capture_output=True, text=True, check=True).stdout
    got = [(tok.rsplit(":", 1)[0], float(tok.rsplit(":", 1)[1])) for tok in out.split()[1:]]
    want = cg.Index(corpus_4k[:6], ids=paths).retrieve(corpus_4k[2])
    assert [g[0] for g in got] == [w[0] for w in want]
    assert all(abs(g[1] - w[1]) <= 1e-9 * max(1.0, abs(w[1])) for g, w in zip(got, want))


def test_cpp_match_example_matches_python(corpus_4k, tmp_path):
    """examples/match.cpp prints the reference CLI's two lines
    (cdvz.cpp:82-89): format_double of global_similarity and the local match
    count, equal to Index.match_pairs for the same pair."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "match"
    lib_dir = os.path.dirname(cg.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(root, "examples", "match.cpp"), f"-L{lib_dir}",
                    "-lcdvz_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)

    def fmt(v):
        for prec in range(1, 18):
            s = "%.*g" % (prec, v)
            if float(s) == v:
                return s
        return "%.17g" % v

    for qa, qb in [(0, 1), (2, 2), (5, 30)]:
        (tmp_path / "a.cdvz").write_bytes(corpus_4k[qa])
        (tmp_path / "b.cdvz").write_bytes(corpus_4k[qb])
        p = subprocess.run([str(exe), str(tmp_path / "a.cdvz"), str(tmp_path / "b.cdvz")], capture_output=True,
                           text=True)
        assert p.returncode == 0, p.stderr
        idx = cg.Index([corpus_4k[qb]])
        sim, loc = idx.match_pairs([corpus_4k[qa]], [(0, 0)])
        idx.close()
        assert p.stdout == f"global_similarity {fmt(float(sim[0]))}\nlocal_match_count {int(loc[0])}\n"
