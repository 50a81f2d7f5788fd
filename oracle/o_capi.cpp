// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Flat C entry points so the Python tests (and bench.py's cpu_baseline leg)
// can drive the oracle through ctypes. Errors return nonzero and leave a
// message in orc_last_error(): 1 usage, 2 data, 3 internal (the reference
// CLI's exit-code contract, proj/tools/cdvz.cpp:308-317).
#include <atomic>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>

#include "oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const UsageError& e) {
    g_err = e.what();
    return 1;
  } catch (const DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

struct Trace {
  EncodeTrace tr;
  Pyramid pyr;
  std::vector<uint8_t> container;
};

void put_kp(std::vector<double>& v, const Keypoint& k) {
  v.insert(v.end(), {k.x, k.y, k.sigma, double(k.octave), k.p, k.rho, k.p_ss, k.d});
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// synth_image(seed, w, h) quantised to bytes exactly like save_pgm.
int orc_synth_u8(uint64_t seed, int w, int h, uint8_t* out) {
  return guarded([&] {
    const auto bytes = plane_to_u8(synth_image(seed, w, h));
    std::memcpy(out, bytes.data(), bytes.size());
  });
}

// synth_image for frames base + i*golden, i in [0, count), on `threads` host threads.
int orc_synth_frames_u8(uint64_t base_seed, int count, int w, int h, int threads, uint8_t* out) {
  return guarded([&] {
    std::atomic<int> next{0};
    auto body = [&] {
      for (int i; (i = next.fetch_add(1)) < count;) {
        const auto bytes = plane_to_u8(synth_image(corpus_seed(base_seed, i), w, h));
        std::memcpy(out + std::size_t(i) * w * h, bytes.data(), bytes.size());
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(body);
    for (auto& t : pool) t.join();
  });
}

// train_model(synth_corpus(corpus_seed, count, w, h), {seed, gmm, em}) -> bundle text.
int orc_train_bundle(uint64_t corpus_base, int count, int w, int h, uint64_t seed, int gmm, int em,
                     char* out, size_t cap, size_t* out_len) {
  return guarded([&] {
    std::vector<Plane> corpus;
    for (int i = 0; i < count; ++i) corpus.push_back(synth_image(corpus_seed(corpus_base, i), w, h));
    TrainOptions o;
    o.seed = seed;
    o.gmm_components = gmm;
    o.em_iterations = em;
    const std::string text = serialize_model(train_model(corpus, o));
    *out_len = text.size();
    if (out && cap >= text.size()) std::memcpy(out, text.data(), text.size());
  });
}

// The oracle's detector beta of a bundle, row-major 4x4.
int orc_bundle_beta(const char* text, size_t len, double* out16) {
  return guarded([&] {
    const ModelBundle b = parse_model(std::string(text, len));
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) out16[i * 4 + j] = b.detector.beta[std::size_t(i)][std::size_t(j)];
  });
}

// Canonical re-serialisation and CRC of a bundle text (model_io.cpp:84).
int orc_bundle_crc(const char* text, size_t len, uint32_t* crc, int* components) {
  return guarded([&] {
    const ModelBundle b = parse_model(std::string(text, len));
    *crc = b.crc();
    *components = b.gmm.components();
  });
}

// encode_image on u8 pixels -> CDVZ1 container bytes; stage_ms[5] accumulates.
int orc_encode_u8(const char* bundle_text, size_t len, const uint8_t* px, int w, int h, size_t stride,
                  int mode_id, int max_side, uint8_t* out, size_t cap, size_t* out_len, double* stage_ms) {
  return guarded([&] {
    const ModelBundle b = parse_model(std::string(bundle_text, len));
    StageTimes st;
    const EncodedImage e = encode_image(plane_from_u8(px, w, h, stride), b, mode_by_id(mode_id), max_side, &st);
    const auto bytes = serialize_container(e);
    *out_len = bytes.size();
    if (cap < bytes.size()) throw DataError("output buffer too small");
    std::memcpy(out, bytes.data(), bytes.size());
    if (stage_ms)
      for (int i = 0; i < 5; ++i) stage_ms[i] += st.ms[i];
  });
}

// encode_image(load_image(P6)) on interleaved RGB bytes -> CDVZ1 container bytes.
int orc_encode_rgb(const char* bundle_text, size_t len, const uint8_t* rgb, int w, int h, size_t stride, int mode_id,
                   int max_side, uint8_t* out, size_t cap, size_t* out_len) {
  return guarded([&] {
    const ModelBundle b = parse_model(std::string(bundle_text, len));
    const EncodedImage e = encode_image(plane_from_rgb(rgb, w, h, stride), b, mode_by_id(mode_id), max_side, nullptr);
    const auto bytes = serialize_container(e);
    *out_len = bytes.size();
    if (cap < bytes.size()) throw DataError("output buffer too small");
    std::memcpy(out, bytes.data(), bytes.size());
  });
}

// synth_image(seed, w, h) as doubles (the unquantised GrayImage).
int orc_synth_f64(uint64_t seed, int w, int h, double* out) {
  return guarded([&] {
    const Plane p = synth_image(seed, w, h);
    std::memcpy(out, p.px.data(), sizeof(double) * p.px.size());
  });
}

// encode_image on an f64 GrayImage (validate() included) -> container bytes;
// norms (optional, cap nc) receives SCFVDescriptor::norms, *n_norms its size.
int orc_encode_f64(const char* bundle_text, size_t len, const double* px, int w, int h, int mode_id, int max_side,
                   uint8_t* out, size_t cap, size_t* out_len, double* norms, size_t norms_cap, size_t* n_norms) {
  return guarded([&] {
    const ModelBundle b = parse_model(std::string(bundle_text, len));
    Plane img;
    img.w = w;
    img.h = h;
    img.px.assign(px, px + std::size_t(w) * h);
    const EncodedImage e = encode_image(img, b, mode_by_id(mode_id), max_side, nullptr);
    const auto bytes = serialize_container(e);
    *out_len = bytes.size();
    if (cap < bytes.size()) throw DataError("output buffer too small");
    std::memcpy(out, bytes.data(), bytes.size());
    if (n_norms) *n_norms = e.global_desc.norms.size();
    if (norms && norms_cap >= e.global_desc.norms.size())
      std::memcpy(norms, e.global_desc.norms.data(), sizeof(double) * e.global_desc.norms.size());
  });
}

// The grey plane load_image makes of RGB bytes (image.cpp:82-86).
int orc_grey_rgb(const uint8_t* rgb, int w, int h, size_t stride, double* out) {
  return guarded([&] {
    const Plane p = plane_from_rgb(rgb, w, h, stride);
    std::memcpy(out, p.px.data(), sizeof(double) * p.px.size());
  });
}

// Frame-parallel batch encode (BASELINE.md CPU mode B): `threads` workers each
// running a single-threaded encode. out is count * slot bytes; lens[count].
int orc_encode_batch_u8(const char* bundle_text, size_t len, const uint8_t* px, int count, int w, int h,
                        int mode_id, int max_side, int threads, uint8_t* out, size_t slot, size_t* lens) {
  return guarded([&] {
    const ModelBundle b = parse_model(std::string(bundle_text, len));
    const ModeSpec& mode = mode_by_id(mode_id);
    std::atomic<int> next{0};
    std::atomic<int> failed{0};
    auto body = [&] {
      for (int i; (i = next.fetch_add(1)) < count;) {
        try {
          const auto bytes = serialize_container(
              encode_image(plane_from_u8(px + std::size_t(i) * w * h, w, h, std::size_t(w)), b, mode, max_side));
          lens[i] = bytes.size();
          if (bytes.size() <= slot) std::memcpy(out + std::size_t(i) * slot, bytes.data(), bytes.size());
        } catch (...) {
          lens[i] = 0;
          failed.fetch_add(1);
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(body);
    for (auto& t : pool) t.join();
    if (failed.load()) throw DataError("one or more frames failed to encode");
  });
}

// Full encode with every intermediate retained, for stage-level parity.
int orc_trace_u8(const char* bundle_text, size_t len, const uint8_t* px, int w, int h, int mode_id, int max_side,
                 void** handle) {
  return guarded([&] {
    const ModelBundle b = parse_model(std::string(bundle_text, len));
    auto t = std::make_unique<Trace>();
    const Plane img = plane_from_u8(px, w, h, std::size_t(w));
    const EncodedImage e = encode_image(img, b, mode_by_id(mode_id), max_side, nullptr, &t->tr);
    t->container = serialize_container(e);
    detect_keypoints(resize_max_side(img, max_side), b.detector, &t->pyr);
    *handle = t.release();
  });
}

void orc_trace_free(void* handle) { delete static_cast<Trace*>(handle); }

// Named trace arrays as flat doubles:
//   cand:<o>      x y sigma p                       per candidate of octave o
//   refined:<o>   x y sigma octave p rho p_ss d     per refined point of octave o
//   keypoints / selected                            (keypoint layout above)
//   oriented      keypoint layout + theta
//   descriptors   128 per oriented point
//   x gamma gm gv SCFV matrices (row-major)
//   gauss:<o>:<k> octave o level k raster
//   container     container bytes, one double per byte
//   dims          prep_w prep_h
int orc_trace_get(void* handle, const char* name, double* dst, size_t cap, size_t* n) {
  return guarded([&] {
    const Trace& t = *static_cast<Trace*>(handle);
    std::vector<double> v;
    std::string s(name);
    auto arg = [&](std::size_t pos) { return std::stoi(s.substr(pos)); };
    if (s.rfind("cand:", 0) == 0) {
      const int o = arg(5);
      if (o < int(t.tr.detect.candidates.size()))
        for (const auto& c : t.tr.detect.candidates[std::size_t(o)]) v.insert(v.end(), {double(c.x), double(c.y), c.sigma, c.p});
    } else if (s.rfind("refined:", 0) == 0) {
      const int o = arg(8);
      if (o < int(t.tr.detect.refined.size()))
        for (const auto& k : t.tr.detect.refined[std::size_t(o)]) put_kp(v, k);
    } else if (s == "keypoints") {
      for (const auto& k : t.tr.keypoints) put_kp(v, k);
    } else if (s == "selected") {
      for (const auto& k : t.tr.selected) put_kp(v, k);
    } else if (s == "oriented") {
      for (const auto& o : t.tr.oriented) { put_kp(v, o.pt); v.push_back(o.theta); }
    } else if (s == "descriptors") {
      for (const auto& d : t.tr.descriptors) v.insert(v.end(), d.v.begin(), d.v.end());
    } else if (s == "x") { v = t.tr.x.a; }
    else if (s == "gamma") { v = t.tr.gamma.a; }
    else if (s == "gm") { v = t.tr.gm.a; }
    else if (s == "gv") { v = t.tr.gv.a; }
    else if (s.rfind("gauss:", 0) == 0) {
      const auto c2 = s.find(':', 6);
      const int o = std::stoi(s.substr(6, c2 - 6)), k = std::stoi(s.substr(c2 + 1));
      if (o < int(t.pyr.octaves.size())) v = t.pyr.octaves[std::size_t(o)].gauss[std::size_t(k)].px;
    } else if (s == "container") {
      for (uint8_t c : t.container) v.push_back(c);
    } else if (s == "dims") {
      v = {double(t.tr.prep_w), double(t.tr.prep_h), double(t.pyr.octaves.size())};
    } else {
      throw UsageError("unknown trace array '" + s + "'");
    }
    *n = v.size();
    if (dst && cap >= v.size()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
  });
}

// retrieve(query, index) for nq queries over an index of n containers (all
// given as CDVZ1 bytes: blob + offsets[count+1]). Item ids are "idx%08d" so the
// reference's id tie-break is the index position. out_order / out_score are
// nq x n (item index, score) in ranked order.
int orc_retrieve(const uint8_t* index_blob, const size_t* index_off, int n, const uint8_t* query_blob,
                 const size_t* query_off, int nq, double ratio, int depth, int32_t* out_order, double* out_score) {
  return guarded([&] {
    std::vector<EncodedImage> items(std::size_t(std::max(0, n)));
    std::vector<std::pair<std::string, const EncodedImage*>> index;
    char id[32];
    for (int i = 0; i < n; ++i) {
      items[std::size_t(i)] = parse_container(std::vector<uint8_t>(index_blob + index_off[i], index_blob + index_off[i + 1]));
      std::snprintf(id, sizeof id, "idx%08d", i);
      index.emplace_back(id, &items[std::size_t(i)]);
    }
    MatchOptions opts;
    opts.ratio_test = ratio;
    opts.rerank_depth = depth;
    for (int q = 0; q < nq; ++q) {
      const EncodedImage query =
          parse_container(std::vector<uint8_t>(query_blob + query_off[q], query_blob + query_off[q + 1]));
      const RankedList list = retrieve(query, index, opts);
      for (std::size_t r = 0; r < list.items.size(); ++r) {
        out_order[std::size_t(q) * n + r] = std::stoi(list.items[r].id.substr(3));
        out_score[std::size_t(q) * n + r] = list.items[r].score;
      }
    }
  });
}

// match_pair(a, b) on two CDVZ1 containers.
int orc_match_pair(const uint8_t* a, size_t alen, const uint8_t* b, size_t blen, double ratio, double* global_sim,
                   int* local_matches) {
  return guarded([&] {
    MatchOptions opts;
    opts.ratio_test = ratio;
    const MatchResult r = match_pair(parse_container(std::vector<uint8_t>(a, a + alen)),
                                     parse_container(std::vector<uint8_t>(b, b + blen)), opts);
    *global_sim = r.global_similarity;
    *local_matches = r.local_match_count;
  });
}

}  // extern "C"
