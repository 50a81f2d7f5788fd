// TEST INFRASTRUCTURE ONLY — flat C entry points over the REFERENCE'S OWN
// sources (/root/reference/proj/src/*.cpp compiled against the Eigen-subset
// in oracle/refbuild/include), built into oracle/_ref/libref.so by
// oracle/refbuild/Makefile. Tests and bench.py's reference leg drive the
// reference through these: its encode_image / serialize_container / train_model
// / synth_image, with its own Engine (intra-frame worker threads) or frame
// parallelism on top. Errors: 1 UsageError, 2 DataError, 3 other (the
// reference CLI's exit codes, proj/tools/cdvz.cpp:308-317).
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "cdvz/common.hpp"
#include "cdvz/container.hpp"
#include "cdvz/descriptor.hpp"
#include "cdvz/image.hpp"
#include "cdvz/model_io.hpp"
#include "cdvz/parallel.hpp"
#include "cdvz/pipeline.hpp"
#include "cdvz/relevance.hpp"
#include "cdvz/scale_space.hpp"
#include "cdvz/synthetic.hpp"
#include "cdvz/transform_coding.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const cdvz::UsageError& e) {
    g_err = e.what();
    return 1;
  } catch (const cdvz::DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// load_image's PGM branch on bytes in memory (image.cpp:79-90).
cdvz::GrayImage from_u8(const uint8_t* px, int w, int h, size_t stride) {
  cdvz::GrayImage img = cdvz::make_image(w, h);
  const double inv = 1.0 / 255.0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) img.pix(y, x) = px[size_t(y) * stride + size_t(x)] * inv;
  return img;
}

cdvz::GrayImage from_f64(const double* px, int w, int h) {
  cdvz::GrayImage img = cdvz::make_image(w, h);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) img.pix(y, x) = px[size_t(y) * size_t(w) + size_t(x)];
  return img;
}

// One parsed bundle reused across calls with the same text.
const cdvz::ModelBundle& bundle_of(const char* text, size_t len) {
  thread_local std::string last;
  thread_local std::unique_ptr<cdvz::ModelBundle> cached;
  if (!cached || last.size() != len || std::memcmp(last.data(), text, len) != 0) {
    last.assign(text, len);
    cached = std::make_unique<cdvz::ModelBundle>(cdvz::parse_model(last));
  }
  return *cached;
}

void emit(const std::vector<uint8_t>& bytes, uint8_t* out, size_t cap, size_t* out_len) {
  *out_len = bytes.size();
  if (cap < bytes.size()) throw cdvz::DataError("output buffer too small");
  std::memcpy(out, bytes.data(), bytes.size());
}

void put_pt(std::vector<double>& v, const cdvz::InterestPoint& p) {
  v.insert(v.end(), {p.x, p.y, p.sigma, double(p.octave), p.p, p.rho, p.p_ss, p.d});
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// synth_image(seed, w, h) (synthetic.cpp:11-53) as doubles, and as bytes the
// way save_pgm writes them (image.cpp:95-105).
int ref_synth_f64(uint64_t seed, int w, int h, double* out) {
  return guarded([&] {
    const cdvz::GrayImage img = cdvz::synth_image(seed, w, h);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) out[size_t(y) * size_t(w) + size_t(x)] = img.pix(y, x);
  });
}
int ref_synth_u8(uint64_t seed, int w, int h, uint8_t* out) {
  return guarded([&] {
    const cdvz::GrayImage img = cdvz::synth_image(seed, w, h);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        out[size_t(y) * size_t(w) + size_t(x)] = static_cast<uint8_t>(std::lround(img.pix(y, x) * 255.0));
  });
}

// model_crc and component count of a bundle text (model_io.cpp:84, 141-273).
int ref_bundle_crc(const char* text, size_t len, uint32_t* crc, int* components) {
  return guarded([&] {
    const cdvz::ModelBundle& b = bundle_of(text, len);
    *crc = b.crc();
    *components = b.gmm.components();
  });
}

// serialize_model(parse_model(text)) — the canonical text the CRC covers.
int ref_bundle_canonical(const char* text, size_t len, char* out, size_t cap, size_t* out_len) {
  return guarded([&] {
    const std::string s = cdvz::serialize_model(bundle_of(text, len));
    *out_len = s.size();
    if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
  });
}

// The detector's beta of a bundle (compute_beta through FullPivLU,
// scale_space.cpp:56-73), row-major 4x4.
int ref_bundle_beta(const char* text, size_t len, double* out16) {
  return guarded([&] {
    const cdvz::ModelBundle& b = bundle_of(text, len);
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) out16[i * 4 + j] = b.detector.beta(i, j);
  });
}

// train_model(synth_corpus(corpus_base, count, w, h), {seed, gmm, em}) (pipeline.cpp:99-166).
int ref_train_bundle(uint64_t corpus_base, int count, int w, int h, uint64_t seed, int gmm, int em, int workers,
                     char* out, size_t cap, size_t* out_len) {
  return guarded([&] {
    cdvz::TrainOptions o;
    o.seed = seed;
    o.gmm_components = gmm;
    o.em_iterations = em;
    cdvz::Engine eng;
    eng.workers = workers;
    const std::string s = cdvz::serialize_model(cdvz::train_model(cdvz::synth_corpus(corpus_base, count, w, h), o, eng));
    *out_len = s.size();
    if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
  });
}

// encode_image + serialize_container on one 8-bit frame (PGM semantics), with
// Engine{workers} (0 = the reference default, hardware concurrency) and the
// reference's StageTimings accumulated into stage_ms[5] when given.
int ref_encode_u8(const char* text, size_t len, const uint8_t* px, int w, int h, size_t stride, int mode_id,
                  int max_side, int workers, uint8_t* out, size_t cap, size_t* out_len, double* stage_ms) {
  return guarded([&] {
    const cdvz::ModelBundle& b = bundle_of(text, len);
    cdvz::Engine eng;
    eng.workers = workers;
    cdvz::StageTimings st;
    cdvz::EncodeOptions opts;
    opts.max_side = max_side;
    const auto enc = cdvz::encode_image(from_u8(px, w, h, stride), b, cdvz::mode_by_id(mode_id), eng,
                                        stage_ms ? &st : nullptr, opts);
    emit(cdvz::serialize_container(enc), out, cap, out_len);
    if (stage_ms) {
      const char* labels[5] = {"detection", "selection", "description", "compression", "aggregation"};
      for (const auto& e : st.entries())
        for (int i = 0; i < 5; ++i)
          if (e.stage == labels[i]) stage_ms[i] += e.total_ms;
    }
  });
}

// encode_image on an f64 GrayImage; norms receives SCFVDescriptor::norms.
int ref_encode_f64(const char* text, size_t len, const double* px, int w, int h, int mode_id, int max_side,
                   uint8_t* out, size_t cap, size_t* out_len, double* norms, size_t norms_cap, size_t* n_norms) {
  return guarded([&] {
    const cdvz::ModelBundle& b = bundle_of(text, len);
    cdvz::Engine eng;
    eng.workers = 1;
    cdvz::EncodeOptions opts;
    opts.max_side = max_side;
    const auto enc = cdvz::encode_image(from_f64(px, w, h), b, cdvz::mode_by_id(mode_id), eng, nullptr, opts);
    emit(cdvz::serialize_container(enc), out, cap, out_len);
    if (n_norms) *n_norms = enc.global_desc.norms.size();
    if (norms && norms_cap >= enc.global_desc.norms.size())
      std::memcpy(norms, enc.global_desc.norms.data(), sizeof(double) * enc.global_desc.norms.size());
  });
}

// Batch of `count` 8-bit frames: `threads` frames in flight, each encoded with
// Engine{workers} (BASELINE.md CPU mode A: threads 1, workers nproc; mode B:
// threads nproc, workers 1). Containers at out + i * slot, lengths in lens.
int ref_encode_batch_u8(const char* text, size_t len, const uint8_t* px, int count, int w, int h, int mode_id,
                        int max_side, int threads, int workers, uint8_t* out, size_t slot, size_t* lens) {
  return guarded([&] {
    const std::string bundle_text(text, len);
    const cdvz::ModelBundle b = cdvz::parse_model(bundle_text);
    const cdvz::ModeSpec& mode = cdvz::mode_by_id(mode_id);
    std::atomic<int> next{0}, failed{0};
    auto body = [&] {
      cdvz::Engine eng;
      eng.workers = workers;
      cdvz::EncodeOptions opts;
      opts.max_side = max_side;
      for (int i; (i = next.fetch_add(1)) < count;) {
        try {
          const auto bytes = cdvz::serialize_container(
              cdvz::encode_image(from_u8(px + size_t(i) * size_t(w) * size_t(h), w, h, size_t(w)), b, mode, eng, nullptr, opts));
          lens[i] = bytes.size();
          if (bytes.size() <= slot) std::memcpy(out + size_t(i) * slot, bytes.data(), bytes.size());
        } catch (...) {
          lens[i] = 0;
          failed.fetch_add(1);
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(body);
    for (auto& t : pool) t.join();
    if (failed.load()) throw cdvz::DataError("one or more frames failed to encode");
  });
}

// Stage outputs of extract (pipeline.cpp:14-35) for one 8-bit frame, as flat
// doubles: "keypoints" (after dedup), "selected", "oriented" (keypoint layout
// + theta) and "descriptors" (128 per oriented point). Point layout:
// x y sigma octave p rho p_ss d.
int ref_stages_u8(const char* text, size_t len, const uint8_t* px, int w, int h, int max_side, const char* name,
                  double* dst, size_t cap, size_t* n) {
  return guarded([&] {
    const cdvz::ModelBundle& b = bundle_of(text, len);
    const cdvz::GrayImage prepared = cdvz::resize_max_side(from_u8(px, w, h, size_t(w)), max_side);
    cdvz::Pyramid pyr;
    cdvz::Engine eng;
    eng.workers = 1;
    auto points = cdvz::detect_keypoints(prepared, b.detector, &pyr, eng);
    cdvz::fill_center_distance(points, prepared.width(), prepared.height());
    std::vector<double> v;
    const std::string s(name);
    if (s == "keypoints") {
      for (const auto& p : points) put_pt(v, p);
    } else {
      const auto sel = cdvz::select_top(points, b.relevance, static_cast<std::size_t>(b.select_n));
      if (s == "selected") {
        for (const auto& p : sel) put_pt(v, p);
      } else {
        const auto oriented = cdvz::assign_orientations(pyr, b.detector.sigmas, sel, eng);
        if (s == "oriented") {
          for (const auto& o : oriented) {
            put_pt(v, o.pt);
            v.push_back(o.theta);
          }
        } else if (s == "descriptors") {
          for (const auto& d : cdvz::describe_batch(pyr, b.detector.sigmas, oriented, eng))
            for (int i = 0; i < 128; ++i) v.push_back(d.values[i]);
        } else {
          throw cdvz::UsageError("unknown stage '" + s + "'");
        }
      }
    }
    *n = v.size();
    if (dst && cap >= v.size()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
  });
}

}  // extern "C"
