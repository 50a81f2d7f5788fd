// cdvz_gpu.hpp — header-only C++ shim over include/cdvz_gpu.h that mirrors the
// reference's extraction API (proj/include/cdvz/pipeline.hpp:14-20,
// container.hpp:27, model_io.hpp:30-33, transform_coding.hpp:22-24,
// parallel.hpp:117-134) for C++ callers:
//
//   reference                                        this shim
//   ModelBundle load_model(path)                     cdvz::gpu::ModelBundle::load(path)
//   const ModeSpec& mode_by_name(name)               cdvz::gpu::mode_by_name(name)
//   EncodedImage encode_image(img, bundle, mode,     EncodedImage cdvz::gpu::encode_image(
//       Engine, StageTimings*, EncodeOptions)            img, bundle, mode, Engine, StageTimings*, EncodeOptions)
//                                                    (GrayImage of doubles, the same signature)
//   serialize_container(enc) / parse_container(b)    cdvz::gpu::serialize_container / parse_container
//   (8-bit / PGM / PPM / batch fast paths)           encode_image(GrayImage8 | PnmImage, ...) -> CDVZ1 bytes,
//                                                    encode_batch(frames, ...) over one or several GPUs
//   RankedList retrieve(query, id, index, opts)      cdvz::gpu::retrieve({(id, bytes)...}, Index, opts)
//   MatchResult match_pair(a, b, opts)               cdvz::gpu::match_pair(a_bytes, Index, item, opts)
//
// GrayImage holds the reference's doubles in [0, 1] (image.hpp:11-18); the
// byte fast paths take 8-bit rasters read as b/255 (load_image,
// image.cpp:79-87). Errors keep the reference's exception types: UsageError
// (bad mode name), DataError (bad raster / bundle), std::runtime_error for
// device failures (the CLI's exit code 3). The Engine argument has no GPU
// meaning (results never depend on it, parallel.hpp:16-18) and is ignored.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cdvz_gpu.h"

namespace cdvz {
namespace gpu {

struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void raise_for(int code, const char* msg) {
  if (code == CDVZ_GPU_OK) return;
  if (code == CDVZ_GPU_USAGE) throw UsageError(msg);
  if (code == CDVZ_GPU_DATA) throw DataError(msg);
  throw std::runtime_error(msg);
}
// raise_for with the context's last error, read after `code` is computed (the
// message must not be an argument evaluated alongside the call).
inline void check(int code, const cdvz_gpu_ctx* ctx = nullptr) {
  if (code != CDVZ_GPU_OK) raise_for(code, cdvz_gpu_last_error(ctx));
}
inline void check_index(int code, const cdvz_gpu_index* idx) {
  if (code != CDVZ_GPU_OK) raise_for(code, cdvz_gpu_index_last_error(idx));
}

struct ModeSpec {  // transform_coding.hpp:13-20
  int id;
  const char* name;
  std::size_t budget_bytes;
  int elements;
  double scfv_fraction;
  bool variance_planes;
};

inline const ModeSpec* default_modes() {
  static const ModeSpec modes[6] = {
      {0, "512B", 512, 20, 32.0 / 512.0, false},  {1, "1K", 1024, 32, 64.0 / 512.0, false},
      {2, "2K", 2048, 64, 128.0 / 512.0, false},  {3, "4K", 4096, 103, 256.0 / 512.0, false},
      {4, "8K", 8192, 103, 320.0 / 512.0, true},  {5, "16K", 16384, 128, 512.0 / 512.0, true},
  };
  return modes;
}

inline const ModeSpec& mode_by_name(const std::string& name) {
  for (int i = 0; i < 6; ++i)
    if (name == default_modes()[i].name) return default_modes()[i];
  throw UsageError("unknown mode '" + name + "' (expected 512B, 1K, 2K, 4K, 8K or 16K)");
}

inline const ModeSpec& mode_by_id(int id) {
  for (int i = 0; i < 6; ++i)
    if (default_modes()[i].id == id) return default_modes()[i];
  throw DataError("unknown mode id " + std::to_string(id));
}

struct GrayImage8 {  // GrayImage (image.hpp:14-18) as bytes
  int width = 0, height = 0;
  std::vector<uint8_t> pix;  // row-major, width * height
};

struct EncodeOptions {  // pipeline.hpp:14-16
  int max_side = 640;
};

struct Engine {  // parallel.hpp:19-23 — accepted for signature parity; the GPU's results never depend on it
  int workers = 0;
  int tile_size = 32;
};

struct GrayImage {  // image.hpp:14-18: row-major doubles in [0, 1], rows = height
  int w = 0, h = 0;
  std::vector<double> pix;
  int width() const { return w; }
  int height() const { return h; }
  double& operator()(int y, int x) { return pix[std::size_t(y) * std::size_t(w) + std::size_t(x)]; }
  double operator()(int y, int x) const { return pix[std::size_t(y) * std::size_t(w) + std::size_t(x)]; }
};

inline GrayImage make_image(int width, int height, double fill = 0.0) {  // image.cpp:40-44
  GrayImage img;
  img.w = width;
  img.h = height;
  img.pix.assign(std::size_t(std::max(0, width)) * std::size_t(std::max(0, height)), fill);
  return img;
}

struct TernaryCode {  // transform_coding.hpp:56-62
  std::uint16_t xq = 0, yq = 0;
  std::uint8_t sigma_q = 0;
  std::uint8_t theta_q = 0;
  std::uint8_t mode = 0;
  std::vector<std::int8_t> symbols;
};

struct SCFVDescriptor {  // scfv.hpp:30-40
  int n_components = 0;
  bool has_variance = false;
  std::vector<std::uint8_t> mask;
  std::vector<std::uint32_t> mean_planes;
  std::vector<std::uint32_t> var_planes;
  std::vector<double> norms;  // scfv_delta of each selected component (not serialized)
  bool selected(int c) const { return (mask[std::size_t(c / 8)] >> (c % 8)) & 1u; }
  int popcount() const {
    int n = 0;
    for (auto b : mask) n += __builtin_popcount(b);
    return n;
  }
};

struct EncodedImage {  // container.hpp:19-25
  int mode_id = 0;
  int width = 0, height = 0;
  std::uint32_t model_crc = 0;
  SCFVDescriptor global_desc;
  std::vector<TernaryCode> codes;
};

namespace detail {
inline std::uint32_t crc32(const std::uint8_t* p, std::size_t n) {  // common.cpp:11-35
  static const auto table = [] {
    std::vector<std::uint32_t> t(256);
    for (std::uint32_t i = 0; i < 256; ++i) {
      std::uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[i] = c;
    }
    return t;
  }();
  std::uint32_t c = 0xFFFFFFFFu;
  for (std::size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}
inline void put16(std::vector<std::uint8_t>& o, std::uint32_t v) {
  o.push_back(std::uint8_t(v & 0xFF));
  o.push_back(std::uint8_t((v >> 8) & 0xFF));
}
inline void put32(std::vector<std::uint8_t>& o, std::uint32_t v) {
  put16(o, v & 0xFFFF);
  put16(o, v >> 16);
}
inline std::uint32_t get16(const std::vector<std::uint8_t>& b, std::size_t o) { return b[o] | (std::uint32_t(b[o + 1]) << 8); }
inline std::uint32_t get32(const std::vector<std::uint8_t>& b, std::size_t o) { return get16(b, o) | (get16(b, o + 2) << 16); }
}  // namespace detail

// serialize_container (container.cpp:32-58) with serialize_scfv
// (scfv.cpp:285-298) and pack_local (transform_coding.cpp:232-270).
inline std::vector<std::uint8_t> serialize_container(const EncodedImage& enc) {
  const ModeSpec& mode = mode_by_id(enc.mode_id);
  std::vector<std::uint8_t> global(enc.global_desc.mask);
  for (std::size_t r = 0; r < enc.global_desc.mean_planes.size(); ++r) {
    detail::put32(global, enc.global_desc.mean_planes[r]);
    if (enc.global_desc.has_variance) detail::put32(global, enc.global_desc.var_planes[r]);
  }
  if (enc.codes.size() > 0xFFFF) throw DataError("too many codes for one local block");
  std::vector<std::uint8_t> local{std::uint8_t(mode.id), std::uint8_t(mode.elements)};
  detail::put16(local, std::uint32_t(enc.codes.size()));
  for (const auto& c : enc.codes) {
    if (c.mode != mode.id) throw DataError("code mode does not match block mode");
    if (c.symbols.size() != std::size_t(mode.elements)) throw DataError("code symbol count does not match block mode");
    detail::put16(local, c.xq);
    detail::put16(local, c.yq);
    local.push_back(c.sigma_q);
    local.push_back(c.theta_q);
    std::uint8_t packed = 0;
    int filled = 0;
    for (std::int8_t sym : c.symbols) {
      if (sym < -1 || sym > 1) throw DataError("symbol outside {-1, 0, +1}");
      packed |= std::uint8_t((sym == 0 ? 0 : sym == 1 ? 1 : 2) << (2 * filled));
      if (++filled == 4) {
        local.push_back(packed);
        packed = 0;
        filled = 0;
      }
    }
    if (filled > 0) local.push_back(packed);
  }
  if (global.size() + local.size() > mode.budget_bytes) throw DataError("encoded payload exceeds the mode budget");
  if (enc.width < 1 || enc.width > 0xFFFF || enc.height < 1 || enc.height > 0xFFFF)
    throw DataError("image dimensions do not fit the container header");
  if (enc.global_desc.n_components < 1 || enc.global_desc.n_components > 0xFFFF)
    throw DataError("component count does not fit the container header");
  std::vector<std::uint8_t> out{'C', 'D', 'V', 'Z', '1', std::uint8_t(enc.mode_id)};
  detail::put16(out, std::uint32_t(enc.width));
  detail::put16(out, std::uint32_t(enc.height));
  detail::put16(out, std::uint32_t(enc.global_desc.n_components));
  detail::put32(out, enc.model_crc);
  detail::put32(out, std::uint32_t(global.size()));
  detail::put32(out, std::uint32_t(local.size()));
  out.insert(out.end(), global.begin(), global.end());
  out.insert(out.end(), local.begin(), local.end());
  detail::put32(out, detail::crc32(out.data(), out.size()));
  return out;
}

// parse_container (container.cpp:60-93) with parse_scfv (scfv.cpp:300-326)
// and unpack_local (transform_coding.cpp:272-305), the same checks.
inline EncodedImage parse_container(const std::vector<std::uint8_t>& bytes) {
  if (bytes.size() < 28) throw DataError("container truncated");
  static const char magic[5] = {'C', 'D', 'V', 'Z', '1'};
  for (int i = 0; i < 5; ++i)
    if (bytes[std::size_t(i)] != std::uint8_t(magic[i])) throw DataError("container magic mismatch");
  const std::size_t body = bytes.size() - 4;
  if (detail::crc32(bytes.data(), body) != detail::get32(bytes, body)) throw DataError("container checksum mismatch");
  EncodedImage enc;
  enc.mode_id = bytes[5];
  const ModeSpec& mode = mode_by_id(enc.mode_id);
  enc.width = int(detail::get16(bytes, 6));
  enc.height = int(detail::get16(bytes, 8));
  const int nc = int(detail::get16(bytes, 10));
  enc.model_crc = detail::get32(bytes, 12);
  const std::size_t glen = detail::get32(bytes, 16), llen = detail::get32(bytes, 20);
  if (24 + glen + llen != body) throw DataError("container section lengths disagree with its size");
  SCFVDescriptor& d = enc.global_desc;
  d.n_components = nc;
  d.has_variance = mode.variance_planes;
  const std::size_t mask_bytes = std::size_t((nc + 7) / 8);
  if (glen < mask_bytes) throw DataError("global descriptor block truncated");
  d.mask.assign(bytes.begin() + 24, bytes.begin() + 24 + long(mask_bytes));
  const int sel = d.popcount();
  if (glen != mask_bytes + std::size_t(sel) * (d.has_variance ? 8 : 4))
    throw DataError("global descriptor length does not match its mask");
  std::size_t off = 24 + mask_bytes;
  for (int r = 0; r < sel; ++r) {
    d.mean_planes.push_back(detail::get32(bytes, off));
    off += 4;
    if (d.has_variance) {
      d.var_planes.push_back(detail::get32(bytes, off));
      off += 4;
    }
  }
  const std::size_t lb = 24 + glen;
  if (llen < 4) throw DataError("local block truncated");
  const int lmode = bytes[lb], elements = bytes[lb + 1];
  const std::size_t count = detail::get16(bytes, lb + 2);
  if (lmode > 5) throw DataError("local block has an unknown mode id");
  if (elements < 1 || elements > 128) throw DataError("local block has an invalid element count");
  const std::size_t per = 6 + (std::size_t(elements) * 2 + 7) / 8;
  if (llen != 4 + count * per) throw DataError("local block length does not match its header");
  off = lb + 4;
  enc.codes.resize(count);
  for (auto& c : enc.codes) {
    c.mode = std::uint8_t(lmode);
    c.xq = std::uint16_t(detail::get16(bytes, off));
    c.yq = std::uint16_t(detail::get16(bytes, off + 2));
    c.sigma_q = bytes[off + 4];
    c.theta_q = bytes[off + 5];
    off += 6;
    c.symbols.resize(std::size_t(elements));
    for (int i = 0; i < elements; ++i) {
      const unsigned bits = (bytes[off + std::size_t(i / 4)] >> (2 * (i % 4))) & 3u;
      if (bits == 3) throw DataError("reserved symbol pattern in local block");
      c.symbols[std::size_t(i)] = std::int8_t(bits == 0 ? 0 : bits == 1 ? 1 : -1);
    }
    off += (std::size_t(elements) * 2 + 7) / 8;
  }
  return enc;
}

class StageTimings {  // parallel.hpp:117-134: device ms per label
 public:
  struct Entry { std::string stage; long long calls = 0; double total_ms = 0.0; };
  void add(const std::string& stage, double ms) {
    for (auto& e : entries_)
      if (e.stage == stage) { e.calls += 1; e.total_ms += ms; return; }
    entries_.push_back({stage, 1, ms});
  }
  const std::vector<Entry>& entries() const { return entries_; }
  double total_ms() const {
    double s = 0.0;
    for (const auto& e : entries_) s += e.total_ms;
    return s;
  }
  // The reference's CSV (parallel.cpp:106-118): stage,calls,total_ms,percent.
  std::string to_csv() const {
    std::ostringstream out;
    out << "stage,calls,total_ms,percent\n";
    const double sum = total_ms();
    for (const auto& e : entries_) {
      char line[160];
      std::snprintf(line, sizeof(line), "%s,%lld,%.3f,%.3f\n", e.stage.c_str(), e.calls, e.total_ms,
                    sum > 0.0 ? 100.0 * e.total_ms / sum : 0.0);
      out << line;
    }
    return out.str();
  }
  void clear() { entries_.clear(); }
 private:
  std::vector<Entry> entries_;
};

// A parsed bundle plus one GPU context per device it is used on.
class ModelBundle {
 public:
  explicit ModelBundle(std::string text) : text_(std::move(text)) {
    int code = cdvz_gpu_bundle_check(text_.data(), text_.size(), &crc_, &components_);
    check(code);
  }
  static ModelBundle load(const std::string& path) {  // load_model (model_io.cpp:282-288)
    std::ifstream in(path, std::ios::binary);
    if (!in) throw DataError("cannot read model bundle: " + path);
    std::stringstream buf;
    buf << in.rdbuf();
    return ModelBundle(buf.str());
  }
  void save(const std::string& path) const {  // save_model (model_io.cpp:274-280)
    std::ofstream out(path, std::ios::binary);
    if (!out) throw DataError("cannot write model bundle: " + path);
    out.write(text_.data(), std::streamsize(text_.size()));
  }
  uint32_t crc() const { return crc_; }
  int components() const { return components_; }
  const std::string& text() const { return text_; }
  cdvz_gpu_ctx* context(int device = 0, int max_batch = 256) const {
    auto it = ctx_.find(device);
    if (it != ctx_.end()) return it->second.get();
    cdvz_gpu_ctx* c = nullptr;
    check(cdvz_gpu_create(text_.data(), text_.size(), device, max_batch, &c));
    ctx_[device] = std::shared_ptr<cdvz_gpu_ctx>(c, cdvz_gpu_destroy);
    return c;
  }
  // A frame-sharded context over several devices (cdvz_gpu_create_multi).
  cdvz_gpu_ctx* context(const std::vector<int>& devices, int max_batch = 256) const {
    if (devices.size() == 1) return context(devices[0], max_batch);
    auto it = multi_.find(devices);
    if (it != multi_.end()) return it->second.get();
    cdvz_gpu_ctx* c = nullptr;
    check(cdvz_gpu_create_multi(text_.data(), text_.size(), devices.data(), int(devices.size()), max_batch, &c));
    multi_[devices] = std::shared_ptr<cdvz_gpu_ctx>(c, cdvz_gpu_destroy);
    return c;
  }
 private:
  std::string text_;
  uint32_t crc_ = 0;
  int components_ = 0;
  mutable std::map<int, std::shared_ptr<cdvz_gpu_ctx>> ctx_;
  mutable std::map<std::vector<int>, std::shared_ptr<cdvz_gpu_ctx>> multi_;
};

struct TrainOptions {  // pipeline.hpp:22-28
  std::uint64_t seed = 7;
  int gmm_components = 8;
  int em_iterations = 25;
  int select_n = 300;
  int max_side = 640;
  int relevance_bins = 16;
};

// train_model (pipeline.hpp:34-35, pipeline.cpp:99-166) on the GPU
// (cdvz_gpu_train_model). The corpus images must share one
// size (synth_corpus's do). `eng` is accepted for signature parity.
inline ModelBundle train_model(const std::vector<GrayImage>& corpus, const TrainOptions& opts = {},
                               const Engine& eng = {}, int device = 0) {
  (void)eng;
  if (corpus.size() < 20) throw DataError("training corpus needs at least 20 images");
  const int w = corpus[0].w, h = corpus[0].h;
  std::vector<double> pix;
  pix.reserve(corpus.size() * std::size_t(w) * h);
  for (const auto& g : corpus) {
    if (g.w != w || g.h != h) throw UsageError("the GPU trainer takes a corpus of one image size");
    pix.insert(pix.end(), g.pix.begin(), g.pix.end());
  }
  std::size_t len = 0;
  std::string text(std::size_t(1 << 20) + 2048 * std::size_t(std::max(1, opts.gmm_components)), '\0');
  check(cdvz_gpu_train_model(device, pix.data(), int(corpus.size()), w, h, std::size_t(w), opts.seed,
                                 opts.gmm_components, opts.em_iterations, opts.select_n, opts.max_side,
                                 opts.relevance_bins, text.data(), text.size(), &len));
  text.resize(len);
  return ModelBundle(std::move(text));
}

inline void add_timings(cdvz_gpu_ctx* ctx, StageTimings* timings) {
  if (!timings) return;
  double ms[5];
  check(cdvz_gpu_stage_times(ctx, ms), ctx);
  const char* labels[5] = {"detection", "selection", "description", "compression", "aggregation"};
  for (int i = 0; i < 5; ++i) timings->add(labels[i], ms[i]);
}

// encode_image (pipeline.cpp:54-97) with the reference's signature: a
// GrayImage of doubles in, the EncodedImage out (its bytes are the GPU's
// container, decoded; norms come from the device's scfv_delta values).
inline EncodedImage encode_image(const GrayImage& img, const ModelBundle& bundle, const ModeSpec& mode,
                                 const Engine& eng = {}, StageTimings* timings = nullptr,
                                 const EncodeOptions& opts = {}) {
  (void)eng;
  if (img.pix.size() != std::size_t(std::max(0, img.w)) * std::size_t(std::max(0, img.h)))
    throw DataError("image raster size does not match its dimensions");
  cdvz_gpu_ctx* ctx = bundle.context(0);
  std::vector<uint8_t> buf(cdvz_gpu_container_slot(mode.id));
  std::size_t offsets[2] = {0, 0};
  int status = 0;
  check(cdvz_gpu_encode_batch_f64(ctx, img.pix.data(), img.w, img.h, std::size_t(img.w), 1, mode.id, opts.max_side,
                                      buf.data(), buf.size(), offsets, &status), ctx);
  if (status == CDVZ_GPU_DATA) throw DataError("image values must be finite and in [0, 1]");
  raise_for(status, "frame failed on the device");
  buf.resize(offsets[1]);
  EncodedImage enc = parse_container(buf);
  std::size_t n = 0;
  check(cdvz_gpu_debug_get(ctx, "norms", 0, nullptr, 0, &n), ctx);
  enc.global_desc.norms.resize(n);
  check(cdvz_gpu_debug_get(ctx, "norms", 0, enc.global_desc.norms.data(), n, &n), ctx);
  add_timings(ctx, timings);
  return enc;
}

// Batch encode: frames of one size -> CDVZ1 containers in frame order, on one
// device or frame-sharded over several (`devices`).
inline std::vector<std::vector<uint8_t>> encode_batch(const std::vector<const GrayImage8*>& frames,
                                                      const ModelBundle& bundle, const ModeSpec& mode,
                                                      StageTimings* timings, const EncodeOptions& opts,
                                                      const std::vector<int>& devices) {
  std::vector<std::vector<uint8_t>> out(frames.size());
  if (frames.empty()) return out;
  const int w = frames[0]->width, h = frames[0]->height;
  std::vector<uint8_t> pix(std::size_t(w) * h * frames.size());
  for (std::size_t i = 0; i < frames.size(); ++i) {
    if (frames[i]->width != w || frames[i]->height != h) throw UsageError("frames of one batch must share a size");
    std::copy(frames[i]->pix.begin(), frames[i]->pix.end(), pix.begin() + long(i) * w * h);
  }
  cdvz_gpu_ctx* ctx = bundle.context(devices);
  const std::size_t slot = cdvz_gpu_container_slot(mode.id);
  std::vector<uint8_t> buf(slot * frames.size());
  std::vector<std::size_t> offsets(frames.size() + 1);
  std::vector<int> status(frames.size());
  check(cdvz_gpu_encode_batch(ctx, pix.data(), w, h, std::size_t(w), int(frames.size()), mode.id, opts.max_side,
                                  buf.data(), buf.size(), offsets.data(), status.data()), ctx);
  for (std::size_t i = 0; i < frames.size(); ++i) {
    raise_for(status[i], "frame failed on the device");
    out[i].assign(buf.begin() + long(offsets[i]), buf.begin() + long(offsets[i + 1]));
  }
  add_timings(ctx, timings);
  return out;
}

inline std::vector<std::vector<uint8_t>> encode_batch(const std::vector<const GrayImage8*>& frames,
                                                      const ModelBundle& bundle, const ModeSpec& mode,
                                                      StageTimings* timings = nullptr, const EncodeOptions& opts = {},
                                                      int device = 0) {
  return encode_batch(frames, bundle, mode, timings, opts, std::vector<int>{device});
}

// encode_image + serialize_container (pipeline.cpp:54-97, container.cpp:32-58).
// A stream of batches (a video feed, a crawl) through
// cdvz_gpu_encode_batch_submit / _wait: submit packs the frames, enqueues the
// copies and kernels and returns; wait() hands back the containers. Two
// batches in flight per context overlap one batch's copies and kernels with
// the previous one's tail. No reference counterpart (the reference encodes
// one image per call); the containers equal encode_batch's.
class PendingBatch {
 public:
  std::vector<std::vector<uint8_t>> wait() {
    if (!ctx_) throw UsageError("batch already waited for");
    cdvz_gpu_ctx* ctx = ctx_;
    ctx_ = nullptr;
    check(cdvz_gpu_encode_batch_wait(ctx, ticket_), ctx);
    std::vector<std::vector<uint8_t>> out(status_.size());
    for (std::size_t i = 0; i < status_.size(); ++i) {
      raise_for(status_[i], "frame failed on the device");
      out[i].assign(buf_.begin() + long(offsets_[i]), buf_.begin() + long(offsets_[i + 1]));
    }
    return out;
  }
  ~PendingBatch() {
    if (ctx_) cdvz_gpu_encode_batch_wait(ctx_, ticket_);  // buffers must outlive the device work
  }
  PendingBatch(const PendingBatch&) = delete;
  PendingBatch& operator=(const PendingBatch&) = delete;

 private:
  friend std::unique_ptr<PendingBatch> submit_batch(const std::vector<const GrayImage8*>&, const ModelBundle&,
                                                    const ModeSpec&, const EncodeOptions&, const std::vector<int>&);
  PendingBatch() = default;
  cdvz_gpu_ctx* ctx_ = nullptr;
  std::uint64_t ticket_ = 0;
  std::vector<uint8_t> pix_, buf_;
  std::vector<std::size_t> offsets_;
  std::vector<int> status_;
};

inline std::unique_ptr<PendingBatch> submit_batch(const std::vector<const GrayImage8*>& frames,
                                                  const ModelBundle& bundle, const ModeSpec& mode,
                                                  const EncodeOptions& opts = {},
                                                  const std::vector<int>& devices = {0}) {
  std::unique_ptr<PendingBatch> p(new PendingBatch());
  if (frames.empty()) throw UsageError("empty batch");
  const int w = frames[0]->width, h = frames[0]->height;
  p->pix_.resize(std::size_t(w) * h * frames.size());
  for (std::size_t i = 0; i < frames.size(); ++i) {
    if (frames[i]->width != w || frames[i]->height != h) throw UsageError("frames of one batch must share a size");
    std::copy(frames[i]->pix.begin(), frames[i]->pix.end(), p->pix_.begin() + long(i) * w * h);
  }
  cdvz_gpu_ctx* ctx = bundle.context(devices);
  p->buf_.resize(cdvz_gpu_container_slot(mode.id) * frames.size());
  p->offsets_.resize(frames.size() + 1);
  p->status_.resize(frames.size());
  check(cdvz_gpu_encode_batch_submit(ctx, p->pix_.data(), w, h, std::size_t(w), int(frames.size()), mode.id,
                                     opts.max_side, p->buf_.data(), p->buf_.size(), p->offsets_.data(),
                                     p->status_.data(), &p->ticket_),
        ctx);
  p->ctx_ = ctx;
  return p;
}

inline std::vector<uint8_t> encode_image(const GrayImage8& img, const ModelBundle& bundle, const ModeSpec& mode,
                                         StageTimings* timings = nullptr, const EncodeOptions& opts = {}) {
  return encode_batch({&img}, bundle, mode, timings, opts)[0];
}

// ------------------------------------------------ ingest (image.cpp:53-92)
// A binary PGM (channels 1) or PPM (channels 3) raster as load_image reads it;
// the grey conversion of a PPM happens on the device.
struct PnmImage {
  int width = 0, height = 0, channels = 1;
  std::vector<uint8_t> raster;  // width * height * channels bytes, row-major
};

inline PnmImage load_pnm(const std::string& path) {  // load_image's file handling and header checks
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open image file: " + path);
  const std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  PnmImage img;
  std::size_t off = 0;
  check(cdvz_gpu_pnm_parse(reinterpret_cast<const uint8_t*>(bytes.data()), bytes.size(), &img.width, &img.height,
                               &img.channels, &off));
  img.raster.assign(bytes.begin() + long(off), bytes.begin() + long(off) + long(img.width) * img.height * img.channels);
  return img;
}

// load_image's raster conversion (image.cpp:78-90): grey = v / 255, colour =
// (0.299 r + 0.587 g + 0.114 b) / 255, in the reference's operation order.
inline GrayImage to_gray(const PnmImage& img) {
  GrayImage g = make_image(img.width, img.height);
  const double inv = 1.0 / 255.0;
  for (std::size_t i = 0; i < g.pix.size(); ++i) {
    const uint8_t* px = img.raster.data() + i * std::size_t(img.channels);
    g.pix[i] = img.channels == 3 ? (0.299 * px[0] + 0.587 * px[1] + 0.114 * px[2]) * inv : px[0] * inv;
  }
  return g;
}

// encode_image(load_image(path), ...) for an in-memory PGM/PPM raster.
inline std::vector<uint8_t> encode_image(const PnmImage& img, const ModelBundle& bundle, const ModeSpec& mode,
                                         StageTimings* timings = nullptr, const EncodeOptions& opts = {},
                                         int device = 0) {
  cdvz_gpu_ctx* ctx = bundle.context(device);
  std::vector<uint8_t> buf(cdvz_gpu_container_slot(mode.id));
  std::size_t offsets[2] = {0, 0};
  int status = 0;
  const std::size_t stride = std::size_t(img.width) * img.channels;
  auto fn = img.channels == 3 ? cdvz_gpu_encode_batch_rgb : cdvz_gpu_encode_batch;
  check(fn(ctx, img.raster.data(), img.width, img.height, stride, 1, mode.id, opts.max_side, buf.data(), buf.size(),
               offsets, &status), ctx);
  raise_for(status, "frame failed on the device");
  buf.resize(offsets[1]);
  add_timings(ctx, timings);
  return buf;
}

// ------------------------------------------------ retrieval (eval.hpp:17-55)
struct MatchResult {  // eval.hpp:17-20
  double global_similarity = -1.0;
  int local_match_count = 0;
};
struct RankedItem {  // eval.hpp:22-25
  std::string id;
  double score = 0.0;
};
struct RankedList {  // eval.hpp:27-30
  std::string query;
  std::vector<RankedItem> items;
};
struct MatchOptions {  // eval.hpp:32-35
  double ratio_test = 0.85;
  int rerank_depth = 50;
};

// The `index` argument of retrieve (a vector of (id, container) pairs),
// decoded once onto a device.
class Index {
 public:
  Index(const std::vector<std::pair<std::string, std::vector<uint8_t>>>& items, int device = 0) {
    std::vector<uint8_t> blob;
    std::vector<std::size_t> off{0};
    for (const auto& it : items) {
      blob.insert(blob.end(), it.second.begin(), it.second.end());
      off.push_back(blob.size());
      ids_.push_back(it.first);
    }
    std::vector<int32_t> order(items.size()), rank(items.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = int32_t(i);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return ids_[a] < ids_[b]; });
    for (std::size_t r = 0; r < order.size(); ++r) rank[std::size_t(order[r])] = int32_t(r);
    cdvz_gpu_index* idx = nullptr;
    check_index(cdvz_gpu_index_create(device, blob.empty() ? nullptr : blob.data(), off.data(), int(items.size()),
                                    rank.data(), &idx), nullptr);
    idx_.reset(idx, cdvz_gpu_index_destroy);
  }
  cdvz_gpu_index* handle() const { return idx_.get(); }
  const std::vector<std::string>& ids() const { return ids_; }

 private:
  std::shared_ptr<cdvz_gpu_index> idx_;
  std::vector<std::string> ids_;
};

// retrieve (eval.cpp:76-124) for a batch of query containers.
inline std::vector<RankedList> retrieve(const std::vector<std::pair<std::string, std::vector<uint8_t>>>& queries,
                                        const Index& index, const MatchOptions& opts = {}) {
  std::vector<uint8_t> blob;
  std::vector<std::size_t> off{0};
  for (const auto& q : queries) {
    blob.insert(blob.end(), q.second.begin(), q.second.end());
    off.push_back(blob.size());
  }
  const std::size_t n = index.ids().size();
  std::vector<int32_t> items(queries.size() * n);
  std::vector<double> scores(queries.size() * n);
  std::vector<RankedList> out(queries.size());
  if (queries.empty()) return out;
  check_index(cdvz_gpu_retrieve(index.handle(), blob.data(), off.data(), int(queries.size()), opts.ratio_test,
                              opts.rerank_depth, 0, items.data(), scores.data()), index.handle());
  for (std::size_t q = 0; q < queries.size(); ++q) {
    out[q].query = queries[q].first;
    for (std::size_t r = 0; r < n; ++r)
      out[q].items.push_back({index.ids()[std::size_t(items[q * n + r])], scores[q * n + r]});
  }
  return out;
}

// format_double (common.cpp:37-49): the shortest %.*g that parses back exactly.
inline std::string format_double(double v) {
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) return buf;
  }
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

// match_pair (eval.cpp:66-74) of query container a and index item i.
inline MatchResult match_pair(const std::vector<uint8_t>& a, const Index& index, int item,
                              const MatchOptions& opts = {}) {
  const std::size_t off[2] = {0, a.size()};
  const int32_t pair[2] = {0, item};
  MatchResult r;
  int32_t local = 0;
  check_index(cdvz_gpu_match_pairs(index.handle(), a.data(), off, 1, pair, 1, opts.ratio_test, &r.global_similarity,
                                 &local), index.handle());
  r.local_match_count = local;
  return r;
}

}  // namespace gpu
}  // namespace cdvz
