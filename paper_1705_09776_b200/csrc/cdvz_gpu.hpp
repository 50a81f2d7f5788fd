// cdvz_gpu.hpp — header-only C++ shim over include/cdvz_gpu.h that mirrors the
// reference's extraction API (proj/include/cdvz/pipeline.hpp:14-20,
// container.hpp:27, model_io.hpp:30-33, transform_coding.hpp:22-24,
// parallel.hpp:117-134) for C++ callers:
//
//   reference                                        this shim
//   ModelBundle load_model(path)                     cdvz::gpu::ModelBundle::load(path)
//   const ModeSpec& mode_by_name(name)               cdvz::gpu::mode_by_name(name)
//   EncodedImage encode_image(img, bundle, mode,     std::vector<uint8_t> cdvz::gpu::encode_image(
//       Engine, StageTimings*, EncodeOptions)            img, bundle, mode, timings, opts)
//   serialize_container(enc)                         (returned directly: CDVZ1 bytes)
//   RankedList retrieve(query, id, index, opts)      cdvz::gpu::retrieve({(id, bytes)...}, Index, opts)
//   MatchResult match_pair(a, b, opts)               cdvz::gpu::match_pair(a_bytes, Index, item, opts)
//
// Images are 8-bit grey rasters (the byte/255 semantics of load_image,
// image.cpp:79-87). Errors keep the reference's exception types: UsageError
// (bad mode name), DataError (bad raster / bundle), std::runtime_error for
// device failures (the CLI's exit code 3). The Engine argument has no GPU
// meaning (results never depend on it, parallel.hpp:16-18) and is dropped.
#pragma once

#include <algorithm>
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
 private:
  std::vector<Entry> entries_;
};

// A parsed bundle plus one GPU context per device it is used on.
class ModelBundle {
 public:
  explicit ModelBundle(std::string text) : text_(std::move(text)) {
    int code = cdvz_gpu_bundle_check(text_.data(), text_.size(), &crc_, &components_);
    raise_for(code, cdvz_gpu_last_error(nullptr));
  }
  static ModelBundle load(const std::string& path) {  // load_model (model_io.cpp:282-288)
    std::ifstream in(path, std::ios::binary);
    if (!in) throw DataError("cannot read model bundle: " + path);
    std::stringstream buf;
    buf << in.rdbuf();
    return ModelBundle(buf.str());
  }
  uint32_t crc() const { return crc_; }
  int components() const { return components_; }
  const std::string& text() const { return text_; }
  cdvz_gpu_ctx* context(int device = 0, int max_batch = 256) const {
    auto it = ctx_.find(device);
    if (it != ctx_.end()) return it->second.get();
    cdvz_gpu_ctx* c = nullptr;
    raise_for(cdvz_gpu_create(text_.data(), text_.size(), device, max_batch, &c), cdvz_gpu_last_error(nullptr));
    ctx_[device] = std::shared_ptr<cdvz_gpu_ctx>(c, cdvz_gpu_destroy);
    return c;
  }
 private:
  std::string text_;
  uint32_t crc_ = 0;
  int components_ = 0;
  mutable std::map<int, std::shared_ptr<cdvz_gpu_ctx>> ctx_;
};

// Batch encode: frames of one size -> CDVZ1 containers in frame order.
inline std::vector<std::vector<uint8_t>> encode_batch(const std::vector<const GrayImage8*>& frames,
                                                      const ModelBundle& bundle, const ModeSpec& mode,
                                                      StageTimings* timings = nullptr, const EncodeOptions& opts = {},
                                                      int device = 0) {
  std::vector<std::vector<uint8_t>> out(frames.size());
  if (frames.empty()) return out;
  const int w = frames[0]->width, h = frames[0]->height;
  std::vector<uint8_t> pix(std::size_t(w) * h * frames.size());
  for (std::size_t i = 0; i < frames.size(); ++i) {
    if (frames[i]->width != w || frames[i]->height != h) throw UsageError("frames of one batch must share a size");
    std::copy(frames[i]->pix.begin(), frames[i]->pix.end(), pix.begin() + long(i) * w * h);
  }
  cdvz_gpu_ctx* ctx = bundle.context(device);
  const std::size_t slot = cdvz_gpu_container_slot(mode.id);
  std::vector<uint8_t> buf(slot * frames.size());
  std::vector<std::size_t> offsets(frames.size() + 1);
  std::vector<int> status(frames.size());
  raise_for(cdvz_gpu_encode_batch(ctx, pix.data(), w, h, std::size_t(w), int(frames.size()), mode.id, opts.max_side,
                                  buf.data(), buf.size(), offsets.data(), status.data()),
            cdvz_gpu_last_error(ctx));
  for (std::size_t i = 0; i < frames.size(); ++i) {
    raise_for(status[i], "frame failed on the device");
    out[i].assign(buf.begin() + long(offsets[i]), buf.begin() + long(offsets[i + 1]));
  }
  if (timings) {
    double ms[5];
    cdvz_gpu_stage_times(ctx, ms);
    const char* labels[5] = {"detection", "selection", "description", "compression", "aggregation"};
    for (int i = 0; i < 5; ++i) timings->add(labels[i], ms[i]);
  }
  return out;
}

// encode_image + serialize_container (pipeline.cpp:54-97, container.cpp:32-58).
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
  raise_for(cdvz_gpu_pnm_parse(reinterpret_cast<const uint8_t*>(bytes.data()), bytes.size(), &img.width, &img.height,
                               &img.channels, &off),
            cdvz_gpu_last_error(nullptr));
  img.raster.assign(bytes.begin() + long(off), bytes.begin() + long(off) + long(img.width) * img.height * img.channels);
  return img;
}

// encode_image(load_image(path), ...) for an in-memory PGM/PPM raster.
inline std::vector<uint8_t> encode_image(const PnmImage& img, const ModelBundle& bundle, const ModeSpec& mode,
                                         const EncodeOptions& opts = {}, int device = 0) {
  cdvz_gpu_ctx* ctx = bundle.context(device);
  std::vector<uint8_t> buf(cdvz_gpu_container_slot(mode.id));
  std::size_t offsets[2] = {0, 0};
  int status = 0;
  const std::size_t stride = std::size_t(img.width) * img.channels;
  auto fn = img.channels == 3 ? cdvz_gpu_encode_batch_rgb : cdvz_gpu_encode_batch;
  raise_for(fn(ctx, img.raster.data(), img.width, img.height, stride, 1, mode.id, opts.max_side, buf.data(), buf.size(),
               offsets, &status),
            cdvz_gpu_last_error(ctx));
  raise_for(status, "frame failed on the device");
  buf.resize(offsets[1]);
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
    raise_for(cdvz_gpu_index_create(device, blob.empty() ? nullptr : blob.data(), off.data(), int(items.size()),
                                    rank.data(), &idx),
              cdvz_gpu_index_last_error(nullptr));
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
  raise_for(cdvz_gpu_retrieve(index.handle(), blob.data(), off.data(), int(queries.size()), opts.ratio_test,
                              opts.rerank_depth, 0, items.data(), scores.data()),
            cdvz_gpu_index_last_error(index.handle()));
  for (std::size_t q = 0; q < queries.size(); ++q) {
    out[q].query = queries[q].first;
    for (std::size_t r = 0; r < n; ++r)
      out[q].items.push_back({index.ids()[std::size_t(items[q * n + r])], scores[q * n + r]});
  }
  return out;
}

// match_pair (eval.cpp:66-74) of query container a and index item i.
inline MatchResult match_pair(const std::vector<uint8_t>& a, const Index& index, int item,
                              const MatchOptions& opts = {}) {
  const std::size_t off[2] = {0, a.size()};
  const int32_t pair[2] = {0, item};
  MatchResult r;
  int32_t local = 0;
  raise_for(cdvz_gpu_match_pairs(index.handle(), a.data(), off, 1, pair, 1, opts.ratio_test, &r.global_similarity,
                                 &local),
            cdvz_gpu_index_last_error(index.handle()));
  r.local_match_count = local;
  return r;
}

}  // namespace gpu
}  // namespace cdvz
