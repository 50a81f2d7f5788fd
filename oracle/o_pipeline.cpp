// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/pipeline.cpp.
#include <algorithm>
#include <chrono>
#include <cmath>

#include "oracle.hpp"

namespace orc {

namespace {
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

// pipeline.cpp:54-97 — detection, selection, description, compression,
// aggregation. Codes are truncated to the budget after compression; the SCFV
// aggregates every descriptor.
EncodedImage encode_image(const Plane& img, const ModelBundle& b, const ModeSpec& mode, int max_side,
                          StageTimes* times, EncodeTrace* trace) {
  validate_plane(img);
  const Plane prep = resize_max_side(img, max_side);

  double t0 = now_ms();
  Pyramid pyr;
  DetectTrace dtrace;
  std::vector<Keypoint> pts = detect_keypoints(prep, b.detector, &pyr, trace ? &dtrace : nullptr);
  double t1 = now_ms();
  fill_center_distance(pts, prep.w, prep.h);
  std::vector<Keypoint> sel = select_top(pts, b.relevance, std::size_t(b.select_n));
  double t2 = now_ms();
  std::vector<OrientedPoint> oriented = assign_orientations(pyr, b.detector.sigmas, sel);
  std::vector<RawDescriptor> desc = describe_batch(pyr, b.detector.sigmas, oriented);
  double t3 = now_ms();

  const int nc = b.gmm.components();
  const int k = std::min(nc, std::max(1, static_cast<int>(std::lround(nc * mode.scfv_fraction))));
  const std::size_t global_bytes = scfv_serialized_bytes(nc, k, mode.variance_planes);
  if (global_bytes + kLocalHeaderBytes > mode.budget_bytes) throw DataError("global descriptor alone exceeds the mode budget");
  const std::size_t max_codes = (mode.budget_bytes - global_bytes - kLocalHeaderBytes) / packed_code_bytes(mode.elements);

  EncodedImage e;
  e.mode_id = mode.id;
  e.width = prep.w;
  e.height = prep.h;
  e.model_crc = b.crc();

  for (const RawDescriptor& r : desc) {  // pipeline.cpp:37-50
    TernaryCode c = quantize_ternary(transform_descriptor(r.v, b.transforms), b.quantizer, mode);
    c.xq = quantize_coord(r.point.pt.x, prep.w);
    c.yq = quantize_coord(r.point.pt.y, prep.h);
    c.sigma_q = quantize_sigma_log(r.point.pt.sigma);
    c.theta_q = quantize_theta(r.point.theta);
    e.codes.push_back(std::move(c));
  }
  if (e.codes.size() > max_codes) e.codes.resize(max_codes);
  double t4 = now_ms();

  Mat raw(int(desc.size()), 128);
  for (std::size_t t = 0; t < desc.size(); ++t)
    for (int j = 0; j < 128; ++j) raw(int(t), j) = desc[t].v[std::size_t(j)];
  Mat x = pca_reduce(raw, b.pca);
  Mat gamma = posteriors_matrix(x, b.gmm);
  Mat gm = fv_mean_matrix(x, gamma, b.gmm);
  Mat gv;
  if (mode.variance_planes) gv = fv_var_matrix(x, gamma, b.gmm);
  e.global_desc = scfv_encode(gm, gv, b.gmm, mode);
  double t5 = now_ms();

  if (times) {
    times->ms[0] += t1 - t0;
    times->ms[1] += t2 - t1;
    times->ms[2] += t3 - t2;
    times->ms[3] += t4 - t3;
    times->ms[4] += t5 - t4;
  }
  if (trace) {
    trace->prep_w = prep.w;
    trace->prep_h = prep.h;
    trace->detect = std::move(dtrace);
    trace->keypoints = std::move(pts);
    trace->selected = std::move(sel);
    trace->oriented = std::move(oriented);
    trace->descriptors = std::move(desc);
    trace->x = std::move(x);
    trace->gamma = std::move(gamma);
    trace->gm = std::move(gm);
    trace->gv = std::move(gv);
  }
  return e;
}

// pipeline.cpp:99-166 — used offline to produce the model bundles the
// benchmarks and parity tests consume.
ModelBundle train_model(const std::vector<Plane>& corpus, const TrainOptions& o) {
  if (corpus.size() < 20) throw DataError("training corpus needs at least 20 images");
  ModelBundle b;
  b.detector = DetectorConfig::defaults();
  b.select_n = o.select_n;
  b.relevance = RelevanceModel::uniform();
  b.transforms = TransformPair::defaults();

  std::vector<std::array<double, 128>> rows;
  std::vector<Labeled> labeled;
  for (std::size_t i = 0; i < corpus.size(); ++i) {
    const Plane prep = resize_max_side(corpus[i], o.max_side);
    Pyramid pyr;
    std::vector<Keypoint> pts = detect_keypoints(prep, b.detector, &pyr);
    fill_center_distance(pts, prep.w, prep.h);
    const std::vector<Keypoint> sel = select_top(pts, b.relevance, std::size_t(b.select_n));
    const auto desc = describe_batch(pyr, b.detector.sigmas, assign_orientations(pyr, b.detector.sigmas, sel));
    for (const auto& d : desc) rows.push_back(d.v);

    SynthTransform t;
    t.quarter_turns = 1 + int(i % 3);
    t.scale = 0.75 + 0.05 * double(i % 4);
    t.blur_sigma = (i % 2) ? 1.0 : 0.5;
    const Plane partner = apply_transform(prep, t);
    const std::vector<Keypoint> ppts = detect_keypoints(partner, b.detector, nullptr);
    std::vector<std::array<double, 3>> mapped(sel.size());
    for (std::size_t s = 0; s < sel.size(); ++s) {
      double mx = sel[s].x, my = sel[s].y, ms = sel[s].sigma;
      map_point(t, prep.w, prep.h, mx, my, ms);
      mapped[s] = {mx, my, ms};
    }
    const auto lab = label_matches_by_geometry(sel, ppts, mapped);
    labeled.insert(labeled.end(), lab.begin(), lab.end());
  }
  Mat raw(int(rows.size()), 128);
  for (std::size_t t = 0; t < rows.size(); ++t)
    for (int j = 0; j < 128; ++j) raw(int(t), j) = rows[t][std::size_t(j)];

  b.relevance = train_relevance_tables(labeled, o.relevance_bins);
  b.pca = train_pca(raw);
  const Mat x = pca_reduce(raw, b.pca);
  b.gmm = train_gmm(x, o.gmm_components, o.em_iterations, o.seed);
  std::vector<std::array<double, 128>> transformed(rows.size());
  for (std::size_t t = 0; t < rows.size(); ++t) transformed[t] = transform_descriptor(rows[t], b.transforms);
  b.quantizer = train_thresholds(transformed);
  b.validate();
  return b;
}

}  // namespace orc
