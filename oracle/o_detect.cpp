// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/scale_space.cpp and proj/src/relevance.cpp.
#include <algorithm>
#include <cmath>

#include "oracle.hpp"

namespace orc {

namespace {

// alpha = beta * l, Eigen's 4x4 lazy product order: ((b0 l0 + b1 l1) + b2 l2) + b3 l3
// (scale_space.cpp:169, 232, 251).
inline void alpha_of(const Mat4& beta, const double l[4], double a[4]) {
  for (int i = 0; i < 4; ++i) {
    double s = beta[i][0] * l[0];
    s = s + beta[i][1] * l[1];
    s = s + beta[i][2] * l[2];
    s = s + beta[i][3] * l[3];
    a[i] = s;
  }
}

// scale_space.cpp:16-18 — Horner.
inline double poly_at(const double a[4], double s) { return a[0] + s * (a[1] + s * (a[2] + s * a[3])); }

// scale_space.cpp:20-43 — stable real roots of 3 a3 s^2 + 2 a2 s + a1.
int derivative_roots(const double a[4], double r[2]) {
  const double qa = 3.0 * a[3], qb = 2.0 * a[2], qc = a[1];
  if (qa == 0.0) {
    if (qb == 0.0) return 0;
    r[0] = -qc / qb;
    return 1;
  }
  const double disc = qb * qb - 4.0 * qa * qc;
  if (disc < 0.0) return 0;
  const double sq = std::sqrt(disc);
  const double q = -0.5 * (qb + std::copysign(sq, qb));
  int n = 0;
  if (q != 0.0) {
    r[n++] = q / qa;
    r[n++] = qc / q;
  } else {
    r[n++] = 0.0;
  }
  if (n == 2 && r[0] == r[1]) n = 1;
  return n;
}

void load_l(const Octave& oct, int y, int x, double l[4]) {
  for (int k = 0; k < 4; ++k) l[k] = oct.log[std::size_t(k)].at(y, x);
}

}  // namespace

// scale_space.cpp:56-73: beta = V^-1 with Eigen::FullPivLU, restated step for
// step (complete pivoting, then FullPivLU::_solve_impl on the identity).
// Pinned bit for bit against the reference's own compute_beta built in
// oracle/_ref (tests/test_ref_pin.py); the product's bundle.cpp runs the same
// sequence.
Mat4 compute_beta(const std::vector<double>& sigmas) {
  if (sigmas.size() != 4) throw DataError("exactly 4 scales are required");
  for (std::size_t i = 0; i < 4; ++i)
    for (std::size_t j = i + 1; j < 4; ++j)
      if (sigmas[i] == sigmas[j]) throw DataError("duplicate scale makes the fit singular");
  double V[4][4];
  for (int k = 0; k < 4; ++k) {
    double pw = 1.0;
    for (int i = 0; i < 4; ++i) {
      V[k][i] = pw;
      pw *= sigmas[std::size_t(k)];
    }
  }
  Mat4 beta{};
  auto& OUT = beta;
  // Complete-pivoting LU of V, P V Q = L U (Eigen FullPivLU::computeInPlace):
  // pivot = largest |v| of the remaining corner, first in column-major order.
  double lu[4][4];
  int rowp[4] = {0, 1, 2, 3}, colq[4] = {0, 1, 2, 3};
  double max_pivot = 0.0;
  int nonzero = 4;
  for (int k = 0; k < 4; ++k) {
    int pr = k, pc = k;
    double best = -1.0;
    for (int j = k; j < 4; ++j)
      for (int i = k; i < 4; ++i)
        if (std::abs(V[i][j]) > best) {
          best = std::abs(V[i][j]);
          pr = i;
          pc = j;
        }
    if (best == 0.0) {
      nonzero = k;
      break;
    }
    max_pivot = std::max(max_pivot, best);
    if (pr != k) {
      for (int j = 0; j < 4; ++j) std::swap(V[k][j], V[pr][j]);
      std::swap(rowp[k], rowp[pr]);
    }
    if (pc != k) {
      for (int i = 0; i < 4; ++i) std::swap(V[i][k], V[i][pc]);
      std::swap(colq[k], colq[pc]);
    }
    for (int i = k + 1; i < 4; ++i) V[i][k] = V[i][k] / V[k][k];
    for (int j = k + 1; j < 4; ++j)
      for (int i = k + 1; i < 4; ++i) V[i][j] = V[i][j] - V[i][k] * V[k][j];
  }
  // isInvertible(): rank 4 with Eigen's threshold |u_ii| > 4 eps max|pivot|.
  int rank = 0;
  for (int i = 0; i < nonzero; ++i) rank += std::abs(V[i][i]) > 4.0 * 2.220446049250313e-16 * max_pivot ? 1 : 0;
  if (rank != 4) throw DataError("scale node matrix is singular");
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) lu[i][j] = V[i][j];
  // inverse() = solve(I) (FullPivLU::_solve_impl): c = P e_col; unit-lower
  // forward solve; upper solve in triangular_solve_matrix's column order
  // (x_i = c_i * (1 / u_ii) for i descending, then removed from the rows
  // above); x = Q c.
  for (int col = 0; col < 4; ++col) {
    double c[4];
    for (int i = 0; i < 4; ++i) c[i] = rowp[i] == col ? 1.0 : 0.0;
    for (int i = 0; i < 4; ++i)
      for (int r = i + 1; r < 4; ++r) c[r] = c[r] - c[i] * lu[r][i];
    for (int i = 3; i >= 0; --i) {
      c[i] = c[i] * (1.0 / lu[i][i]);
      for (int r = 0; r < i; ++r) c[r] = c[r] - c[i] * lu[r][i];
    }
    for (int i = 0; i < 4; ++i) OUT[colq[i]][col] = c[i];
  }
  return beta;
}

// scale_space.cpp:75-83
void DetectorConfig::finalize() {
  if (sigmas.size() != 4) throw DataError("config requires 4 scales");
  for (std::size_t k = 1; k < sigmas.size(); ++k)
    if (!(sigmas[k] > sigmas[k - 1])) throw DataError("scales must be strictly increasing");
  if (!(sigmas.front() > 0.0)) throw DataError("scales must be positive");
  if (num_octaves < 1) throw DataError("at least one octave is required");
  if (!(edge_r > 0.0)) throw DataError("edge ratio parameter must be positive");
  beta = compute_beta(sigmas);
}

// scale_space.cpp:85-91 — sigma_k = 1.4 * 2^(k/4).
DetectorConfig DetectorConfig::defaults() {
  DetectorConfig c;
  c.sigmas.resize(4);
  for (int k = 0; k < 4; ++k) c.sigmas[std::size_t(k)] = 1.4 * std::pow(2.0, k / 4.0);
  c.finalize();
  return c;
}

// scale_space.cpp:141-153 — every level is blurred from the octave base.
Octave build_octave(const Plane& base, const DetectorConfig& cfg, int index) {
  Octave oct;
  oct.index = index;
  oct.base = base;
  for (double sigma : cfg.sigmas) {
    oct.gauss.push_back(gaussian_blur(base, sigma));
    Plane lap = laplacian_3x3(oct.gauss.back());
    const double s2 = sigma * sigma;
    for (double& v : lap.px) v = s2 * v;
    oct.log.push_back(std::move(lap));
  }
  return oct;
}

// scale_space.cpp:155-215
std::vector<Candidate> detect_extrema(const Octave& oct, const DetectorConfig& cfg) {
  const int w = oct.base.w, h = oct.base.h;
  const int margin = static_cast<int>(std::ceil(3.0 * cfg.sigmas.back())) + 2;
  if (w - 2 * margin <= 0 || h - 2 * margin <= 0) return {};
  const double s_lo = cfg.sigmas.front(), s_hi = cfg.sigmas.back();
  std::vector<Candidate> found;
  for (int y = margin; y < h - margin; ++y) {
    for (int x = margin; x < w - margin; ++x) {
      double l[4], a[4], roots[2];
      load_l(oct, y, x, l);
      alpha_of(cfg.beta, l, a);
      const int nr = derivative_roots(a, roots);
      for (int ri = 0; ri < nr; ++ri) {
        const double s = roots[ri];
        if (s < s_lo || s > s_hi) continue;
        const double p = poly_at(a, s);
        if (std::abs(p) < cfg.response_threshold) continue;
        bool ext = true;
        for (int dy = -1; dy <= 1 && ext; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            if (dx == 0 && dy == 0) continue;
            double ln[4], an[4];
            load_l(oct, y + dy, x + dx, ln);
            alpha_of(cfg.beta, ln, an);
            const double pn = poly_at(an, s);
            if (p > 0.0 ? (p <= pn) : (p >= pn)) { ext = false; break; }
          }
        if (ext) found.push_back({x, y, s, p});
      }
    }
  }
  std::sort(found.begin(), found.end(), [](const Candidate& a, const Candidate& b) {
    if (a.y != b.y) return a.y < b.y;
    if (a.x != b.x) return a.x < b.x;
    if (a.sigma != b.sigma) return a.sigma < b.sigma;
    return a.p < b.p;
  });
  return found;
}

// scale_space.cpp:217-270
std::vector<Keypoint> refine_candidates(const std::vector<Candidate>& cands, const Octave& oct,
                                        const DetectorConfig& cfg) {
  const double rho_limit = cfg.rho_limit();
  const double oct_scale = std::ldexp(1.0, oct.index);
  std::vector<Keypoint> out;
  for (const Candidate& c : cands) {
    double p3[3][3];
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        double l[4], a[4];
        load_l(oct, c.y + dy, c.x + dx, l);
        alpha_of(cfg.beta, l, a);
        p3[dy + 1][dx + 1] = poly_at(a, c.sigma);
      }
    const double gx = 0.5 * (p3[1][2] - p3[1][0]);
    const double gy = 0.5 * (p3[2][1] - p3[0][1]);
    const double hxx = p3[1][2] + p3[1][0] - 2.0 * p3[1][1];
    const double hyy = p3[2][1] + p3[0][1] - 2.0 * p3[1][1];
    const double hxy = 0.25 * (p3[2][2] - p3[2][0] - p3[0][2] + p3[0][0]);
    const double det = hxx * hyy - hxy * hxy;
    if (det <= 0.0) continue;
    const double rho = (hxx + hyy) * (hxx + hyy) / det;
    if (rho > rho_limit) continue;
    const double ox = -(hyy * gx - hxy * gy) / det;
    const double oy = (hxy * gx - hxx * gy) / det;
    if (std::abs(ox) > 0.6 || std::abs(oy) > 0.6) continue;
    double l[4], a[4];
    load_l(oct, c.y, c.x, l);
    alpha_of(cfg.beta, l, a);
    Keypoint k;
    k.x = (c.x + ox) * oct_scale;
    k.y = (c.y + oy) * oct_scale;
    k.sigma = c.sigma * oct_scale;
    k.octave = oct.index;
    k.p = c.p;
    k.rho = rho;
    k.p_ss = 2.0 * a[2] + 6.0 * a[3] * c.sigma;
    out.push_back(k);
  }
  return out;
}

// scale_space.cpp:272-302 — decisions against the original lists; previous
// survivors first, then current survivors; |p| ties drop the current point.
std::vector<Keypoint> dedup_across_octaves(const std::vector<Keypoint>& cur, const std::vector<Keypoint>& prev) {
  std::vector<char> drop_cur(cur.size(), 0), drop_prev(prev.size(), 0);
  for (std::size_t i = 0; i < cur.size(); ++i)
    for (std::size_t j = 0; j < prev.size(); ++j) {
      const double dx = cur[i].x - prev[j].x, dy = cur[i].y - prev[j].y;
      if (dx * dx + dy * dy >= 4.0) continue;
      const double ratio = cur[i].sigma / prev[j].sigma;
      if (!(ratio >= 1.0 / 1.3 && ratio <= 1.3)) continue;
      if (std::abs(prev[j].p) >= std::abs(cur[i].p)) drop_cur[i] = 1;
      else drop_prev[j] = 1;
    }
  std::vector<Keypoint> merged;
  for (std::size_t j = 0; j < prev.size(); ++j)
    if (!drop_prev[j]) merged.push_back(prev[j]);
  for (std::size_t i = 0; i < cur.size(); ++i)
    if (!drop_cur[i]) merged.push_back(cur[i]);
  return merged;
}

// scale_space.cpp:304-326
std::vector<Keypoint> detect_keypoints(const Plane& img, const DetectorConfig& cfg, Pyramid* pyr,
                                       DetectTrace* trace) {
  validate_plane(img);
  if (pyr) pyr->octaves.clear();
  std::vector<Keypoint> acc;
  Plane base = img;
  for (int o = 0; o < cfg.num_octaves; ++o) {
    if (base.w < 16 || base.h < 16) break;
    Octave oct = build_octave(base, cfg, o);
    const auto cands = detect_extrema(oct, cfg);
    auto pts = refine_candidates(cands, oct, cfg);
    if (trace) {
      trace->candidates.push_back(cands);
      trace->refined.push_back(pts);
    }
    acc = (o == 0) ? std::move(pts) : dedup_across_octaves(pts, acc);
    if (o + 1 < cfg.num_octaves) {
      const Plane& last = oct.gauss.back();
      if (last.w >= 16 && last.h >= 16) base = downsample_half(last);
      else base = Plane();
    }
    if (pyr) pyr->octaves.push_back(std::move(oct));
    if (base.w < 16 || base.h < 16) break;
  }
  return acc;
}

// ---------------------------------------------------------------- relevance

// relevance.cpp:24-30 — upper_bound, clamped to the first/last bin.
double LookupTable::operator()(double x) const {
  const auto it = std::upper_bound(edges.begin(), edges.end(), x);
  long bin = long(it - edges.begin()) - 1;
  bin = std::clamp<long>(bin, 0, long(values.size()) - 1);
  return values[std::size_t(bin)];
}

void LookupTable::validate() const {
  if (values.empty() || edges.size() != values.size() + 1) throw DataError("lookup table needs B+1 edges for B values");
  for (std::size_t i = 1; i < edges.size(); ++i)
    if (!(edges[i] > edges[i - 1])) throw DataError("lookup table edges must be increasing");
  for (double v : values)
    if (!(v >= 0.0 && v <= 1.0)) throw DataError("lookup table values must lie in [0, 1]");
}

void RelevanceModel::validate() const {
  for (const auto& t : tables) t.validate();
}

RelevanceModel RelevanceModel::uniform() {
  RelevanceModel m;
  for (auto& t : m.tables) { t.edges = {0.0, 1.0}; t.values = {1.0}; }
  return m;
}

static double stat_of(const Keypoint& k, int c) {
  switch (c) {
    case 0: return k.sigma;
    case 1: return k.p;
    case 2: return k.d;
    case 3: return k.rho;
    default: return k.p_ss;
  }
}

// relevance.cpp:54-59
double relevance(const Keypoint& k, const RelevanceModel& m) {
  double score = 1.0;
  for (int c = 0; c < 5; ++c) score *= m.tables[std::size_t(c)](stat_of(k, c));
  return score;
}

// relevance.cpp:61-69
void fill_center_distance(std::vector<Keypoint>& pts, int w, int h) {
  const double cx = (w - 1) / 2.0, cy = (h - 1) / 2.0;
  const double half_diag = 0.5 * std::hypot(static_cast<double>(w - 1), static_cast<double>(h - 1));
  for (auto& k : pts) {
    const double dist = std::hypot(k.x - cx, k.y - cy);
    k.d = half_diag > 0.0 ? std::min(dist / half_diag, 1.0) : 0.0;
  }
}

// relevance.cpp:71-93 — total order: score desc, |p| desc, y asc, x asc, index asc.
std::vector<Keypoint> select_top(const std::vector<Keypoint>& pts, const RelevanceModel& m, std::size_t n) {
  if (n < 1) throw DataError("selection budget must be at least 1");
  std::vector<std::pair<double, std::size_t>> scored(pts.size());
  for (std::size_t i = 0; i < pts.size(); ++i) scored[i] = {relevance(pts[i], m), i};
  std::sort(scored.begin(), scored.end(), [&](const auto& a, const auto& b) {
    if (a.first != b.first) return a.first > b.first;
    const Keypoint& pa = pts[a.second];
    const Keypoint& pb = pts[b.second];
    const double ap = std::abs(pa.p), bp = std::abs(pb.p);
    if (ap != bp) return ap > bp;
    if (pa.y != pb.y) return pa.y < pb.y;
    if (pa.x != pb.x) return pa.x < pb.x;
    return a.second < b.second;
  });
  std::vector<Keypoint> out;
  for (std::size_t i = 0; i < scored.size() && i < n; ++i) out.push_back(pts[scored[i].second]);
  return out;
}

// relevance.cpp:95-149
RelevanceModel train_relevance_tables(const std::vector<Labeled>& samples, int bins, int min_bin_samples) {
  if (samples.empty()) throw DataError("relevance training corpus is empty");
  if (bins < 1) throw DataError("bin count must be positive");
  std::size_t matched = 0;
  for (const auto& s : samples) matched += s.matched ? 1u : 0u;
  const double global_rate = double(matched) / double(samples.size());
  RelevanceModel model;
  for (int c = 0; c < 5; ++c) {
    double lo = INFINITY, hi = -INFINITY;
    for (const auto& s : samples) {
      const double v = stat_of(s.k, c);
      lo = std::min(lo, v);
      hi = std::max(hi, v);
    }
    if (!(hi > lo)) { lo -= 0.5; hi += 0.5; }
    LookupTable t;
    t.edges.resize(std::size_t(bins) + 1);
    for (int b = 0; b <= bins; ++b) t.edges[std::size_t(b)] = lo + (hi - lo) * b / bins;
    std::vector<std::size_t> count(std::size_t(bins), 0), hits(std::size_t(bins), 0);
    const double width = (hi - lo) / bins;
    for (const auto& s : samples) {
      const double v = stat_of(s.k, c);
      long b = static_cast<long>((v - lo) / width);
      b = std::clamp<long>(b, 0, bins - 1);
      count[std::size_t(b)] += 1;
      hits[std::size_t(b)] += s.matched ? 1u : 0u;
    }
    t.values.resize(std::size_t(bins));
    for (int b = 0; b < bins; ++b) {
      const auto i = std::size_t(b);
      t.values[i] = count[i] < std::size_t(min_bin_samples) ? global_rate : double(hits[i]) / double(count[i]);
    }
    model.tables[std::size_t(c)] = std::move(t);
  }
  model.validate();
  return model;
}

// relevance.cpp:151-171
std::vector<Labeled> label_matches_by_geometry(const std::vector<Keypoint>& a, const std::vector<Keypoint>& b,
                                               const std::vector<std::array<double, 3>>& mapped,
                                               double xy_tol, double ratio_tol) {
  if (a.size() != mapped.size()) throw DataError("mapped point list must parallel the source points");
  std::vector<Labeled> out;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const auto& m = mapped[i];
    bool hit = false;
    for (const auto& q : b) {
      if (std::hypot(q.x - m[0], q.y - m[1]) > xy_tol) continue;
      const double ratio = q.sigma / m[2];
      if (ratio >= 1.0 / ratio_tol && ratio <= ratio_tol) { hit = true; break; }
    }
    out.push_back({a[i], hit});
  }
  return out;
}

}  // namespace orc
