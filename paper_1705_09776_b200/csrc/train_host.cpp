// Host-side pieces of the GPU trainer; see train_host.hpp. Each function cites
// the reference code it follows.
#include "train_host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

namespace cdvz_gpu {

SynthTransform partner_transform(std::size_t i) {  // pipeline.cpp:125-129
  SynthTransform t;
  t.quarter_turns = 1 + static_cast<int>(i % 3);
  t.scale = 0.75 + 0.05 * static_cast<double>(i % 4);
  t.blur_sigma = (i % 2) ? 1.0 : 0.5;
  return t;
}

void transform_size(const SynthTransform& t, int w, int h, int& ow, int& oh) {  // synthetic.cpp:78-84
  int k = t.quarter_turns % 4;
  if (k < 0) k += 4;
  ow = (k % 2) ? h : w;
  oh = (k % 2) ? w : h;
  if (t.scale != 1.0) {
    const int sw = std::max(8, static_cast<int>(std::lround(ow * t.scale)));
    const int sh = std::max(8, static_cast<int>(std::lround(oh * t.scale)));
    ow = sw;
    oh = sh;
  }
}

void map_point(const SynthTransform& t, int src_w, int src_h, double& x, double& y, double& sigma) {
  int w = src_w, h = src_h;  // synthetic.cpp:92-111
  int k = t.quarter_turns % 4;
  if (k < 0) k += 4;
  for (int turn = 0; turn < k; ++turn) {
    const double nx = h - 1 - y;
    const double ny = x;
    x = nx;
    y = ny;
    std::swap(w, h);
  }
  if (t.scale != 1.0) {
    const int out_w = std::max(8, static_cast<int>(std::lround(w * t.scale)));
    const int out_h = std::max(8, static_cast<int>(std::lround(h * t.scale)));
    x = (x + 0.5) * out_w / w - 0.5;
    y = (y + 0.5) * out_h / h - 0.5;
    sigma *= 0.5 * (static_cast<double>(out_w) / w + static_cast<double>(out_h) / h);
  }
}

void label_matches(const std::vector<TrainPoint>& a, const std::vector<TrainPoint>& b,
                   const std::vector<std::array<double, 3>>& mapped, double xy_tol, double ratio_tol,
                   std::vector<std::pair<TrainPoint, bool>>& out) {
  if (a.size() != mapped.size()) throw DataError("mapped point list must parallel the source points");
  for (std::size_t i = 0; i < a.size(); ++i) {  // relevance.cpp:147-170
    const auto& m = mapped[i];
    bool matched = false;
    for (const auto& q : b) {
      if (std::hypot(q.x - m[0], q.y - m[1]) > xy_tol) continue;
      const double ratio = q.sigma / m[2];
      if (ratio >= 1.0 / ratio_tol && ratio <= ratio_tol) {
        matched = true;
        break;
      }
    }
    out.push_back({a[i], matched});
  }
}

std::array<LutTable, 5> train_relevance(const std::vector<std::pair<TrainPoint, bool>>& samples, int bins,
                                        int min_bin_samples) {
  if (samples.empty()) throw DataError("relevance training corpus is empty");  // relevance.cpp:95-145
  if (bins < 1) throw DataError("bin count must be positive");
  std::size_t matched_total = 0;
  for (const auto& s : samples) matched_total += s.second ? 1u : 0u;
  const double global_rate = static_cast<double>(matched_total) / static_cast<double>(samples.size());
  auto value = [](const TrainPoint& p, int c) {  // FeatureStats::value (relevance.cpp:13-22)
    switch (c) {
      case 0: return p.sigma;
      case 1: return p.p;
      case 2: return p.d;
      case 3: return p.rho;
      default: return p.pss;
    }
  };
  std::array<LutTable, 5> out;
  for (int c = 0; c < 5; ++c) {
    double lo = std::numeric_limits<double>::infinity(), hi = -std::numeric_limits<double>::infinity();
    for (const auto& s : samples) {
      const double v = value(s.first, c);
      lo = std::min(lo, v);
      hi = std::max(hi, v);
    }
    if (!(hi > lo)) {
      lo -= 0.5;
      hi += 0.5;
    }
    LutTable t;
    t.edges.resize(static_cast<std::size_t>(bins) + 1);
    for (int b = 0; b <= bins; ++b) t.edges[static_cast<std::size_t>(b)] = lo + (hi - lo) * b / bins;
    std::vector<std::size_t> count(static_cast<std::size_t>(bins), 0), hits(static_cast<std::size_t>(bins), 0);
    const double width = (hi - lo) / bins;
    for (const auto& s : samples) {
      auto b = static_cast<std::ptrdiff_t>((value(s.first, c) - lo) / width);
      b = std::clamp<std::ptrdiff_t>(b, 0, bins - 1);
      count[static_cast<std::size_t>(b)] += 1;
      hits[static_cast<std::size_t>(b)] += s.second ? 1u : 0u;
    }
    t.values.resize(static_cast<std::size_t>(bins));
    for (int b = 0; b < bins; ++b) {
      const auto i = static_cast<std::size_t>(b);
      t.values[i] = count[i] < static_cast<std::size_t>(min_bin_samples)
                        ? global_rate
                        : static_cast<double>(hits[i]) / static_cast<double>(count[i]);
    }
    out[static_cast<std::size_t>(c)] = std::move(t);
  }
  return out;
}

// Cyclic Jacobi on a symmetric 128 x 128 matrix (the reference uses Eigen's
// SelfAdjointEigenSolver, scfv.cpp:337; any accurate solver gives the same
// eigenvectors up to sign and rounding, and train_pca fixes the sign).
void sym_eigen128(const std::vector<double>& a_in, std::vector<double>& vals, std::vector<double>& vecs) {
  constexpr int N = 128;
  std::vector<double> a(a_in);
  vecs.assign(std::size_t(N) * N, 0.0);
  for (int i = 0; i < N; ++i) vecs[std::size_t(i) * N + i] = 1.0;
  double scale = 0.0;
  for (double v : a) scale = std::max(scale, std::abs(v));
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < N; ++p)
      for (int q = p + 1; q < N; ++q) off += a[std::size_t(p) * N + q] * a[std::size_t(p) * N + q];
    if (off <= 1e-30 * scale * scale) break;
    for (int p = 0; p < N; ++p)
      for (int q = p + 1; q < N; ++q) {
        const double apq = a[std::size_t(p) * N + q];
        if (std::abs(apq) <= 1e-300) continue;
        const double app = a[std::size_t(p) * N + p], aqq = a[std::size_t(q) * N + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < N; ++k) {  // A <- J^T A J (columns p, q, then rows p, q)
          const double akp = a[std::size_t(k) * N + p], akq = a[std::size_t(k) * N + q];
          a[std::size_t(k) * N + p] = c * akp - s * akq;
          a[std::size_t(k) * N + q] = s * akp + c * akq;
        }
        for (int k = 0; k < N; ++k) {
          const double apk = a[std::size_t(p) * N + k], aqk = a[std::size_t(q) * N + k];
          a[std::size_t(p) * N + k] = c * apk - s * aqk;
          a[std::size_t(q) * N + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < N; ++k) {
          const double vkp = vecs[std::size_t(k) * N + p], vkq = vecs[std::size_t(k) * N + q];
          vecs[std::size_t(k) * N + p] = c * vkp - s * vkq;
          vecs[std::size_t(k) * N + q] = s * vkp + c * vkq;
        }
      }
  }
  std::vector<int> order(N);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return a[std::size_t(x) * N + x] < a[std::size_t(y) * N + y]; });
  std::vector<double> sorted(std::size_t(N) * N);
  vals.resize(N);
  for (int j = 0; j < N; ++j) {
    vals[std::size_t(j)] = a[std::size_t(order[std::size_t(j)]) * N + order[std::size_t(j)]];
    for (int k = 0; k < N; ++k) sorted[std::size_t(k) * N + j] = vecs[std::size_t(k) * N + order[std::size_t(j)]];
  }
  vecs.swap(sorted);
}

std::vector<long long> kmeanspp(const std::vector<double>& x, long long n, int nc, std::mt19937_64& rng) {
  // scfv.cpp:368-393: rowwise squared distances (sequential sums), the
  // packet-order total, a uniform draw and the first cumulative crossing.
  auto sqdist = [&](long long t, long long c) {
    double s = 0.0;
    for (int j = 0; j < 32; ++j) {
      const double d = x[std::size_t(t) * 32 + j] - x[std::size_t(c) * 32 + j];
      s = j ? s + d * d : d * d;
    }
    return s;
  };
  std::vector<long long> centers;
  centers.push_back(static_cast<long long>(rng() % static_cast<std::uint64_t>(n)));
  std::vector<double> dist2(static_cast<std::size_t>(n));
  for (long long t = 0; t < n; ++t) dist2[std::size_t(t)] = sqdist(t, centers[0]);
  while (static_cast<int>(centers.size()) < nc) {
    const double total = eigen_packet_sum(dist2.data(), dist2.size());
    long long pick = 0;
    if (total > 0.0) {
      const double target = std::uniform_real_distribution<double>(0.0, total)(rng);
      double run = 0.0;
      pick = n - 1;
      for (long long t = 0; t < n; ++t) {
        run += dist2[std::size_t(t)];
        if (run >= target) {
          pick = t;
          break;
        }
      }
    } else {
      pick = static_cast<long long>(rng() % static_cast<std::uint64_t>(n));
    }
    centers.push_back(pick);
    for (long long t = 0; t < n; ++t) dist2[std::size_t(t)] = std::min(dist2[std::size_t(t)], sqdist(t, pick));
  }
  return centers;
}

void train_thresholds(const std::vector<double>& tr, long long n, double p0, Bundle& b) {
  if (n < 1000) throw DataError("threshold training needs at least 1000 descriptors");  // transform_coding.cpp:126-172
  auto quantile = [n](const std::vector<double>& sorted, double q) {
    const double pos = q * static_cast<double>(n - 1);
    const auto lo = static_cast<std::size_t>(pos);
    const double frac = pos - static_cast<double>(lo);
    if (lo + 1 >= sorted.size()) return sorted.back();
    return sorted[lo] * (1.0 - frac) + sorted[lo + 1] * frac;
  };
  double variance[128];
  std::vector<double> column(static_cast<std::size_t>(n)), sq(static_cast<std::size_t>(n));
  for (int e = 0; e < 128; ++e) {
    for (long long t = 0; t < n; ++t) column[std::size_t(t)] = tr[std::size_t(t) * 128 + e];
    const double mean = eigen_packet_sum(column.data(), column.size()) / static_cast<double>(n);
    for (long long t = 0; t < n; ++t) {
      const double d = column[std::size_t(t)] - mean;
      sq[std::size_t(t)] = d * d;
    }
    variance[e] = eigen_packet_sum(sq.data(), sq.size()) / static_cast<double>(n);
    std::sort(column.begin(), column.end());
    double lo = quantile(column, (1.0 - p0) / 2.0);
    double hi = quantile(column, (1.0 + p0) / 2.0);
    b.degenerate[e] = 0;
    if (!(lo < hi)) {
      b.degenerate[e] = 1;
      const double eps = std::max(1e-9, 1e-9 * std::abs(lo));
      hi = lo + eps;
      lo -= eps;
    }
    b.t0[e] = lo;
    b.t1[e] = hi;
  }
  std::iota(b.priority, b.priority + 128, 0);
  std::sort(b.priority, b.priority + 128, [&](int x, int y) {
    const bool dx = b.degenerate[x], dy = b.degenerate[y];
    if (dx != dy) return !dx;
    if (variance[x] != variance[y]) return variance[x] > variance[y];
    return x < y;
  });
}

}  // namespace cdvz_gpu
