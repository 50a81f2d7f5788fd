// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/descriptor.cpp and proj/src/transform_coding.cpp.
#include <algorithm>
#include <cmath>
#include <numbers>
#include <numeric>

#include "oracle.hpp"

namespace orc {

namespace {

constexpr double kTwoPi = 2.0 * std::numbers::pi;

// descriptor.cpp:20-23
double wrap_angle(double a) {
  a = std::fmod(a, kTwoPi);
  return a < 0.0 ? a + kTwoPi : a;
}

// descriptor.cpp:25-35 — a term is skipped when its fraction is exactly 0.
double sample_bilinear(const Plane& img, double qx, double qy) {
  const int x0 = static_cast<int>(std::floor(qx));
  const int y0 = static_cast<int>(std::floor(qy));
  const double fx = qx - x0, fy = qy - y0;
  double v = (1.0 - fy) * (1.0 - fx) * img.at(y0, x0);
  if (fx > 0.0) v += (1.0 - fy) * fx * img.at(y0, x0 + 1);
  if (fy > 0.0) v += fy * (1.0 - fx) * img.at(y0 + 1, x0);
  if (fx > 0.0 && fy > 0.0) v += fy * fx * img.at(y0 + 1, x0 + 1);
  return v;
}

struct Geometry {  // descriptor.cpp:37-58
  double half = 0, step = 0;
  int samples = 0, sub_per_axis = 0;
  double cos_t = 1, sin_t = 0, inv_cell = 0, gauss_denom = 0;
};

Geometry make_geometry(double sigma, double theta) {
  Geometry g;
  g.half = 6.0 * sigma;
  g.samples = std::max(1, static_cast<int>(std::ceil(12.0 * sigma)));
  g.step = 2.0 * g.half / g.samples;
  g.sub_per_axis = (g.samples + 16 - 1) / 16;
  g.cos_t = std::cos(theta);
  g.sin_t = std::sin(theta);
  g.inv_cell = 1.0 / (3.0 * sigma);
  g.gauss_denom = 2.0 * g.half * g.half;
  return g;
}

// descriptor.cpp:63-119 — one 16x16-sample block, row-major sample order,
// trilinear weights ((w * wv) * wu) * wo added in (dv, du, dob) order.
std::array<double, 128> subpatch(const Plane& img, double cx, double cy, double theta, const Geometry& g, int sub) {
  std::array<double, 128> acc{};
  const int sx = sub % g.sub_per_axis, sy = sub / g.sub_per_axis;
  const int i_lo = sx * 16, j_lo = sy * 16;
  const int i_hi = std::min(g.samples, i_lo + 16), j_hi = std::min(g.samples, j_lo + 16);
  const int w = img.w, h = img.h;
  for (int j = j_lo; j < j_hi; ++j) {
    const double v = (j + 0.5) * g.step - g.half;
    for (int i = i_lo; i < i_hi; ++i) {
      const double u = (i + 0.5) * g.step - g.half;
      const double px = cx + u * g.cos_t - v * g.sin_t;
      const double py = cy + u * g.sin_t + v * g.cos_t;
      if (px < 1.0 || px > w - 2.0 || py < 1.0 || py > h - 2.0) continue;
      const double gx = 0.5 * (sample_bilinear(img, px + 1.0, py) - sample_bilinear(img, px - 1.0, py));
      const double gy = 0.5 * (sample_bilinear(img, px, py + 1.0) - sample_bilinear(img, px, py - 1.0));
      const double mag = std::hypot(gx, gy);
      if (mag == 0.0) continue;
      const double weight = mag * std::exp(-(u * u + v * v) / g.gauss_denom);
      const double phi = wrap_angle(std::atan2(gy, gx) - theta);
      const double cu = u * g.inv_cell + 1.5, cv = v * g.inv_cell + 1.5;
      const double ob = phi / kTwoPi * 8 - 0.5;
      const int cu0 = static_cast<int>(std::floor(cu)), cv0 = static_cast<int>(std::floor(cv));
      const int ob0 = static_cast<int>(std::floor(ob));
      const double fu = cu - cu0, fv = cv - cv0, fo = ob - ob0;
      for (int dv = 0; dv <= 1; ++dv) {
        const int cyc = cv0 + dv;
        if (cyc < 0 || cyc >= 4) continue;
        const double wv = dv ? fv : 1.0 - fv;
        for (int du = 0; du <= 1; ++du) {
          const int cxc = cu0 + du;
          if (cxc < 0 || cxc >= 4) continue;
          const double wu = du ? fu : 1.0 - fu;
          for (int dob = 0; dob <= 1; ++dob) {
            const int bin = ((ob0 + dob) % 8 + 8) % 8;
            const double wo = dob ? fo : 1.0 - fo;
            acc[std::size_t((cyc * 4 + cxc) * 8 + bin)] += weight * wv * wu * wo;
          }
        }
      }
    }
  }
  return acc;
}

std::array<double, 128> merge_partials(const std::vector<std::array<double, 128>>& parts) {
  std::array<double, 128> sum{};
  for (const auto& p : parts)
    for (int i = 0; i < 128; ++i) sum[std::size_t(i)] += p[std::size_t(i)];
  return normalize_descriptor(sum);
}

}  // namespace

// descriptor.cpp:124-139. v.norm() = sqrt of the Eigen-ordered sum of squares
// (eigen_sum); v /= norm divides each element.
std::array<double, 128> normalize_descriptor(std::array<double, 128> v) {
  for (int round = 0; round < 5; ++round) {
    double sq[128];
    for (int i = 0; i < 128; ++i) sq[i] = v[std::size_t(i)] * v[std::size_t(i)];
    const double norm = std::sqrt(eigen_sum(sq, 128));
    if (norm == 0.0) return v;
    for (double& e : v) e /= norm;
    bool clipped = false;
    for (double& e : v)
      if (e > 0.2) { e = 0.2; clipped = true; }
    if (!clipped) return v;
  }
  return v;
}

// descriptor.cpp:149-170 — nearest sigma node, first minimum wins.
LocalFrame resolve_frame(const Pyramid& pyr, const std::vector<double>& sigmas, const Keypoint& k) {
  if (k.octave < 0 || std::size_t(k.octave) >= pyr.octaves.size())
    throw DataError("interest point references a missing octave");
  const Octave& oct = pyr.octaves[std::size_t(k.octave)];
  const double inv = std::ldexp(1.0, -k.octave);
  LocalFrame f;
  f.x = k.x * inv;
  f.y = k.y * inv;
  f.sigma = k.sigma * inv;
  std::size_t best = 0;
  double best_gap = std::abs(sigmas[0] - f.sigma);
  for (std::size_t i = 1; i < sigmas.size(); ++i) {
    const double gap = std::abs(sigmas[i] - f.sigma);
    if (gap < best_gap) { best_gap = gap; best = i; }
  }
  f.level = &oct.gauss[best];
  f.level_index = int(best);
  return f;
}

// descriptor.cpp:172-232
std::vector<double> dominant_orientations(const Plane& lvl, double x, double y, double sigma) {
  const double radius = 3.96 * sigma;
  const double window = 1.5 * sigma;
  const double denom = 2.0 * window * window;
  const int w = lvl.w, h = lvl.h;
  double hist[36] = {0.0};
  const int x_lo = std::max(1, static_cast<int>(std::ceil(x - radius)));
  const int x_hi = std::min(w - 2, static_cast<int>(std::floor(x + radius)));
  const int y_lo = std::max(1, static_cast<int>(std::ceil(y - radius)));
  const int y_hi = std::min(h - 2, static_cast<int>(std::floor(y + radius)));
  for (int iy = y_lo; iy <= y_hi; ++iy)
    for (int ix = x_lo; ix <= x_hi; ++ix) {
      const double dx = ix - x, dy = iy - y;
      const double d2 = dx * dx + dy * dy;
      if (d2 >= radius * radius) continue;
      const double gx = 0.5 * (lvl.at(iy, ix + 1) - lvl.at(iy, ix - 1));
      const double gy = 0.5 * (lvl.at(iy + 1, ix) - lvl.at(iy - 1, ix));
      const double mag = std::hypot(gx, gy);
      if (mag == 0.0) continue;
      const double ang = wrap_angle(std::atan2(gy, gx));
      const int bin = static_cast<int>(std::floor(ang / kTwoPi * 36 + 0.5)) % 36;
      hist[bin] += mag * std::exp(-d2 / denom);
    }
  for (int pass = 0; pass < 2; ++pass) {
    double sm[36];
    for (int b = 0; b < 36; ++b) sm[b] = (hist[(b + 35) % 36] + hist[b] + hist[(b + 1) % 36]) / 3.0;
    for (int b = 0; b < 36; ++b) hist[b] = sm[b];
  }
  double peak = 0.0;
  for (double v : hist) peak = std::max(peak, v);
  if (peak == 0.0) return {0.0};
  std::vector<double> thetas;
  const double bin_width = kTwoPi / 36;
  for (int b = 0; b < 36; ++b) {
    const double v = hist[b], l = hist[(b + 35) % 36], r = hist[(b + 1) % 36];
    if (v <= 0.8 * peak || v < l || v < r) continue;
    const double fit = l - 2.0 * v + r;
    const double delta = std::abs(fit) > 1e-12 ? 0.5 * (l - r) / fit : 0.0;
    thetas.push_back(wrap_angle((b + delta) * bin_width));
  }
  if (thetas.empty()) thetas.push_back(0.0);
  return thetas;
}

// descriptor.cpp:234-241
std::array<double, 128> describe(const Plane& lvl, double x, double y, double sigma, double theta) {
  const Geometry g = make_geometry(sigma, theta);
  std::vector<std::array<double, 128>> parts;
  for (int sp = 0; sp < g.sub_per_axis * g.sub_per_axis; ++sp) parts.push_back(subpatch(lvl, x, y, theta, g, sp));
  return merge_partials(parts);
}

// descriptor.cpp:243-256 — peaks expand in bin order, input order kept.
std::vector<OrientedPoint> assign_orientations(const Pyramid& pyr, const std::vector<double>& sigmas,
                                               const std::vector<Keypoint>& pts) {
  std::vector<OrientedPoint> out;
  for (const Keypoint& k : pts) {
    const LocalFrame f = resolve_frame(pyr, sigmas, k);
    for (double th : dominant_orientations(*f.level, f.x, f.y, f.sigma)) out.push_back({k, th});
  }
  return out;
}

// descriptor.cpp:258-304 (identical to describe() per point by construction).
std::vector<RawDescriptor> describe_batch(const Pyramid& pyr, const std::vector<double>& sigmas,
                                          const std::vector<OrientedPoint>& pts) {
  std::vector<RawDescriptor> out(pts.size());
  for (std::size_t i = 0; i < pts.size(); ++i) {
    const LocalFrame f = resolve_frame(pyr, sigmas, pts[i].pt);
    out[i].v = describe(*f.level, f.x, f.y, f.sigma, pts[i].theta);
    out[i].point = pts[i];
  }
  return out;
}

// ---------------------------------------------------------------- transform coding

// transform_coding.cpp:21-31
const std::array<ModeSpec, 6>& default_modes() {
  static const std::array<ModeSpec, 6> modes = {{
      {0, "512B", 512, 20, 32.0 / 512.0, false},
      {1, "1K", 1024, 32, 64.0 / 512.0, false},
      {2, "2K", 2048, 64, 128.0 / 512.0, false},
      {3, "4K", 4096, 103, 256.0 / 512.0, false},
      {4, "8K", 8192, 103, 320.0 / 512.0, true},
      {5, "16K", 16384, 128, 512.0 / 512.0, true},
  }};
  return modes;
}

const ModeSpec& mode_by_id(int id) {
  for (const auto& m : default_modes())
    if (m.id == id) return m;
  throw DataError("unknown mode id " + std::to_string(id));
}

const ModeSpec& mode_by_name(const std::string& name) {
  for (const auto& m : default_modes())
    if (name == m.name) return m;
  throw UsageError("unknown mode '" + name + "' (expected 512B, 1K, 2K, 4K, 8K or 16K)");
}

// transform_coding.cpp:44-57
void TransformPair::validate() const {
  if (scale == 0.0) throw DataError("transform scale must be nonzero");
  for (const Mat8* m : {&a, &b})
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double g = 0.0;
        for (int k = 0; k < 8; ++k) g += (*m)[i][k] * (*m)[j][k];
        if (i != j && std::abs(g) > 1e-9) throw DataError("transform rows are not orthogonal");
        if (i == j && g <= 0.0) throw DataError("transform has a zero row");
      }
}

// transform_coding.cpp:59-79 — Sylvester Hadamard A, B = A with rows rotated by one.
TransformPair TransformPair::defaults() {
  TransformPair tp;
  Mat8 hm{};
  hm[0][0] = 1.0;
  for (int n = 1; n < 8; n *= 2)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double v = hm[i][j];
        hm[i][j + n] = v;
        hm[i + n][j] = v;
        hm[i + n][j + n] = -v;
      }
  tp.a = hm;
  for (int i = 0; i < 8; ++i) tp.b[i] = hm[(i + 1) % 8];
  tp.scale = 1.0 / 8.0;
  tp.validate();
  return tp;
}

// transform_coding.cpp:81-91 — per cell: scale * (M * h), product summed in column order.
std::array<double, 128> transform_descriptor(const std::array<double, 128>& raw, const TransformPair& tp) {
  std::array<double, 128> out{};
  for (int cell = 0; cell < 16; ++cell) {
    const int cx = cell % 4, cy = cell / 4;
    const Mat8& m = (((cx + cy) & 1) == 0) ? tp.a : tp.b;
    for (int i = 0; i < 8; ++i) {
      double s = m[i][0] * raw[std::size_t(cell * 8)];
      for (int k = 1; k < 8; ++k) s = s + m[i][k] * raw[std::size_t(cell * 8 + k)];
      out[std::size_t(cell * 8 + i)] = tp.scale * s;
    }
  }
  return out;
}

namespace {
Mat8 invert8(const Mat8& m) {  // Gauss-Jordan, partial pivoting (test helper only)
  double a[8][16];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 16; ++j) a[i][j] = j < 8 ? m[i][j] : (j - 8 == i ? 1.0 : 0.0);
  for (int c = 0; c < 8; ++c) {
    int p = c;
    for (int r = c + 1; r < 8; ++r)
      if (std::abs(a[r][c]) > std::abs(a[p][c])) p = r;
    for (int j = 0; j < 16; ++j) std::swap(a[c][j], a[p][j]);
    const double d = a[c][c];
    for (int j = 0; j < 16; ++j) a[c][j] /= d;
    for (int r = 0; r < 8; ++r) {
      if (r == c) continue;
      const double f = a[r][c];
      for (int j = 0; j < 16; ++j) a[r][j] -= f * a[c][j];
    }
  }
  Mat8 out{};
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) out[i][j] = a[i][8 + j];
  return out;
}
}  // namespace

// transform_coding.cpp:93-105
std::array<double, 128> inverse_transform_descriptor(const std::array<double, 128>& t, const TransformPair& tp) {
  const Mat8 ia = invert8(tp.a), ib = invert8(tp.b);
  std::array<double, 128> out{};
  for (int cell = 0; cell < 16; ++cell) {
    const Mat8& m = ((((cell % 4) + (cell / 4)) & 1) == 0) ? ia : ib;
    for (int i = 0; i < 8; ++i) {
      double s = 0.0;
      for (int k = 0; k < 8; ++k) s += m[i][k] * (t[std::size_t(cell * 8 + k)] / tp.scale);
      out[std::size_t(cell * 8 + i)] = s;
    }
  }
  return out;
}

void QuantizerModel::validate() const {
  for (int e = 0; e < 128; ++e)
    if (!(t0[std::size_t(e)] < t1[std::size_t(e)])) throw DataError("quantizer thresholds must satisfy t0 < t1");
  std::array<int, 128> seen{};
  for (int e : priority)
    if (e < 0 || e >= 128 || seen[std::size_t(e)]++) throw DataError("quantizer priority must be a permutation of 0..127");
}

QuantizerModel QuantizerModel::neutral() {
  QuantizerModel q;
  q.t0.fill(-1.0);
  q.t1.fill(1.0);
  std::iota(q.priority.begin(), q.priority.end(), 0);
  q.degenerate.fill(0);
  return q;
}

// transform_coding.cpp:126-171
QuantizerModel train_thresholds(const std::vector<std::array<double, 128>>& rows, double p0) {
  if (rows.size() < 1000) throw DataError("threshold training needs at least 1000 descriptors");
  if (!(p0 > 0.0 && p0 < 1.0)) throw DataError("band mass must lie in (0, 1)");
  const std::size_t n = rows.size();
  auto quantile = [n](const std::vector<double>& sorted, double q) {
    const double pos = q * static_cast<double>(n - 1);
    const auto lo = static_cast<std::size_t>(pos);
    const double frac = pos - static_cast<double>(lo);
    if (lo + 1 >= sorted.size()) return sorted.back();
    return sorted[lo] * (1.0 - frac) + sorted[lo + 1] * frac;
  };
  QuantizerModel q;
  q.degenerate.fill(0);
  std::array<double, 128> var{};
  std::vector<double> col(n);
  for (int e = 0; e < 128; ++e) {
    for (std::size_t t = 0; t < n; ++t) col[t] = rows[t][std::size_t(e)];
    double mean_sum = 0.0;  // column mean (sequential sum)
    for (std::size_t t = 0; t < n; ++t) mean_sum += col[t];
    const double mean = mean_sum / double(n);
    double ss = 0.0;
    for (std::size_t t = 0; t < n; ++t) ss += (col[t] - mean) * (col[t] - mean);
    var[std::size_t(e)] = ss / double(n);
    std::sort(col.begin(), col.end());
    double lo = quantile(col, (1.0 - p0) / 2.0), hi = quantile(col, (1.0 + p0) / 2.0);
    if (!(lo < hi)) {
      q.degenerate[std::size_t(e)] = 1;
      const double eps = std::max(1e-9, 1e-9 * std::abs(lo));
      hi = lo + eps;
      lo -= eps;
    }
    q.t0[std::size_t(e)] = lo;
    q.t1[std::size_t(e)] = hi;
  }
  std::iota(q.priority.begin(), q.priority.end(), 0);
  std::sort(q.priority.begin(), q.priority.end(), [&](int x, int y) {
    const bool dx = q.degenerate[std::size_t(x)], dy = q.degenerate[std::size_t(y)];
    if (dx != dy) return !dx;
    if (var[std::size_t(x)] != var[std::size_t(y)]) return var[std::size_t(x)] > var[std::size_t(y)];
    return x < y;
  });
  q.validate();
  return q;
}

// transform_coding.cpp:173-200
uint16_t quantize_coord(double v, int extent) {
  if (extent < 2) throw DataError("coordinate extent must be at least 2");
  const double c = std::clamp(v, 0.0, static_cast<double>(extent - 1));
  return static_cast<uint16_t>(std::lround(c / (extent - 1) * 65535.0));
}
double dequantize_coord(uint16_t q, int extent) { return static_cast<double>(q) / 65535.0 * (extent - 1); }

uint8_t quantize_sigma_log(double sigma) {
  const double s = std::clamp(sigma, 0.5, 64.0);
  const double t = std::log2(s / 0.5) / std::log2(64.0 / 0.5);
  return static_cast<uint8_t>(std::lround(t * 255.0));
}
double dequantize_sigma_log(uint8_t q) { return 0.5 * std::pow(64.0 / 0.5, static_cast<double>(q) / 255.0); }

uint8_t quantize_theta(double theta) {
  double t = theta / kTwoPi;
  t -= std::floor(t);
  return static_cast<uint8_t>(static_cast<int>(std::lround(t * 256.0)) & 0xFF);
}
double dequantize_theta(uint8_t q) { return static_cast<double>(q) / 256.0 * kTwoPi; }

// transform_coding.cpp:202-217 — inclusive middle band.
TernaryCode quantize_ternary(const std::array<double, 128>& t, const QuantizerModel& qm, const ModeSpec& mode) {
  if (mode.elements < 1 || mode.elements > 128) throw DataError("invalid element count for mode");
  TernaryCode c;
  c.mode = static_cast<uint8_t>(mode.id);
  c.symbols.resize(std::size_t(mode.elements));
  for (int j = 0; j < mode.elements; ++j) {
    const int e = qm.priority[std::size_t(j)];
    const double v = t[std::size_t(e)];
    int8_t s = 0;
    if (v < qm.t0[std::size_t(e)]) s = -1;
    else if (v > qm.t1[std::size_t(e)]) s = 1;
    c.symbols[std::size_t(j)] = s;
  }
  return c;
}

int ternary_distance(const TernaryCode& a, const TernaryCode& b) {
  if (a.mode != b.mode || a.symbols.size() != b.symbols.size())
    throw DataError("ternary codes from different modes cannot be compared");
  int d = 0;
  for (std::size_t i = 0; i < a.symbols.size(); ++i) d += std::abs(int(a.symbols[i]) - int(b.symbols[i]));
  return d;
}

std::size_t packed_code_bytes(int elements) { return 6 + (std::size_t(elements) * 2 + 7) / 8; }

// transform_coding.cpp:232-270 — 00 zero, 01 plus, 10 minus, LSB-first.
std::vector<uint8_t> pack_local(const std::vector<TernaryCode>& codes, const ModeSpec& mode) {
  if (codes.size() > 0xFFFF) throw DataError("too many codes for one local block");
  std::vector<uint8_t> out;
  out.push_back(uint8_t(mode.id));
  out.push_back(uint8_t(mode.elements));
  out.push_back(uint8_t(codes.size() & 0xFF));
  out.push_back(uint8_t(codes.size() >> 8));
  for (const auto& c : codes) {
    if (c.mode != mode.id) throw DataError("code mode does not match block mode");
    if (c.symbols.size() != std::size_t(mode.elements)) throw DataError("code symbol count does not match block mode");
    out.push_back(uint8_t(c.xq & 0xFF));
    out.push_back(uint8_t(c.xq >> 8));
    out.push_back(uint8_t(c.yq & 0xFF));
    out.push_back(uint8_t(c.yq >> 8));
    out.push_back(c.sigma_q);
    out.push_back(c.theta_q);
    uint8_t byte = 0;
    int filled = 0;
    for (int8_t s : c.symbols) {
      uint8_t bits;
      if (s == 0) bits = 0;
      else if (s == 1) bits = 1;
      else if (s == -1) bits = 2;
      else throw DataError("symbol outside {-1, 0, +1}");
      byte |= uint8_t(bits << (2 * filled));
      if (++filled == 4) { out.push_back(byte); byte = 0; filled = 0; }
    }
    if (filled > 0) out.push_back(byte);
  }
  return out;
}

// transform_coding.cpp:272-305
std::vector<TernaryCode> unpack_local(const std::vector<uint8_t>& bytes) {
  if (bytes.size() < kLocalHeaderBytes) throw DataError("local block truncated");
  const int mode_id = bytes[0], elements = bytes[1];
  const std::size_t count = std::size_t(bytes[2]) | (std::size_t(bytes[3]) << 8);
  if (mode_id > 5) throw DataError("local block has an unknown mode id");
  if (elements < 1 || elements > 128) throw DataError("local block has an invalid element count");
  const std::size_t per = packed_code_bytes(elements);
  if (bytes.size() != kLocalHeaderBytes + count * per) throw DataError("local block length does not match its header");
  std::vector<TernaryCode> codes(count);
  std::size_t off = kLocalHeaderBytes;
  for (auto& c : codes) {
    c.mode = uint8_t(mode_id);
    c.xq = uint16_t(bytes[off] | (bytes[off + 1] << 8));
    c.yq = uint16_t(bytes[off + 2] | (bytes[off + 3] << 8));
    c.sigma_q = bytes[off + 4];
    c.theta_q = bytes[off + 5];
    off += 6;
    c.symbols.resize(std::size_t(elements));
    for (int i = 0; i < elements; ++i) {
      const uint8_t bits = (bytes[off + std::size_t(i / 4)] >> (2 * (i % 4))) & 3u;
      if (bits == 0) c.symbols[std::size_t(i)] = 0;
      else if (bits == 1) c.symbols[std::size_t(i)] = 1;
      else if (bits == 2) c.symbols[std::size_t(i)] = -1;
      else throw DataError("reserved symbol pattern in local block");
    }
    off += (std::size_t(elements) * 2 + 7) / 8;
  }
  return codes;
}

}  // namespace orc
