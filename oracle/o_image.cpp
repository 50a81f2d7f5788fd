// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/common.cpp, proj/src/image.cpp and proj/src/synthetic.cpp.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <numbers>
#include <random>

#include "oracle.hpp"

namespace orc {

// proj/src/common.cpp:11-35 — reflected CRC-32, polynomial 0xEDB88320.
uint32_t crc32(const void* data, std::size_t len, uint32_t seed) {
  static const auto table = [] {
    std::array<uint32_t, 256> t{};
    for (uint32_t n = 0; n < 256; ++n) {
      uint32_t c = n;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
      t[n] = c;
    }
    return t;
  }();
  const auto* p = static_cast<const unsigned char*>(data);
  uint32_t c = seed ^ 0xFFFFFFFFu;
  for (std::size_t i = 0; i < len; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// proj/src/common.cpp:37-49 — shortest "%.*g" that parses back bit-exactly.
std::string format_double(double v) {
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    double back = 0.0;
    const std::size_t n = std::string_view(buf).size();
    auto r = std::from_chars(buf, buf + n, back);
    if (r.ec == std::errc() && back == v) return buf;
  }
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// proj/src/common.cpp:51-57
double parse_double(std::string_view s) {
  double v = 0.0;
  auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc() || r.ptr != s.data() + s.size())
    throw DataError("invalid floating point literal: '" + std::string(s) + "'");
  return v;
}

double eigen_sum(const double* v, std::size_t n) {
  if (n == 0) return 0.0;
  if (n < 4) {  // fewer than two packets: first packet (if any) reduced, rest sequential
    if (n < 2) return v[0];
    double r = v[0] + v[1];
    for (std::size_t i = 2; i < n; ++i) r += v[i];
    return r;
  }
  const std::size_t end2 = (n / 4) * 4, end1 = (n / 2) * 2;
  double a0 = v[0], a1 = v[1], b0 = v[2], b1 = v[3];
  for (std::size_t i = 4; i < end2; i += 4) {
    a0 += v[i]; a1 += v[i + 1]; b0 += v[i + 2]; b1 += v[i + 3];
  }
  a0 += b0; a1 += b1;
  if (end1 > end2) { a0 += v[end2]; a1 += v[end2 + 1]; }
  double r = a0 + a1;
  for (std::size_t i = end1; i < n; ++i) r += v[i];
  return r;
}

// ---------------------------------------------------------------- image

// proj/src/image.cpp:46-51
void validate_plane(const Plane& img) {
  if (img.w < 8 || img.h < 8) throw DataError("image smaller than 8 px per side");
  for (double v : img.px)
    if (!std::isfinite(v) || v < 0.0 || v > 1.0) throw DataError("image values must be finite and in [0, 1]");
}

// proj/src/image.cpp:79-87 — grey byte b maps to b * (1/255).
Plane plane_from_u8(const uint8_t* bytes, int w, int h, std::size_t stride) {
  Plane img(w, h);
  const double inv = 1.0 / 255.0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) img.at(y, x) = bytes[std::size_t(y) * stride + x] * inv;
  return img;
}

// proj/src/image.cpp:82-86 (load_image, P6 branch)
Plane plane_from_rgb(const uint8_t* rgb, int w, int h, std::size_t stride) {
  Plane img(w, h);
  const double inv = 1.0 / 255.0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const uint8_t* p = rgb + std::size_t(y) * stride + std::size_t(3) * x;
      img.at(y, x) = (0.299 * p[0] + 0.587 * p[1] + 0.114 * p[2]) * inv;
    }
  return img;
}

// proj/src/image.cpp:101-102
std::vector<uint8_t> plane_to_u8(const Plane& img) {
  std::vector<uint8_t> out(img.px.size());
  for (std::size_t i = 0; i < out.size(); ++i) out[i] = static_cast<uint8_t>(std::lround(img.px[i] * 255.0));
  return out;
}

// proj/src/image.cpp:107-129 — half-pixel aligned bilinear, clamped source.
Plane rescale_bilinear(const Plane& img, int ow, int oh) {
  if (ow < 1 || oh < 1) throw DataError("rescale target must be positive");
  const double sx = static_cast<double>(img.w) / ow;
  const double sy = static_cast<double>(img.h) / oh;
  Plane out(ow, oh);
  for (int y = 0; y < oh; ++y) {
    double fy_src = (y + 0.5) * sy - 0.5;
    fy_src = std::min(std::max(fy_src, 0.0), static_cast<double>(img.h - 1));
    const int y0 = static_cast<int>(fy_src);
    const int y1 = std::min(y0 + 1, img.h - 1);
    const double fy = fy_src - y0;
    for (int x = 0; x < ow; ++x) {
      double fx_src = (x + 0.5) * sx - 0.5;
      fx_src = std::min(std::max(fx_src, 0.0), static_cast<double>(img.w - 1));
      const int x0 = static_cast<int>(fx_src);
      const int x1 = std::min(x0 + 1, img.w - 1);
      const double fx = fx_src - x0;
      const double top = (1.0 - fx) * img.at(y0, x0) + fx * img.at(y0, x1);
      const double bot = (1.0 - fx) * img.at(y1, x0) + fx * img.at(y1, x1);
      out.at(y, x) = (1.0 - fy) * top + fy * bot;
    }
  }
  return out;
}

// proj/src/image.cpp:131-145
Plane resize_max_side(const Plane& img, int limit) {
  if (limit < 8) throw DataError("max-side limit must be at least 8");
  const int longer = std::max(img.w, img.h);
  if (longer <= limit) return img;
  const double scale = static_cast<double>(limit) / longer;
  int ow = limit, oh = limit;
  if (img.w >= img.h) oh = std::max(8, static_cast<int>(std::lround(img.h * scale)));
  else ow = std::max(8, static_cast<int>(std::lround(img.w * scale)));
  return rescale_bilinear(img, ow, oh);
}

// proj/src/image.cpp:147-155
Plane downsample_half(const Plane& img) {
  if (img.w < 16 || img.h < 16) throw DataError("image too small to downsample");
  Plane out(img.w / 2, img.h / 2);
  for (int y = 0; y < out.h; ++y)
    for (int x = 0; x < out.w; ++x) out.at(y, x) = img.at(2 * y, 2 * x);
  return out;
}

// proj/src/image.cpp:163-175
std::vector<double> gaussian_taps(double sigma) {
  if (!(sigma > 0.0)) throw DataError("gaussian sigma must be positive");
  const int r = static_cast<int>(std::ceil(3.0 * sigma));
  std::vector<double> t(std::size_t(2 * r + 1));
  double total = 0.0;
  for (int j = -r; j <= r; ++j) {
    const double e = std::exp(-(static_cast<double>(j) * j) / (2.0 * sigma * sigma));
    t[std::size_t(j + r)] = e;
    total += e;
  }
  for (double& e : t) e /= total;
  return t;
}

// proj/src/image.cpp:177-212 — x pass into an f64 temporary, then y pass; each
// tap sum starts from 0.0 and runs j = -r..r; mirror borders.
Plane gaussian_blur(const Plane& img, double sigma) {
  const auto taps = gaussian_taps(sigma);
  const int r = static_cast<int>(taps.size() / 2);
  const int w = img.w, h = img.h;
  Plane tmp(w, h), out(w, h);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double acc = 0.0;
      for (int j = -r; j <= r; ++j) acc += taps[std::size_t(j + r)] * img.at(y, int(mirror_index(x + j, w)));
      tmp.at(y, x) = acc;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double acc = 0.0;
      for (int j = -r; j <= r; ++j) acc += taps[std::size_t(j + r)] * tmp.at(int(mirror_index(y + j, h)), x);
      out.at(y, x) = acc;
    }
  return out;
}

// proj/src/image.cpp:220-238 — (((up + down) + left) + right) - 4c.
Plane laplacian_3x3(const Plane& img) {
  const int w = img.w, h = img.h;
  Plane out(w, h);
  for (int y = 0; y < h; ++y) {
    const int ym = int(mirror_index(y - 1, h)), yp = int(mirror_index(y + 1, h));
    for (int x = 0; x < w; ++x) {
      const int xm = int(mirror_index(x - 1, w)), xp = int(mirror_index(x + 1, w));
      out.at(y, x) = img.at(ym, x) + img.at(yp, x) + img.at(y, xm) + img.at(y, xp) - 4.0 * img.at(y, x);
    }
  }
  return out;
}

// ---------------------------------------------------------------- synthetic

// proj/src/synthetic.cpp:11-53 — libstdc++'s mt19937_64 and
// uniform_real_distribution reproduce the reference's draws.
Plane synth_image(uint64_t seed, int w, int h) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  Plane canvas(w, h, 0.0);

  const int n_blobs = 8 + static_cast<int>(rng() % 7);
  for (int b = 0; b < n_blobs; ++b) {
    const double cx = (0.12 + 0.76 * unit(rng)) * w;
    const double cy = (0.12 + 0.76 * unit(rng)) * h;
    const double s = 2.0 + 10.0 * unit(rng);
    // Same expression shape as synthetic.cpp:21 so g++ picks the same
    // (unspecified) operand evaluation order for the two draws.
    const double amp = (unit(rng) < 0.5 ? -1.0 : 1.0) * (0.4 + 0.6 * unit(rng));
    const double denom = 2.0 * s * s;
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const double dx = x - cx, dy = y - cy;
        canvas.at(y, x) += amp * std::exp(-(dx * dx + dy * dy) / denom);
      }
  }
  for (int wv = 0; wv < 5; ++wv) {
    const double freq = 1.0 / (6.0 + 26.0 * unit(rng));
    const double angle = unit(rng) * std::numbers::pi;
    const double phase = unit(rng) * 2.0 * std::numbers::pi;
    const double amp = 0.08 + 0.14 * unit(rng);
    const double fx = std::cos(angle) * freq, fy = std::sin(angle) * freq;
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        canvas.at(y, x) += amp * std::sin(2.0 * std::numbers::pi * (fx * x + fy * y) + phase);
  }
  double lo = canvas.px[0], hi = canvas.px[0];
  for (double v : canvas.px) { lo = std::min(lo, v); hi = std::max(hi, v); }
  Plane img(w, h);
  if (hi > lo) {
    const double span = hi - lo;
    for (std::size_t i = 0; i < img.px.size(); ++i) img.px[i] = 0.02 + 0.96 * (canvas.px[i] - lo) / span;
  } else {
    std::fill(img.px.begin(), img.px.end(), 0.5);
  }
  return img;
}

// proj/src/synthetic.cpp:55-61
uint64_t corpus_seed(uint64_t base, int i) { return base + static_cast<uint64_t>(i) * 0x9E3779B97F4A7C15ull; }

// proj/src/synthetic.cpp:63-76 — clockwise quarter turns.
Plane rotate90(const Plane& img, int quarter_turns) {
  int k = quarter_turns % 4;
  if (k < 0) k += 4;
  Plane cur = img;
  for (int t = 0; t < k; ++t) {
    Plane rot(cur.h, cur.w);
    for (int y = 0; y < cur.h; ++y)
      for (int x = 0; x < cur.w; ++x) rot.at(x, cur.h - 1 - y) = cur.at(y, x);
    cur = std::move(rot);
  }
  return cur;
}

// proj/src/synthetic.cpp:78-90
Plane apply_transform(const Plane& img, const SynthTransform& t) {
  Plane out = rotate90(img, t.quarter_turns);
  if (t.scale != 1.0) {
    const int w = std::max(8, static_cast<int>(std::lround(out.w * t.scale)));
    const int h = std::max(8, static_cast<int>(std::lround(out.h * t.scale)));
    out = rescale_bilinear(out, w, h);
  }
  if (t.blur_sigma > 0.0) {
    out = gaussian_blur(out, t.blur_sigma);
    for (double& v : out.px) v = std::max(std::min(v, 1.0), 0.0);
  }
  return out;
}

// proj/src/synthetic.cpp:92-111
void map_point(const SynthTransform& t, int src_w, int src_h, double& x, double& y, double& sigma) {
  int w = src_w, h = src_h;
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
    const int ow = std::max(8, static_cast<int>(std::lround(w * t.scale)));
    const int oh = std::max(8, static_cast<int>(std::lround(h * t.scale)));
    x = (x + 0.5) * ow / w - 0.5;
    y = (y + 0.5) * oh / h - 0.5;
    sigma *= 0.5 * (static_cast<double>(ow) / w + static_cast<double>(oh) / h);
  }
}

}  // namespace orc
