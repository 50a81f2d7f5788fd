// Host-side model bundle handling (see bundle.hpp). The GPU pipeline's
// bit-level parity depends on these host constants matching the reference's
// own derivation: taps from gaussian_kernel (image.cpp:163-175), beta from the
// Vandermonde inverse (scale_space.cpp:56-73, Gauss-Jordan with partial
// pivoting as DESIGN.md §3 records), rho limit and margin.
#include "bundle.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

namespace cdvz_gpu {

namespace {

const char* kLutNames[5] = {"sigma", "p", "d", "rho", "pss"};

// Shortest "%.*g" spelling that reads back to the same bits (common.cpp:37-49).
std::string shortest(double v) {
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    double back = 0.0;
    const auto r = std::from_chars(buf, buf + std::strlen(buf), back);
    if (r.ec == std::errc() && back == v) return buf;
  }
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

double to_double(const std::string& s) {
  double v = 0.0;
  const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc() || r.ptr != s.data() + s.size()) throw DataError("invalid floating point literal: '" + s + "'");
  return v;
}

std::vector<double> numbers(const std::string& line, long expect) {
  std::istringstream in(line);
  std::vector<double> out;
  for (std::string tok; in >> tok;) out.push_back(to_double(tok));
  if (expect >= 0 && long(out.size()) != expect) throw DataError("model bundle row has the wrong arity");
  return out;
}

std::string row_text(const double* v, int n) {
  std::string s;
  for (int i = 0; i < n; ++i) s += (i ? " " : "") + shortest(v[i]);
  return s;
}

void append_section(std::string& out, const char* name, const std::string& body) {
  const std::size_t lines = std::size_t(std::count(body.begin(), body.end(), '\n'));
  char head[96];
  std::snprintf(head, sizeof head, "section %s %zu %08x\n", name, lines, crc32_bytes(body.data(), body.size()));
  out += head;
  out += body;
}

// gaussian_kernel (image.cpp:163-175).
std::vector<double> gaussian_taps(double sigma) {
  const int r = static_cast<int>(std::ceil(3.0 * sigma));
  std::vector<double> t(std::size_t(2 * r + 1));
  double sum = 0.0;
  for (int j = -r; j <= r; ++j) {
    const double e = std::exp(-(static_cast<double>(j) * j) / (2.0 * sigma * sigma));
    t[std::size_t(j + r)] = e;
    sum += e;
  }
  for (double& e : t) e /= sum;
  return t;
}

// compute_beta (scale_space.cpp:56-73): the Vandermonde inverse through the
// reference's Eigen::FullPivLU — complete-pivoting LU, then solve(I) as
// FullPivLU::_solve_impl with triangular_solve_matrix's operation order
// (DESIGN.md §3). Bit-identical to the reference's own compute_beta built
// against oracle/refbuild (tests/test_ref_pin.py).
void vandermonde_inverse(const std::vector<double>& s, double OUT[4][4]) {
  double V[4][4];
  for (int k = 0; k < 4; ++k) {
    double pw = 1.0;
    for (int i = 0; i < 4; ++i) {
      V[k][i] = pw;
      pw *= s[std::size_t(k)];
    }
  }
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
}

void check_lut(const LutTable& t) {
  if (t.values.empty() || t.edges.size() != t.values.size() + 1) throw DataError("lookup table needs B+1 edges for B values");
  for (std::size_t i = 1; i < t.edges.size(); ++i)
    if (!(t.edges[i] > t.edges[i - 1])) throw DataError("lookup table edges must be increasing");
  for (double v : t.values)
    if (!(v >= 0.0 && v <= 1.0)) throw DataError("lookup table values must lie in [0, 1]");
}

// Eigen SSE2 redux order for a contiguous vector.
double packet_sum(const double* v, std::size_t n) {
  if (n < 2) return n ? v[0] : 0.0;
  if (n < 4) { double r = v[0] + v[1]; for (std::size_t i = 2; i < n; ++i) r += v[i]; return r; }
  const std::size_t e2 = n / 4 * 4, e1 = n / 2 * 2;
  double a0 = v[0], a1 = v[1], b0 = v[2], b1 = v[3];
  for (std::size_t i = 4; i < e2; i += 4) { a0 += v[i]; a1 += v[i + 1]; b0 += v[i + 2]; b1 += v[i + 3]; }
  a0 += b0; a1 += b1;
  if (e1 > e2) { a0 += v[e2]; a1 += v[e2 + 1]; }
  double r = a0 + a1;
  for (std::size_t i = e1; i < n; ++i) r += v[i];
  return r;
}

void validate(const Bundle& b) {
  if (b.select_n < 1) throw DataError("selection budget must be positive");
  for (const auto& t : b.relevance) check_lut(t);
  if (b.tr_scale == 0.0) throw DataError("transform scale must be nonzero");
  for (const auto* m : {&b.tr_a, &b.tr_b})
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double g = 0.0;
        for (int k = 0; k < 8; ++k) g += (*m)[i][k] * (*m)[j][k];
        if (i != j && std::abs(g) > 1e-9) throw DataError("transform rows are not orthogonal");
        if (i == j && g <= 0.0) throw DataError("transform has a zero row");
      }
  for (int e = 0; e < 128; ++e)
    if (!(b.t0[e] < b.t1[e])) throw DataError("quantizer thresholds must satisfy t0 < t1");
  int seen[128] = {};
  for (int e : b.priority)
    if (e < 0 || e >= 128 || seen[e]++) throw DataError("quantizer priority must be a permutation of 0..127");
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) {
      double s = 0.0;
      for (int k = 0; k < 128; ++k) s += b.pca_basis[std::size_t(i) * 128 + k] * b.pca_basis[std::size_t(j) * 128 + k];
      if (std::abs(s - (i == j ? 1.0 : 0.0)) > 1e-6) throw DataError("PCA basis rows are not orthonormal");
    }
  if (b.nc < 1) throw DataError("GMM needs at least one component");
  for (double w : b.weights)
    if (!(w > 0.0)) throw DataError("GMM weights must be positive");
  if (std::abs(packet_sum(b.weights.data(), b.weights.size()) - 1.0) > 1e-9) throw DataError("GMM weights must sum to 1");
  for (double s : b.stds)
    if (s < 1e-3 - 1e-15) throw DataError("GMM stds fall below the floor");
}

}  // namespace

uint32_t crc32_bytes(const void* data, std::size_t len) {
  static uint32_t table[256];
  static const bool init = [] {
    for (uint32_t n = 0; n < 256; ++n) {
      uint32_t c = n;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[n] = c;
    }
    return true;
  }();
  (void)init;
  const auto* p = static_cast<const uint8_t*>(data);
  uint32_t c = 0xFFFFFFFFu;
  for (std::size_t i = 0; i < len; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

std::string serialize_bundle(const Bundle& b) {
  std::string out = "CDVZ-MODEL 1\n";
  {
    std::string body = "num_octaves = " + std::to_string(b.num_octaves) + "\nsigmas =";
    for (double s : b.sigmas) body += " " + shortest(s);
    body += "\nresponse_threshold = " + shortest(b.response_threshold) + "\nedge_r = " + shortest(b.edge_r) + "\n";
    append_section(out, "detector", body);
  }
  {
    std::string body = "n = " + std::to_string(b.select_n) + "\nCDVZ-RELEVANCE 1\n";
    for (int c = 0; c < 5; ++c) {
      body += std::string(kLutNames[c]) + " bins:";
      for (double e : b.relevance[std::size_t(c)].edges) body += " " + shortest(e);
      body += " ; values:";
      for (double v : b.relevance[std::size_t(c)].values) body += " " + shortest(v);
      body += "\n";
    }
    append_section(out, "selector", body);
  }
  {
    std::string body;
    for (int r = 0; r < 8; ++r) body += row_text(b.tr_a[r], 8) + "\n";
    for (int r = 0; r < 8; ++r) body += row_text(b.tr_b[r], 8) + "\n";
    body += "scale = " + shortest(b.tr_scale) + "\n";
    append_section(out, "transforms", body);
  }
  {
    std::string body = row_text(b.t0, 128) + "\n" + row_text(b.t1, 128) + "\n";
    for (int e = 0; e < 128; ++e) body += (e ? " " : "") + std::to_string(b.priority[e]);
    body += "\n";
    for (int e = 0; e < 128; ++e) body += (e ? " " : "") + std::to_string(int(b.degenerate[e]));
    body += "\n";
    append_section(out, "quantizer", body);
  }
  {
    std::string body = row_text(b.pca_mean, 128) + "\n";
    for (int r = 0; r < 32; ++r) body += row_text(&b.pca_basis[std::size_t(r) * 128], 128) + "\n";
    append_section(out, "pca", body);
  }
  {
    std::string body = "components = " + std::to_string(b.nc) + "\n" + row_text(b.weights.data(), b.nc) + "\n";
    for (int i = 0; i < b.nc; ++i) body += row_text(&b.means[std::size_t(i) * 32], 32) + "\n";
    for (int i = 0; i < b.nc; ++i) body += row_text(&b.stds[std::size_t(i) * 32], 32) + "\n";
    append_section(out, "gmm", body);
  }
  return out + "end\n";
}

Bundle parse_bundle(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  std::getline(in, line);
  if (line != "CDVZ-MODEL 1") throw DataError("unsupported model bundle version");
  Bundle b;
  b.sigmas.resize(4);
  for (int k = 0; k < 4; ++k) b.sigmas[std::size_t(k)] = 1.4 * std::pow(2.0, k / 4.0);
  unsigned seen = 0;
  while (std::getline(in, line) && line != "end") {
    std::istringstream hs(line);
    std::string kw, name, crc_hex;
    std::size_t lines = 0;
    hs >> kw >> name >> lines >> crc_hex;
    if (kw != "section" || name.empty()) throw DataError("malformed model bundle section header");
    std::string body, l;
    for (std::size_t i = 0; i < lines; ++i) {
      if (!std::getline(in, l)) throw DataError("model bundle section truncated");
      body += l + "\n";
    }
    char computed[16];
    std::snprintf(computed, sizeof computed, "%08x", crc32_bytes(body.data(), body.size()));
    if (crc_hex != computed) throw DataError("model bundle section '" + name + "' checksum mismatch");
    std::istringstream bs(body);
    if (name == "detector") {
      while (std::getline(bs, l)) {
        const auto eq = l.find('=');
        if (eq == std::string::npos) continue;
        std::istringstream ks(l.substr(0, eq)), vs(l.substr(eq + 1));
        std::string key, tok;
        ks >> key;
        if (key == "num_octaves") vs >> b.num_octaves;
        else if (key == "sigmas") { b.sigmas.clear(); while (vs >> tok) b.sigmas.push_back(to_double(tok)); }
        else if (key == "response_threshold") { vs >> tok; b.response_threshold = to_double(tok); }
        else if (key == "edge_r") { vs >> tok; b.edge_r = to_double(tok); }
        else throw DataError("unknown detector key: " + key);
      }
      seen |= 1;
    } else if (name == "selector") {
      std::getline(bs, l);
      std::istringstream ns(l);
      std::string k, eq;
      ns >> k >> eq >> b.select_n;
      if (k != "n" || eq != "=") throw DataError("malformed selector section");
      std::getline(bs, l);
      if (l != "CDVZ-RELEVANCE 1") throw DataError("unsupported relevance table version");
      bool got[5] = {};
      while (std::getline(bs, l)) {
        if (l.empty()) continue;
        std::istringstream ls(l);
        std::string nm, tag, tok;
        ls >> nm >> tag;
        if (tag != "bins:") throw DataError("malformed relevance table line: " + l);
        int idx = -1;
        for (int c = 0; c < 5; ++c)
          if (nm == kLutNames[c]) idx = c;
        if (idx < 0) throw DataError("unknown characteristic: " + nm);
        LutTable t;
        while (ls >> tok && tok != ";") t.edges.push_back(to_double(tok));
        ls >> tag;
        if (tag != "values:") throw DataError("malformed relevance table line: " + l);
        while (ls >> tok) t.values.push_back(to_double(tok));
        check_lut(t);
        b.relevance[std::size_t(idx)] = std::move(t);
        got[idx] = true;
      }
      for (bool g : got)
        if (!g) throw DataError("relevance table file is missing a characteristic");
      seen |= 2;
    } else if (name == "transforms") {
      for (int r = 0; r < 16; ++r) {
        if (!std::getline(bs, l)) throw DataError("transform section truncated");
        const auto v = numbers(l, 8);
        for (int j = 0; j < 8; ++j) (r < 8 ? b.tr_a[r] : b.tr_b[r - 8])[j] = v[std::size_t(j)];
      }
      if (!std::getline(bs, l)) throw DataError("transform section truncated");
      std::istringstream ss(l);
      std::string k, eq, tok;
      ss >> k >> eq >> tok;
      if (k != "scale" || eq != "=") throw DataError("malformed transform scale line");
      b.tr_scale = to_double(tok);
      seen |= 4;
    } else if (name == "quantizer") {
      std::getline(bs, l);
      auto a = numbers(l, 128);
      std::getline(bs, l);
      auto c = numbers(l, 128);
      for (int e = 0; e < 128; ++e) { b.t0[e] = a[std::size_t(e)]; b.t1[e] = c[std::size_t(e)]; }
      std::getline(bs, l);
      std::istringstream ps(l);
      for (int e = 0; e < 128; ++e)
        if (!(ps >> b.priority[e])) throw DataError("quantizer priority truncated");
      std::getline(bs, l);
      std::istringstream ds(l);
      for (int e = 0; e < 128; ++e) {
        int f = 0;
        if (!(ds >> f)) throw DataError("quantizer flags truncated");
        b.degenerate[e] = uint8_t(f);
      }
      seen |= 8;
    } else if (name == "pca") {
      std::getline(bs, l);
      const auto mu = numbers(l, 128);
      std::copy(mu.begin(), mu.end(), b.pca_mean);
      b.pca_basis.clear();
      for (int r = 0; r < 32; ++r) {
        if (!std::getline(bs, l)) throw DataError("pca section truncated");
        const auto v = numbers(l, 128);
        b.pca_basis.insert(b.pca_basis.end(), v.begin(), v.end());
      }
      seen |= 16;
    } else if (name == "gmm") {
      std::getline(bs, l);
      std::istringstream cs(l);
      std::string k, eq;
      int nc = 0;
      cs >> k >> eq >> nc;
      if (k != "components" || eq != "=" || nc < 1) throw DataError("malformed gmm section");
      b.nc = nc;
      std::getline(bs, l);
      b.weights = numbers(l, nc);
      b.means.clear();
      b.stds.clear();
      for (int part = 0; part < 2; ++part)
        for (int i = 0; i < nc; ++i) {
          if (!std::getline(bs, l)) throw DataError("gmm section truncated");
          const auto v = numbers(l, 32);
          auto& dst = part ? b.stds : b.means;
          dst.insert(dst.end(), v.begin(), v.end());
        }
      seen |= 32;
    } else {
      throw DataError("unknown model bundle section: " + name);
    }
  }
  if (seen != 63) throw DataError("model bundle is missing sections");

  // finalize() (scale_space.cpp:75-83)
  if (b.sigmas.size() != 4) throw DataError("config requires 4 scales");
  for (std::size_t k = 1; k < 4; ++k)
    if (!(b.sigmas[k] > b.sigmas[k - 1])) throw DataError("scales must be strictly increasing");
  if (!(b.sigmas[0] > 0.0)) throw DataError("scales must be positive");
  if (b.num_octaves < 1) throw DataError("at least one octave is required");
  if (!(b.edge_r > 0.0)) throw DataError("edge ratio parameter must be positive");
  vandermonde_inverse(b.sigmas, b.beta);
  validate(b);

  for (int k = 0; k < 4; ++k) {
    b.taps[k] = gaussian_taps(b.sigmas[std::size_t(k)]);
    b.radius[k] = int(b.taps[k].size() / 2);
  }
  // The blur kernels are instantiated for radii up to 8 (setup_model): one limit for
  // cdvz_gpu_bundle_check and cdvz_gpu_create alike.
  if (b.radius[3] > 8) throw UsageError("detector scales above sigma 2.66 (Gaussian radius > 8) are not supported by the GPU kernels");
  b.margin = static_cast<int>(std::ceil(3.0 * b.sigmas[3])) + 2;
  b.rho_limit = (b.edge_r + 1.0) * (b.edge_r + 1.0) / b.edge_r;
  const std::string canon = serialize_bundle(b);
  b.model_crc = crc32_bytes(canon.data(), canon.size());
  return b;
}

const Mode& mode_by_id(int id) {
  static const Mode modes[6] = {
      {0, "512B", 512, 20, 32.0 / 512.0, false},  {1, "1K", 1024, 32, 64.0 / 512.0, false},
      {2, "2K", 2048, 64, 128.0 / 512.0, false},  {3, "4K", 4096, 103, 256.0 / 512.0, false},
      {4, "8K", 8192, 103, 320.0 / 512.0, true},  {5, "16K", 16384, 128, 512.0 / 512.0, true},
  };
  for (const auto& m : modes)
    if (m.id == id) return m;
  throw DataError("unknown mode id " + std::to_string(id));
}

Budget budget_for(const Mode& m, int nc) {
  Budget b;
  b.k = std::min(nc, std::max(1, static_cast<int>(std::lround(nc * m.fraction))));
  b.global_bytes = std::size_t((nc + 7) / 8) + std::size_t(b.k) * (m.variance ? 8 : 4);
  if (b.global_bytes + 4 > m.budget) throw DataError("global descriptor alone exceeds the mode budget");
  b.code_bytes = 6 + (std::size_t(m.elements) * 2 + 7) / 8;
  b.max_codes = (m.budget - b.global_bytes - 4) / b.code_bytes;
  return b;
}

// Public forms of two helpers the trainer shares (train_host.cpp, context.cu).
std::vector<double> gaussian_kernel_taps(double sigma) { return gaussian_taps(sigma); }
double eigen_packet_sum(const double* v, std::size_t n) { return packet_sum(v, n); }

}  // namespace cdvz_gpu
