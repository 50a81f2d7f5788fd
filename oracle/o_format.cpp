// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/model_io.cpp and proj/src/container.cpp.
#include <cstdio>
#include <sstream>

#include "oracle.hpp"

namespace orc {

namespace {

const char* kStatNames[5] = {"sigma", "p", "d", "rho", "pss"};  // relevance.hpp:26-27

std::string join_doubles(const double* v, int n) {
  std::string s;
  for (int i = 0; i < n; ++i) {
    if (i) s += ' ';
    s += format_double(v[i]);
  }
  return s;
}

std::vector<double> split_doubles(const std::string& line, int expect) {
  std::istringstream in(line);
  std::vector<double> v;
  std::string tok;
  while (in >> tok) v.push_back(parse_double(tok));
  if (expect >= 0 && int(v.size()) != expect) throw DataError("model bundle row has the wrong arity");
  return v;
}

// model_io.cpp:12-19
void emit_section(std::string& out, const char* name, const std::string& body) {
  std::size_t lines = 0;
  for (char c : body) lines += (c == '\n');
  char head[96];
  std::snprintf(head, sizeof head, "section %s %zu %08x\n", name, lines, crc32(body.data(), body.size()));
  out += head;
  out += body;
}

// relevance.cpp:173-184
std::string relevance_text(const RelevanceModel& m) {
  std::string s = "CDVZ-RELEVANCE 1\n";
  for (int c = 0; c < 5; ++c) {
    const auto& t = m.tables[std::size_t(c)];
    s += kStatNames[c];
    s += " bins:";
    for (double e : t.edges) s += " " + format_double(e);
    s += " ; values:";
    for (double v : t.values) s += " " + format_double(v);
    s += "\n";
  }
  return s;
}

// relevance.cpp:186-214
RelevanceModel parse_relevance(std::istream& in) {
  std::string header;
  std::getline(in, header);
  if (header != "CDVZ-RELEVANCE 1") throw DataError("unsupported relevance table version");
  RelevanceModel m;
  bool seen[5] = {false, false, false, false, false};
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string name, kw, tok;
    ls >> name >> kw;
    if (kw != "bins:") throw DataError("malformed relevance table line: " + line);
    int idx = -1;
    for (int c = 0; c < 5; ++c)
      if (name == kStatNames[c]) idx = c;
    if (idx < 0) throw DataError("unknown characteristic: " + name);
    LookupTable t;
    while (ls >> tok && tok != ";") t.edges.push_back(parse_double(tok));
    ls >> kw;
    if (kw != "values:") throw DataError("malformed relevance table line: " + line);
    while (ls >> tok) t.values.push_back(parse_double(tok));
    t.validate();
    m.tables[std::size_t(idx)] = std::move(t);
    seen[idx] = true;
  }
  for (bool s : seen)
    if (!s) throw DataError("relevance table file is missing a characteristic");
  return m;
}

}  // namespace

void ModelBundle::validate() const {
  if (select_n < 1) throw DataError("selection budget must be positive");
  relevance.validate();
  transforms.validate();
  quantizer.validate();
  pca.validate();
  gmm.validate();
}

uint32_t ModelBundle::crc() const {
  const std::string t = serialize_model(*this);
  return crc32(t.data(), t.size());
}

// model_io.cpp:86-139
std::string serialize_model(const ModelBundle& b) {
  std::string out = "CDVZ-MODEL 1\n";
  {
    std::string body = "num_octaves = " + std::to_string(b.detector.num_octaves) + "\n";
    body += "sigmas =";
    for (double s : b.detector.sigmas) body += " " + format_double(s);
    body += "\n";
    body += "response_threshold = " + format_double(b.detector.response_threshold) + "\n";
    body += "edge_r = " + format_double(b.detector.edge_r) + "\n";
    emit_section(out, "detector", body);
  }
  emit_section(out, "selector", "n = " + std::to_string(b.select_n) + "\n" + relevance_text(b.relevance));
  {
    std::string body;
    for (int r = 0; r < 8; ++r) body += join_doubles(b.transforms.a[std::size_t(r)].data(), 8) + "\n";
    for (int r = 0; r < 8; ++r) body += join_doubles(b.transforms.b[std::size_t(r)].data(), 8) + "\n";
    body += "scale = " + format_double(b.transforms.scale) + "\n";
    emit_section(out, "transforms", body);
  }
  {
    std::string body = join_doubles(b.quantizer.t0.data(), 128) + "\n" + join_doubles(b.quantizer.t1.data(), 128) + "\n";
    for (int e = 0; e < 128; ++e) body += (e ? " " : "") + std::to_string(b.quantizer.priority[std::size_t(e)]);
    body += "\n";
    for (int e = 0; e < 128; ++e) body += (e ? " " : "") + std::to_string(int(b.quantizer.degenerate[std::size_t(e)]));
    body += "\n";
    emit_section(out, "quantizer", body);
  }
  {
    std::string body = join_doubles(b.pca.mean.data(), 128) + "\n";
    for (int r = 0; r < 32; ++r) body += join_doubles(&b.pca.basis.a[std::size_t(r) * 128], 128) + "\n";
    emit_section(out, "pca", body);
  }
  {
    const int nc = b.gmm.components();
    std::string body = "components = " + std::to_string(nc) + "\n";
    body += join_doubles(b.gmm.weights.data(), nc) + "\n";
    for (int i = 0; i < nc; ++i) body += join_doubles(&b.gmm.means.a[std::size_t(i) * 32], 32) + "\n";
    for (int i = 0; i < nc; ++i) body += join_doubles(&b.gmm.stds.a[std::size_t(i) * 32], 32) + "\n";
    emit_section(out, "gmm", body);
  }
  out += "end\n";
  return out;
}

// model_io.cpp:141-273
ModelBundle parse_model(const std::string& text) {
  std::istringstream in(text);
  std::string header;
  std::getline(in, header);
  if (header != "CDVZ-MODEL 1") throw DataError("unsupported model bundle version");
  ModelBundle b;
  b.detector = DetectorConfig::defaults();
  bool seen_det = false, seen_sel = false, seen_tr = false, seen_q = false, seen_pca = false, seen_gmm = false;
  std::string head;
  while (std::getline(in, head)) {
    if (head == "end") break;
    std::istringstream hs(head);
    std::string kw, name, crc_hex;
    std::size_t lines = 0;
    hs >> kw >> name >> lines >> crc_hex;
    if (kw != "section" || name.empty()) throw DataError("malformed model bundle section header");
    std::string body, line;
    for (std::size_t i = 0; i < lines; ++i) {
      if (!std::getline(in, line)) throw DataError("model bundle section truncated");
      body += line;
      body += '\n';
    }
    char computed[16];
    std::snprintf(computed, sizeof computed, "%08x", crc32(body.data(), body.size()));
    if (crc_hex != computed)
      throw DataError("model bundle section '" + name + "' checksum mismatch (" + crc_hex + " vs " + computed + ", " +
                      std::to_string(body.size()) + " bytes)");
    std::istringstream bs(body);
    if (name == "detector") {
      while (std::getline(bs, line)) {
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        std::istringstream ks(line.substr(0, eq)), vs(line.substr(eq + 1));
        std::string key, tok;
        ks >> key;
        if (key == "num_octaves") vs >> b.detector.num_octaves;
        else if (key == "sigmas") {
          b.detector.sigmas.clear();
          while (vs >> tok) b.detector.sigmas.push_back(parse_double(tok));
        } else if (key == "response_threshold") { vs >> tok; b.detector.response_threshold = parse_double(tok); }
        else if (key == "edge_r") { vs >> tok; b.detector.edge_r = parse_double(tok); }
        else throw DataError("unknown detector key: " + key);
      }
      b.detector.finalize();
      seen_det = true;
    } else if (name == "selector") {
      std::getline(bs, line);
      std::istringstream ns(line);
      std::string k, eq;
      ns >> k >> eq >> b.select_n;
      if (k != "n" || eq != "=") throw DataError("malformed selector section");
      b.relevance = parse_relevance(bs);
      seen_sel = true;
    } else if (name == "transforms") {
      for (int r = 0; r < 16; ++r) {
        if (!std::getline(bs, line)) throw DataError("transform section truncated");
        const auto v = split_doubles(line, 8);
        auto& row = r < 8 ? b.transforms.a[std::size_t(r)] : b.transforms.b[std::size_t(r - 8)];
        for (int j = 0; j < 8; ++j) row[std::size_t(j)] = v[std::size_t(j)];
      }
      if (!std::getline(bs, line)) throw DataError("transform section truncated");
      std::istringstream ss(line);
      std::string k, eq, tok;
      ss >> k >> eq >> tok;
      if (k != "scale" || eq != "=") throw DataError("malformed transform scale line");
      b.transforms.scale = parse_double(tok);
      seen_tr = true;
    } else if (name == "quantizer") {
      std::getline(bs, line);
      auto t0 = split_doubles(line, 128);
      std::getline(bs, line);
      auto t1 = split_doubles(line, 128);
      for (int e = 0; e < 128; ++e) { b.quantizer.t0[std::size_t(e)] = t0[std::size_t(e)]; b.quantizer.t1[std::size_t(e)] = t1[std::size_t(e)]; }
      std::getline(bs, line);
      {
        std::istringstream ps(line);
        for (int e = 0; e < 128; ++e)
          if (!(ps >> b.quantizer.priority[std::size_t(e)])) throw DataError("quantizer priority truncated");
      }
      std::getline(bs, line);
      {
        std::istringstream ds(line);
        for (int e = 0; e < 128; ++e) {
          int f = 0;
          if (!(ds >> f)) throw DataError("quantizer flags truncated");
          b.quantizer.degenerate[std::size_t(e)] = uint8_t(f);
        }
      }
      seen_q = true;
    } else if (name == "pca") {
      std::getline(bs, line);
      const auto mu = split_doubles(line, 128);
      for (int j = 0; j < 128; ++j) b.pca.mean[std::size_t(j)] = mu[std::size_t(j)];
      for (int r = 0; r < 32; ++r) {
        if (!std::getline(bs, line)) throw DataError("pca section truncated");
        const auto v = split_doubles(line, 128);
        for (int j = 0; j < 128; ++j) b.pca.basis(r, j) = v[std::size_t(j)];
      }
      seen_pca = true;
    } else if (name == "gmm") {
      std::getline(bs, line);
      std::istringstream cs(line);
      std::string k, eq;
      int nc = 0;
      cs >> k >> eq >> nc;
      if (k != "components" || eq != "=" || nc < 1) throw DataError("malformed gmm section");
      std::getline(bs, line);
      b.gmm.weights = split_doubles(line, nc);
      b.gmm.means = Mat(nc, 32);
      b.gmm.stds = Mat(nc, 32);
      for (int part = 0; part < 2; ++part)
        for (int i = 0; i < nc; ++i) {
          if (!std::getline(bs, line)) throw DataError("gmm section truncated");
          const auto v = split_doubles(line, 32);
          for (int j = 0; j < 32; ++j) (part == 0 ? b.gmm.means : b.gmm.stds)(i, j) = v[std::size_t(j)];
        }
      seen_gmm = true;
    } else {
      throw DataError("unknown model bundle section: " + name);
    }
  }
  if (!(seen_det && seen_sel && seen_tr && seen_q && seen_pca && seen_gmm)) throw DataError("model bundle is missing sections");
  b.validate();
  return b;
}

// ---------------------------------------------------------------- container

namespace {
void put16(std::vector<uint8_t>& o, uint16_t v) { o.push_back(uint8_t(v & 0xFF)); o.push_back(uint8_t(v >> 8)); }
void put32(std::vector<uint8_t>& o, uint32_t v) { for (int i = 0; i < 4; ++i) o.push_back(uint8_t((v >> (8 * i)) & 0xFF)); }
uint32_t get32(const std::vector<uint8_t>& b, std::size_t off) {
  return uint32_t(b[off]) | (uint32_t(b[off + 1]) << 8) | (uint32_t(b[off + 2]) << 16) | (uint32_t(b[off + 3]) << 24);
}
}  // namespace

// container.cpp:32-58 — "CDVZ1" | mode | w | h | nc | model_crc | global_len |
// local_len | global | local | crc32(all previous bytes), little endian.
std::vector<uint8_t> serialize_container(const EncodedImage& e) {
  const ModeSpec& mode = mode_by_id(e.mode_id);
  const auto g = serialize_scfv(e.global_desc);
  const auto l = pack_local(e.codes, mode);
  if (g.size() + l.size() > mode.budget_bytes) throw DataError("encoded payload exceeds the mode budget");
  if (e.width < 1 || e.width > 0xFFFF || e.height < 1 || e.height > 0xFFFF)
    throw DataError("image dimensions do not fit the container header");
  if (e.global_desc.n_components < 1 || e.global_desc.n_components > 0xFFFF)
    throw DataError("component count does not fit the container header");
  std::vector<uint8_t> out = {'C', 'D', 'V', 'Z', '1'};
  out.push_back(uint8_t(e.mode_id));
  put16(out, uint16_t(e.width));
  put16(out, uint16_t(e.height));
  put16(out, uint16_t(e.global_desc.n_components));
  put32(out, e.model_crc);
  put32(out, uint32_t(g.size()));
  put32(out, uint32_t(l.size()));
  out.insert(out.end(), g.begin(), g.end());
  out.insert(out.end(), l.begin(), l.end());
  put32(out, crc32(out.data(), out.size()));
  return out;
}

// container.cpp:60-93
EncodedImage parse_container(const std::vector<uint8_t>& b) {
  if (b.size() < kContainerHeaderBytes + kContainerTrailerBytes) throw DataError("container truncated");
  const char magic[5] = {'C', 'D', 'V', 'Z', '1'};
  for (int i = 0; i < 5; ++i)
    if (b[std::size_t(i)] != uint8_t(magic[i])) throw DataError("container magic mismatch");
  const std::size_t body = b.size() - kContainerTrailerBytes;
  if (crc32(b.data(), body) != get32(b, body)) throw DataError("container checksum mismatch");
  EncodedImage e;
  e.mode_id = b[5];
  const ModeSpec& mode = mode_by_id(e.mode_id);
  e.width = b[6] | (b[7] << 8);
  e.height = b[8] | (b[9] << 8);
  const int nc = b[10] | (b[11] << 8);
  e.model_crc = get32(b, 12);
  const std::size_t gl = get32(b, 16), ll = get32(b, 20);
  if (kContainerHeaderBytes + gl + ll != body) throw DataError("container section lengths disagree with its size");
  const std::vector<uint8_t> g(b.begin() + long(kContainerHeaderBytes), b.begin() + long(kContainerHeaderBytes + gl));
  const std::vector<uint8_t> l(b.begin() + long(kContainerHeaderBytes + gl), b.begin() + long(body));
  e.global_desc = parse_scfv(g, nc, mode.variance_planes);
  e.codes = unpack_local(l);
  return e;
}

}  // namespace orc
