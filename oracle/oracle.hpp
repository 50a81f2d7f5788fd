// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// An Eigen-free, line-faithful C++ restatement of the reference extractor
// (/root/reference/proj, "cdvz", arxiv 1705.09776) used as the parity checker
// for the B200 product in paper_1705_09776_b200/. Only tests/, the smoke check
// in __graft_entry__.py and bench.py's cpu_baseline leg may load it. The
// product library never links or calls anything in this directory.
//
// Pinning status: the reference itself cannot be compiled in
// this image (Eigen3, doctest and CLI11 are absent, no network), so the oracle
// is pinned against the reference's own known-answer tests, ported in
// oracle/selftest.cpp, not against a reference binary. Where the reference's
// arithmetic order lives inside Eigen (dense products, vector reductions) the
// order chosen here is stated at the call site; the GPU product reproduces the
// oracle's order so the two agree bit-for-bit wherever libm is not involved.
//
// Every function cites the reference file:line it restates.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace orc {

struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- common
// proj/src/common.cpp:11-35
uint32_t crc32(const void* data, std::size_t len, uint32_t seed = 0);
// proj/include/cdvz/common.hpp:24-30
inline long mirror_index(long i, long n) {
  if (n <= 1) return 0;
  const long period = 2 * n;
  long m = i % period;
  if (m < 0) m += period;
  return m < n ? m : period - 1 - m;
}
// proj/src/common.cpp:37-57
std::string format_double(double v);
double parse_double(std::string_view s);

// Eigen's SSE2 linear-vectorized redux order for a contiguous vector
// (two 2-lane packet accumulators, tail added last): (s0+s2)+(s1+s3) where
// s_l sums the elements whose index is l mod 4. Used wherever the reference
// calls .sum()/.norm()/.mean() on a contiguous Eigen vector.
double eigen_sum(const double* v, std::size_t n);

// ---------------------------------------------------------------- image
// Row-major raster; proj/include/cdvz/image.hpp:11-18.
struct Plane {
  int w = 0, h = 0;
  std::vector<double> px;
  Plane() = default;
  Plane(int w_, int h_, double fill = 0.0) : w(w_), h(h_), px(std::size_t(w_) * h_, fill) {}
  double& at(int y, int x) { return px[std::size_t(y) * w + x]; }
  double at(int y, int x) const { return px[std::size_t(y) * w + x]; }
};

void validate_plane(const Plane& img);                                  // image.cpp:46-51
Plane plane_from_u8(const uint8_t* bytes, int w, int h, std::size_t stride);  // image.cpp:79-87
Plane plane_from_rgb(const uint8_t* rgb, int w, int h, std::size_t stride);    // image.cpp:82-86
std::vector<uint8_t> plane_to_u8(const Plane& img);                     // image.cpp:101-102 (save_pgm)
Plane rescale_bilinear(const Plane& img, int out_w, int out_h);         // image.cpp:107-129
Plane resize_max_side(const Plane& img, int limit = 640);               // image.cpp:131-145
Plane downsample_half(const Plane& img);                                // image.cpp:147-155
std::vector<double> gaussian_taps(double sigma);                        // image.cpp:163-175
Plane gaussian_blur(const Plane& img, double sigma);                    // image.cpp:177-212
Plane laplacian_3x3(const Plane& img);                                  // image.cpp:220-238

// ---------------------------------------------------------------- synthetic
Plane synth_image(uint64_t seed, int w, int h);                         // synthetic.cpp:11-53
uint64_t corpus_seed(uint64_t base, int i);                             // synthetic.cpp:55-61
Plane rotate90(const Plane& img, int quarter_turns);                    // synthetic.cpp:63-76
struct SynthTransform { int quarter_turns = 0; double scale = 1.0; double blur_sigma = 0.0; };
Plane apply_transform(const Plane& img, const SynthTransform& t);       // synthetic.cpp:78-90
void map_point(const SynthTransform& t, int src_w, int src_h, double& x, double& y, double& s);  // :92-111

// ---------------------------------------------------------------- detector
using Mat4 = std::array<std::array<double, 4>, 4>;

struct DetectorConfig {                 // scale_space.hpp:16-27
  int num_octaves = 4;
  std::vector<double> sigmas;
  double response_threshold = 0.02;
  double edge_r = 10.0;
  Mat4 beta{};
  double rho_limit() const { return (edge_r + 1.0) * (edge_r + 1.0) / edge_r; }
  void finalize();                      // scale_space.cpp:75-83
  static DetectorConfig defaults();     // scale_space.cpp:85-91
};
Mat4 compute_beta(const std::vector<double>& sigmas);  // scale_space.cpp:56-73

struct Octave {                          // scale_space.hpp:33-38
  int index = 0;
  Plane base;
  std::vector<Plane> gauss, log;
};
Octave build_octave(const Plane& base, const DetectorConfig& cfg, int index);  // scale_space.cpp:141-153

struct Candidate { int x = 0, y = 0; double sigma = 0.0, p = 0.0; };          // scale_space.hpp:44-48
std::vector<Candidate> detect_extrema(const Octave& oct, const DetectorConfig& cfg);  // :155-215

struct Keypoint {                        // scale_space.hpp:56-64 (InterestPoint)
  double x = 0, y = 0, sigma = 0;
  int octave = 0;
  double p = 0, rho = 0, p_ss = 0, d = 0;
};
std::vector<Keypoint> refine_candidates(const std::vector<Candidate>& c, const Octave& oct,
                                        const DetectorConfig& cfg);   // :217-270
std::vector<Keypoint> dedup_across_octaves(const std::vector<Keypoint>& cur,
                                           const std::vector<Keypoint>& prev);  // :272-302

struct Pyramid { std::vector<Octave> octaves; };
struct DetectTrace {                     // per-octave intermediates for stage parity
  std::vector<std::vector<Candidate>> candidates;
  std::vector<std::vector<Keypoint>> refined;
};
std::vector<Keypoint> detect_keypoints(const Plane& img, const DetectorConfig& cfg,
                                       Pyramid* pyr, DetectTrace* trace = nullptr);  // :304-326

// ---------------------------------------------------------------- selector
struct LookupTable {                     // relevance.hpp:30-38
  std::vector<double> edges, values;
  double operator()(double x) const;     // relevance.cpp:24-30
  void validate() const;
};
struct RelevanceModel {
  std::array<LookupTable, 5> tables;     // sigma, p, d, rho, pss
  void validate() const;
  static RelevanceModel uniform();
};
double relevance(const Keypoint& k, const RelevanceModel& m);          // relevance.cpp:54-59
void fill_center_distance(std::vector<Keypoint>& pts, int w, int h);   // relevance.cpp:61-69
std::vector<Keypoint> select_top(const std::vector<Keypoint>& pts, const RelevanceModel& m,
                                 std::size_t n);                      // relevance.cpp:71-93
struct Labeled { Keypoint k; bool matched = false; };
RelevanceModel train_relevance_tables(const std::vector<Labeled>& s, int bins = 16,
                                      int min_bin_samples = 10);      // relevance.cpp:95-149
std::vector<Labeled> label_matches_by_geometry(const std::vector<Keypoint>& a,
                                               const std::vector<Keypoint>& b,
                                               const std::vector<std::array<double, 3>>& mapped,
                                               double xy_tol = 2.0, double ratio_tol = 1.3);  // :151-171

// ---------------------------------------------------------------- descriptor
struct OrientedPoint { Keypoint pt; double theta = 0.0; };
struct RawDescriptor { std::array<double, 128> v{}; OrientedPoint point; };
struct LocalFrame { const Plane* level = nullptr; int level_index = 0; double x = 0, y = 0, sigma = 0; };
LocalFrame resolve_frame(const Pyramid& pyr, const std::vector<double>& sigmas, const Keypoint& k);  // descriptor.cpp:149-170
std::vector<double> dominant_orientations(const Plane& lvl, double x, double y, double sigma);    // :172-232
std::array<double, 128> describe(const Plane& lvl, double x, double y, double sigma, double theta);  // :234-241
std::array<double, 128> normalize_descriptor(std::array<double, 128> v);                          // :124-139
std::vector<OrientedPoint> assign_orientations(const Pyramid& pyr, const std::vector<double>& sigmas,
                                               const std::vector<Keypoint>& pts);   // :243-256
std::vector<RawDescriptor> describe_batch(const Pyramid& pyr, const std::vector<double>& sigmas,
                                          const std::vector<OrientedPoint>& pts);  // :258-304

// ---------------------------------------------------------------- coding
struct ModeSpec {                        // transform_coding.hpp:13-20
  int id; const char* name; std::size_t budget_bytes; int elements; double scfv_fraction; bool variance_planes;
};
const std::array<ModeSpec, 6>& default_modes();   // transform_coding.cpp:21-31
const ModeSpec& mode_by_id(int id);
const ModeSpec& mode_by_name(const std::string& name);

using Mat8 = std::array<std::array<double, 8>, 8>;
struct TransformPair {                   // transform_coding.hpp:30-37
  Mat8 a{}, b{};
  double scale = 1.0;
  void validate() const;
  static TransformPair defaults();       // transform_coding.cpp:59-79
};
std::array<double, 128> transform_descriptor(const std::array<double, 128>& raw, const TransformPair& tp);  // :81-91
std::array<double, 128> inverse_transform_descriptor(const std::array<double, 128>& t, const TransformPair& tp);

struct QuantizerModel {                  // transform_coding.hpp:47-53
  std::array<double, 128> t0{}, t1{};
  std::array<int, 128> priority{};
  std::array<uint8_t, 128> degenerate{};
  void validate() const;
  static QuantizerModel neutral();
};
QuantizerModel train_thresholds(const std::vector<std::array<double, 128>>& rows, double p0 = 1.0 / 3.0);  // :126-171

struct TernaryCode {                     // transform_coding.hpp:57-63
  uint16_t xq = 0, yq = 0;
  uint8_t sigma_q = 0, theta_q = 0, mode = 0;
  std::vector<int8_t> symbols;
};
uint16_t quantize_coord(double v, int extent);      // transform_coding.cpp:173-177
double dequantize_coord(uint16_t q, int extent);
uint8_t quantize_sigma_log(double sigma);           // :183-187
double dequantize_sigma_log(uint8_t q);
uint8_t quantize_theta(double theta);               // :194-198
double dequantize_theta(uint8_t q);
TernaryCode quantize_ternary(const std::array<double, 128>& t, const QuantizerModel& qm, const ModeSpec& mode);  // :202-217
int ternary_distance(const TernaryCode& a, const TernaryCode& b);
std::size_t packed_code_bytes(int elements);
constexpr std::size_t kLocalHeaderBytes = 4;
std::vector<uint8_t> pack_local(const std::vector<TernaryCode>& codes, const ModeSpec& mode);  // :232-270
std::vector<TernaryCode> unpack_local(const std::vector<uint8_t>& bytes);                   // :272-305

// ---------------------------------------------------------------- global (SCFV)
// Dense row-major matrix.
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c, double fill = 0.0) : rows(r), cols(c), a(std::size_t(r) * c, fill) {}
  double& operator()(int r, int c) { return a[std::size_t(r) * cols + c]; }
  double operator()(int r, int c) const { return a[std::size_t(r) * cols + c]; }
};
struct PCAModel {                         // scfv.hpp:12-16
  std::array<double, 128> mean{};
  Mat basis = Mat(32, 128);
  void validate() const;
};
struct GMMModel {                         // scfv.hpp:18-24
  std::vector<double> weights;
  Mat means, stds;                        // nc x 32
  int components() const { return int(weights.size()); }
  void validate() const;
};
constexpr double kGmmSigmaFloor = 1e-3;
struct SCFVDescriptor {                   // scfv.hpp:30-40
  int n_components = 0;
  bool has_variance = false;
  std::vector<uint8_t> mask;
  std::vector<uint32_t> mean_planes, var_planes;
  std::vector<double> norms;
  bool selected(int i) const;
  int popcount() const;
};
Mat pca_reduce(const Mat& raw_rows, const PCAModel& pca);                  // scfv.cpp:82-85
Mat posteriors_naive(const Mat& x, const GMMModel& g);                     // scfv.cpp:94-98
Mat fv_mean_naive(const Mat& x, const Mat& gamma, const GMMModel& g);      // scfv.cpp:100-117
Mat fv_var_naive(const Mat& x, const Mat& gamma, const GMMModel& g);       // scfv.cpp:119-138
Mat posteriors_matrix(const Mat& x, const GMMModel& g);                    // scfv.cpp:140-164
Mat fv_mean_matrix(const Mat& x, const Mat& gamma, const GMMModel& g);     // scfv.cpp:166-180
Mat fv_var_matrix(const Mat& x, const Mat& gamma, const GMMModel& g);      // scfv.cpp:182-203
double scfv_delta(const double* g, int n);                                 // scfv.cpp:205-208
SCFVDescriptor scfv_encode(const Mat& gm, const Mat& gv, const GMMModel& g, const ModeSpec& mode);  // :210-253
double scfv_similarity(const SCFVDescriptor& a, const SCFVDescriptor& b);  // :255-278
std::size_t scfv_serialized_bytes(int nc, int selected, bool has_variance);
std::vector<uint8_t> serialize_scfv(const SCFVDescriptor& d);              // :285-298
SCFVDescriptor parse_scfv(const std::vector<uint8_t>& bytes, int nc, bool has_variance);
PCAModel train_pca(const Mat& corpus);                                     // :328-352
GMMModel train_gmm(const Mat& corpus32, int nc, int iterations, uint64_t seed,
                   std::vector<double>* loglik = nullptr);                 // :354-430

// ---------------------------------------------------------------- model bundle / container
struct ModelBundle {                      // model_io.hpp:14-26
  DetectorConfig detector;
  int select_n = 300;
  RelevanceModel relevance;
  TransformPair transforms;
  QuantizerModel quantizer;
  PCAModel pca;
  GMMModel gmm;
  void validate() const;
  uint32_t crc() const;
};
std::string serialize_model(const ModelBundle& b);   // model_io.cpp:86-139
ModelBundle parse_model(const std::string& text);    // model_io.cpp:141-273

struct EncodedImage {                     // container.hpp:19-25
  int mode_id = 0, width = 0, height = 0;
  uint32_t model_crc = 0;
  SCFVDescriptor global_desc;
  std::vector<TernaryCode> codes;
};
constexpr std::size_t kContainerHeaderBytes = 24, kContainerTrailerBytes = 4;
std::vector<uint8_t> serialize_container(const EncodedImage& e);   // container.cpp:32-58
EncodedImage parse_container(const std::vector<uint8_t>& bytes);   // container.cpp:60-93

// ---------------------------------------------------------------- pipeline
struct StageTimes { double ms[5] = {0, 0, 0, 0, 0}; };   // detection..aggregation
// Everything encode_image computes, for stage-level parity checks.
struct EncodeTrace {
  int prep_w = 0, prep_h = 0;
  DetectTrace detect;
  std::vector<Keypoint> keypoints, selected;
  std::vector<OrientedPoint> oriented;
  std::vector<RawDescriptor> descriptors;
  Mat x, gamma, gm, gv;
};
// pipeline.cpp:54-97
EncodedImage encode_image(const Plane& img, const ModelBundle& b, const ModeSpec& mode,
                          int max_side = 640, StageTimes* times = nullptr, EncodeTrace* trace = nullptr);
// ---------------------------------------------------------------- eval (eval.hpp)
struct MatchOptions { double ratio_test = 0.85; int rerank_depth = 50; };   // eval.hpp:32-35
struct MatchResult { double global_similarity = -1.0; int local_match_count = 0; };
struct RankedItem { std::string id; double score = 0.0; };
struct RankedList { std::vector<RankedItem> items; };
int count_local_matches(const std::vector<TernaryCode>& a, const std::vector<TernaryCode>& b, double ratio = 0.85);
MatchResult match_pair(const EncodedImage& a, const EncodedImage& b, const MatchOptions& opts = {});
RankedList retrieve(const EncodedImage& query, const std::vector<std::pair<std::string, const EncodedImage*>>& index,
                    const MatchOptions& opts = {});

struct TrainOptions { uint64_t seed = 7; int gmm_components = 8; int em_iterations = 25;
                      int select_n = 300; int max_side = 640; int relevance_bins = 16; };
ModelBundle train_model(const std::vector<Plane>& corpus, const TrainOptions& o);  // pipeline.cpp:99-166

}  // namespace orc
