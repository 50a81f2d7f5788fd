// Host-side model bundle for the GPU context: parse, validate, canonicalise
// (for model_crc) and flatten into the tables the kernels read.
// Product code — independent of oracle/ (which the product never links).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace cdvz_gpu {

struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };

uint32_t crc32_bytes(const void* data, std::size_t len);

struct LutTable { std::vector<double> edges, values; };

// Everything in a CDVZ-MODEL 1 bundle (proj/include/cdvz/model_io.hpp:14-26),
// plus the derived detector constants (finalize(), scale_space.cpp:75-83).
struct Bundle {
  int num_octaves = 4;
  std::vector<double> sigmas;
  double response_threshold = 0.02, edge_r = 10.0;
  double beta[4][4] = {};
  int select_n = 300;
  std::array<LutTable, 5> relevance;  // sigma, p, d, rho, pss
  double tr_a[8][8] = {}, tr_b[8][8] = {}, tr_scale = 1.0;
  double t0[128] = {}, t1[128] = {};
  int priority[128] = {};
  uint8_t degenerate[128] = {};
  double pca_mean[128] = {};
  std::vector<double> pca_basis;            // 32 x 128
  int nc = 0;
  std::vector<double> weights, means, stds;  // nc, nc x 32, nc x 32
  uint32_t model_crc = 0;

  // Derived, computed on the host exactly as the reference does.
  std::vector<double> taps[4];  // gaussian_kernel (image.cpp:163-175)
  int radius[4] = {};
  int margin = 0;               // ceil(3 sigma_3) + 2 (scale_space.cpp:45-47)
  double rho_limit = 0.0;       // (r+1)^2 / r
};

Bundle parse_bundle(const std::string& text);       // model_io.cpp:141-273 + validate
std::string serialize_bundle(const Bundle& b);      // model_io.cpp:86-139 (canonical text)

// gaussian_kernel (image.cpp:163-175) and Eigen's SSE2 packet-order sum of a
// contiguous vector.
std::vector<double> gaussian_kernel_taps(double sigma);
double eigen_packet_sum(const double* v, std::size_t n);

struct Mode { int id; const char* name; std::size_t budget; int elements; double fraction; bool variance; };
const Mode& mode_by_id(int id);                     // transform_coding.cpp:21-37

// Budget split of encode_image (pipeline.cpp:62-70).
struct Budget { int k = 0; std::size_t global_bytes = 0, code_bytes = 0, max_codes = 0; };
Budget budget_for(const Mode& m, int nc);

}  // namespace cdvz_gpu
