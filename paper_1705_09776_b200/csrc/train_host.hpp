// Host-side pieces of the GPU trainer (cdvz_gpu_train_model, context.cu): the
// sequential steps of train_model (proj/src/pipeline.cpp:99-166) that are
// either inherently ordered (k-means++ seeding, quantile sorting) or tiny (the
// 128 x 128 eigenproblem, the relevance histograms, point mapping).
// Product code, independent of oracle/.
#pragma once

#include <array>
#include <cstdint>
#include <random>
#include <vector>

#include "bundle.hpp"

namespace cdvz_gpu {

// InterestPoint fields the relevance model reads (FeatureStats,
// proj/include/cdvz/relevance.hpp:13-27) plus the position.
struct TrainPoint {
  double x, y, sigma, p, d, rho, pss;
};

// SynthTransform of train_model's partner image i (pipeline.cpp:125-129).
struct SynthTransform {
  int quarter_turns;
  double scale, blur_sigma;
};
SynthTransform partner_transform(std::size_t i);
// Output size of apply_transform (synthetic.cpp:78-90).
void transform_size(const SynthTransform& t, int w, int h, int& ow, int& oh);
// map_point (synthetic.cpp:92-111).
void map_point(const SynthTransform& t, int src_w, int src_h, double& x, double& y, double& sigma);

// label_matches_by_geometry (relevance.cpp:147-170), appended to `out`.
void label_matches(const std::vector<TrainPoint>& a, const std::vector<TrainPoint>& b,
                   const std::vector<std::array<double, 3>>& mapped, double xy_tol, double ratio_tol,
                   std::vector<std::pair<TrainPoint, bool>>& out);

// train_relevance_tables (relevance.cpp:95-145).
std::array<LutTable, 5> train_relevance(const std::vector<std::pair<TrainPoint, bool>>& samples, int bins,
                                        int min_bin_samples);

// Symmetric eigendecomposition of a 128 x 128 row-major matrix (cyclic Jacobi):
// eigenvalues ascending, eigenvectors as the columns of `vecs` (row-major).
void sym_eigen128(const std::vector<double>& a, std::vector<double>& vals, std::vector<double>& vecs);

// k-means++ seeding of train_gmm (scfv.cpp:368-393): centre row indices.
std::vector<long long> kmeanspp(const std::vector<double>& x, long long n, int nc, std::mt19937_64& rng);

// train_thresholds (transform_coding.cpp:126-172) into b.t0 / t1 / priority / degenerate.
void train_thresholds(const std::vector<double>& transformed, long long n, double p0, Bundle& b);

}  // namespace cdvz_gpu
