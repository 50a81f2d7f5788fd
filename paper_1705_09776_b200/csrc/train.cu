// GPU kernels of train_model (proj/src/pipeline.cpp:99-166): the synthetic
// partner images of the relevance labelling (apply_transform,
// proj/src/synthetic.cpp:63-90), the PCA covariance and projection
// (train_pca / pca_reduce, proj/src/scfv.cpp:82-85,328-352), the EM
// iterations of train_gmm (proj/src/scfv.cpp:354-430) and the descriptor
// transform feeding train_thresholds (transform_descriptor,
// proj/src/transform_coding.cpp:81-91). Pass 1 itself (detection, selection,
// description) is the extractor's own pipeline (context.cu). The sequential
// pieces — k-means++ seeding, the 128 x 128 eigensolver, quantile sorting,
// the relevance histograms — run on the host (train_host.cpp).
//
// Arithmetic follows the reference's order with separately rounded FP64
// operations (--fmad=false): sums over samples ascend, vector reductions use
// the Eigen packet order (packet_sum_seq).
#include "common.cuh"
#include "dmath.cuh"

namespace cdvz_gpu {

namespace {

// Eigen SSE2 redux order over a contiguous vector (the oracle's eigen_sum);
// strided form for columns of a row-major array.
__device__ double packet_sum_strided(const double* v, long long n, long long stride) {
  auto at = [&](long long i) { return v[i * stride]; };
  if (n < 2) return n ? at(0) : 0.0;
  if (n < 4) {
    double r = at(0) + at(1);
    for (long long i = 2; i < n; ++i) r += at(i);
    return r;
  }
  const long long e2 = n / 4 * 4, e1 = n / 2 * 2;
  double a0 = at(0), a1 = at(1), b0 = at(2), b1 = at(3);
  for (long long i = 4; i < e2; i += 4) {
    a0 += at(i);
    a1 += at(i + 1);
    b0 += at(i + 2);
    b1 += at(i + 3);
  }
  a0 += b0;
  a1 += b1;
  if (e1 > e2) {
    a0 += at(e2);
    a1 += at(e2 + 1);
  }
  double r = a0 + a1;
  for (long long i = e1; i < n; ++i) r += at(i);
  return r;
}

// rotate90 (synthetic.cpp:63-76) by k clockwise quarter turns, composed:
// k = 1: out[r][c] = in[h-1-c][r]; 2: in[h-1-r][w-1-c]; 3: in[c][w-1-r].
__global__ void k_rotate90(const double* in, int w, int h, int k, double* out, int ow, int oh) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
  if (c >= ow || r >= oh) return;
  double v;
  if (k == 1) v = in[(long long)(h - 1 - c) * w + r];
  else if (k == 2) v = in[(long long)(h - 1 - r) * w + (w - 1 - c)];
  else if (k == 3) v = in[(long long)c * w + (w - 1 - r)];
  else v = in[(long long)r * w + c];
  out[(long long)r * ow + c] = v;
}

// gaussian_blur (image.cpp:177-212): x pass into tmp, then y pass, taps
// j = -r..r summed from 0.0 in order, mirror-reflected borders; then
// apply_transform's clamp to [0, 1] (synthetic.cpp:87).
__global__ void k_blur_x(const double* in, int w, int h, const double* taps, int r, double* tmp) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w || y >= h) return;
  double acc = 0.0;
  for (int j = -r; j <= r; ++j) acc += taps[j + r] * in[(long long)y * w + mirror_index(x + j, w)];
  tmp[(long long)y * w + x] = acc;
}
__global__ void k_blur_y_clamp(const double* tmp, int w, int h, const double* taps, int r, double* out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w || y >= h) return;
  double acc = 0.0;
  for (int j = -r; j <= r; ++j) acc += taps[j + r] * tmp[(long long)mirror_index(y + j, h) * w + x];
  out[(long long)y * w + x] = fmax(fmin(acc, 1.0), 0.0);  // .min(1.0).max(0.0)
}

// train_pca: cov = centred^T centred / n with the sample index ascending
// (scfv.cpp:335-336); thread per (a, b).
__global__ void k_covariance(const double* cen, long long n, double* cov) {
  const int a = blockIdx.y, b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= 128) return;
  double s = cen[a] * cen[b];
  for (long long t = 1; t < n; ++t) s = s + cen[t * 128 + a] * cen[t * 128 + b];
  cov[a * 128 + b] = s / static_cast<double>(n);
}

// pca_reduce (scfv.cpp:82-85): (raw - mean) basis^T, inner index ascending.
__global__ void k_pca_rows(const double* raw, long long n, const double* mean, const double* basis, double* x) {
  const long long t = blockIdx.x;
  const int r = threadIdx.x;  // 32
  if (t >= n) return;
  const double* row = raw + t * 128;
  double s = (row[0] - mean[0]) * basis[r * 128];
  for (int j = 1; j < 128; ++j) s = s + (row[j] - mean[j]) * basis[r * 128 + j];
  x[t * 32 + r] = s;
}

// E step of train_gmm: log_weighted_densities (scfv.cpp:20-37) — for row t
// and component i, maha = sum_j ((x - mu) / sigma)^2 in j order, then
// log w - 0.5 maha - log_norm - 16 log(2 pi); log w and log_norm come from the
// host (glibc log, as the reference).
__global__ void k_em_logp(const double* x, long long n, int nc, const double* means, const double* stds,
                          const double* log_w, const double* log_norm, double* logp) {
  const long long t = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc || t >= n) return;
  const double* xr = x + t * 32;
  double maha = 0.0;
  for (int j = 0; j < 32; ++j) {
    const double z = (xr[j] - means[i * 32 + j]) / stds[i * 32 + j];
    maha += z * z;
  }
  constexpr double kLog2Pi = 1.8378770664093453;  // scfv.cpp:16
  logp[t * nc + i] = log_w[i] - 0.5 * maha - log_norm[i] - 16.0 * kLog2Pi;
}

// softmax_rows (scfv.cpp:40-48) in place: peak, e = exp(logp - peak), the
// packet-order sum, gamma = e / sum. Thread per row.
__global__ void k_em_softmax(double* logp, long long n, int nc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double* row = logp + t * nc;
  double peak = row[0];
  for (int i = 1; i < nc; ++i) peak = fmax(peak, row[i]);
  for (int i = 0; i < nc; ++i) row[i] = dm::exp(row[i] - peak);
  const double sum = packet_sum_strided(row, nc, 1);
  for (int i = 0; i < nc; ++i) row[i] = row[i] / sum;
}

// M step (scfv.cpp:412-423): nk = column sums of gamma (packet order); mu and
// E[x^2] = gamma_i^T x / nk and gamma_i^T x^2 / nk with the sample index
// ascending. Block per component, thread per dimension (32) + nk.
__global__ void k_em_mstep(const double* gamma, const double* x, long long n, int nc, double* nk, double* mu,
                           double* ex2) {
  const int i = blockIdx.x, j = threadIdx.x;
  __shared__ double s_nk;
  if (j == 0) s_nk = packet_sum_strided(gamma + i, n, nc);
  __syncthreads();
  const double nki = s_nk;
  if (j == 0) nk[i] = nki;
  double m = gamma[i] * x[j], e = gamma[i] * (x[j] * x[j]);
  for (long long t = 1; t < n; ++t) {
    const double g = gamma[t * nc + i], v = x[t * 32 + j];
    m = m + g * v;
    e = e + g * (v * v);
  }
  mu[i * 32 + j] = m / nki;
  ex2[i * 32 + j] = e / nki;
}

// transform_descriptor (transform_coding.cpp:81-91) of every corpus row:
// scale * (M_cell raw_cell), inner index ascending. Thread per (row, cell).
__global__ void k_transform_rows(const double* raw, long long n, const double* ta, const double* tb, double scale,
                                 double* out) {
  const long long t = blockIdx.x;
  const int cell = threadIdx.x;  // 16
  if (t >= n) return;
  const int cx = cell % 4, cy = cell / 4;
  const double* m = ((cx + cy) % 2 == 0) ? ta : tb;  // cell_uses_a: (cx + cy) even
  const double* v = raw + t * 128 + cell * 8;
  for (int r = 0; r < 8; ++r) {
    double s = m[r * 8] * v[0];
    for (int k = 1; k < 8; ++k) s = s + m[r * 8 + k] * v[k];
    out[t * 128 + cell * 8 + r] = scale * s;
  }
}

}  // namespace

cudaError_t launch_rotate90(const double* in, int w, int h, int k, double* out, cudaStream_t st) {
  const int ow = (k % 2) ? h : w, oh = (k % 2) ? w : h;
  k_rotate90<<<dim3((ow + 127) / 128, oh), 128, 0, st>>>(in, w, h, k % 4, out, ow, oh);
  return cudaGetLastError();
}

cudaError_t launch_blur_clamp(const double* in, int w, int h, const double* d_taps, int r, double* tmp, double* out,
                              cudaStream_t st) {
  const dim3 grid((w + 127) / 128, h);
  k_blur_x<<<grid, 128, 0, st>>>(in, w, h, d_taps, r, tmp);
  k_blur_y_clamp<<<grid, 128, 0, st>>>(tmp, w, h, d_taps, r, out);
  return cudaGetLastError();
}

cudaError_t launch_covariance(const double* centred, long long n, double* cov, cudaStream_t st) {
  k_covariance<<<dim3(1, 128), 128, 0, st>>>(centred, n, cov);
  return cudaGetLastError();
}

cudaError_t launch_pca_rows(const double* raw, long long n, const double* mean, const double* basis, double* x,
                            cudaStream_t st) {
  k_pca_rows<<<unsigned(n), 32, 0, st>>>(raw, n, mean, basis, x);
  return cudaGetLastError();
}

cudaError_t launch_em_step(const double* x, long long n, int nc, const double* means, const double* stds,
                           const double* log_w, const double* log_norm, double* gamma, double* nk, double* mu,
                           double* ex2, cudaStream_t st) {
  k_em_logp<<<dim3((nc + 127) / 128, unsigned(n)), 128, 0, st>>>(x, n, nc, means, stds, log_w, log_norm, gamma);
  k_em_softmax<<<unsigned((n + 127) / 128), 128, 0, st>>>(gamma, n, nc);
  k_em_mstep<<<nc, 32, 0, st>>>(gamma, x, n, nc, nk, mu, ex2);
  return cudaGetLastError();
}

cudaError_t launch_transform_rows(const double* raw, long long n, const double* ta, const double* tb, double scale,
                                  double* out, cudaStream_t st) {
  k_transform_rows<<<unsigned(n), 16, 0, st>>>(raw, n, ta, tb, scale, out);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
