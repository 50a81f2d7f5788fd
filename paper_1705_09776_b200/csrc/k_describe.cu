// K5 — dominant orientations, K5b — orientation expansion, K6/K7 — SIFT-style
// description fused with transform coding (Hadamard pair, ternary band
// quantiser, coordinate/scale/angle quantisers).
//
// Replaces resolve_frame / dominant_orientations / assign_orientations /
// subpatch_partial / normalize_descriptor / describe_batch
// (proj/src/descriptor.cpp:25-304) and transform_descriptor / quantize_* /
// compress_descriptors (proj/src/transform_coding.cpp:81-217,
// proj/src/pipeline.cpp:37-50).
//
// Determinism: the reference accumulates every histogram bin in sample order
// (raster order for orientations, row-major per 16x16 sub-patch for
// descriptors) and merges sub-patches in index order. The kernels keep that
// order exactly without atomics: a warp evaluates 32 consecutive samples in
// parallel, parks their contributions in shared memory, and each lane then
// owns a fixed set of bins and adds the parked contributions in sample order.
// For descriptors the ownership is (cell, orientation parity), so each sample
// adds at most one term per lane.
#include "common.cuh"

namespace cdvz_gpu {

namespace {

constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
constexpr int kMaxPeaks = 36;

// wrap_angle (descriptor.cpp:19-22) for |a| < 2 * 2pi without the general
// fmod loop: fmod is exact, and on this range it is a itself or a +- 2pi,
// which Sterbenz's lemma makes exact too (sign of the dividend kept).
__device__ __forceinline__ double wrap_angle(double a) {
  double r = a;
  if (fabs(a) >= kTwoPi) {
    if (fabs(a) < 2.0 * kTwoPi) {
      r = a > 0.0 ? a - kTwoPi : a + kTwoPi;
      if (r == 0.0) r = copysign(0.0, a);
    } else {
      r = fmod(a, kTwoPi);
    }
  }
  return r < 0.0 ? r + kTwoPi : r;
}

// descriptor.cpp:25-35 — a term is skipped when its fraction is exactly 0.
__device__ __forceinline__ double sample_bilinear(const double* img, int w, double qx, double qy) {
  const int x0 = static_cast<int>(floor(qx));
  const int y0 = static_cast<int>(floor(qy));
  const double fx = qx - x0, fy = qy - y0;
  const double* p = img + (long long)y0 * w + x0;
  double v = (1.0 - fy) * (1.0 - fx) * p[0];
  if (fx > 0.0) v += (1.0 - fy) * fx * p[1];
  if (fy > 0.0) v += fy * (1.0 - fx) * p[w];
  if (fx > 0.0 && fy > 0.0) v += fy * fx * p[w + 1];
  return v;
}

struct Frame { const double* lvl; int w, h; double x, y, sigma; };

// resolve_frame (descriptor.cpp:149-170): nearest scale node, first minimum.
__device__ __forceinline__ Frame resolve(const Batch& bt, const DetConst& dc, int f, const KP& k) {
  Frame fr;
  const int o = k.octave;
  const double inv = ldexp(1.0, -o);
  fr.x = k.x * inv;
  fr.y = k.y * inv;
  fr.sigma = k.sigma * inv;
  int best = 0;
  double best_gap = fabs(dc.sigmas[0] - fr.sigma);
  for (int i = 1; i < 4; ++i) {
    const double gap = fabs(dc.sigmas[i] - fr.sigma);
    if (gap < best_gap) { best_gap = gap; best = i; }
  }
  fr.lvl = bt.pyr + f * bt.frame_doubles + bt.plane_off[o][best];
  fr.w = bt.ow[o];
  fr.h = bt.oh[o];
  return fr;
}

}  // namespace

// One warp per selected point (descriptor.cpp:172-232).
__global__ void __launch_bounds__(128) k_orient(Batch bt, DetConst dc) {
  __shared__ double sval[4][32];
  __shared__ int sbin[4][32];
  __shared__ double hist[4][36];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.y;
  const int r = blockIdx.x * 4 + wi;
  if (r >= bt.sel_count[f]) return;  // warp-uniform; no block barrier below
  const KP k = bt.sel[(long long)f * bt.select_n + r];
  const Frame fr = resolve(bt, dc, f, k);
  const double radius = 3.96 * fr.sigma;
  const double window = 1.5 * fr.sigma;
  const double denom = 2.0 * window * window;
  const int x_lo = max(1, static_cast<int>(ceil(fr.x - radius)));
  const int x_hi = min(fr.w - 2, static_cast<int>(floor(fr.x + radius)));
  const int y_lo = max(1, static_cast<int>(ceil(fr.y - radius)));
  const int y_hi = min(fr.h - 2, static_cast<int>(floor(fr.y + radius)));
  const int nx = x_hi - x_lo + 1, ny = y_hi - y_lo + 1;
  const int npx = (nx > 0 && ny > 0) ? nx * ny : 0;
  double acc0 = 0.0, acc1 = 0.0;  // bins lane and lane + 32
  for (int base = 0; base < npx; base += 32) {
    const int q = base + lane;
    int bin = -1;
    double val = 0.0;
    if (q < npx) {
      const int ix = x_lo + q % nx, iy = y_lo + q / nx;
      const double dx = ix - fr.x, dy = iy - fr.y;
      const double d2 = dx * dx + dy * dy;
      if (!(d2 >= radius * radius)) {
        const double* row = fr.lvl + (long long)iy * fr.w + ix;
        const double gx = 0.5 * (row[1] - row[-1]);
        const double gy = 0.5 * (row[fr.w] - row[-fr.w]);
        const double mag = hypot(gx, gy);
        if (mag != 0.0) {
          const double ang = wrap_angle(atan2(gy, gx));
          bin = static_cast<int>(floor(ang / kTwoPi * 36 + 0.5)) % 36;
          val = mag * exp(-d2 / denom);
        }
      }
    }
    sbin[wi][lane] = bin;
    sval[wi][lane] = val;
    __syncwarp();
    const int nsmp = min(32, npx - base);
    for (int s = 0; s < nsmp; ++s) {
      const int b = sbin[wi][s];
      if (b == lane) acc0 += sval[wi][s];
      else if (b == lane + 32) acc1 += sval[wi][s];
    }
    __syncwarp();
  }
  hist[wi][lane] = acc0;
  if (lane < 4) hist[wi][lane + 32] = acc1;
  __syncwarp();
  for (int pass = 0; pass < 2; ++pass) {
    double s0 = (hist[wi][(lane + 35) % 36] + hist[wi][lane] + hist[wi][(lane + 1) % 36]) / 3.0, s1 = 0.0;
    if (lane < 4) s1 = (hist[wi][(lane + 32 + 35) % 36] + hist[wi][lane + 32] + hist[wi][(lane + 33) % 36]) / 3.0;
    __syncwarp();
    hist[wi][lane] = s0;
    if (lane < 4) hist[wi][lane + 32] = s1;
    __syncwarp();
  }
  double peak = fmax(hist[wi][lane], lane < 4 ? hist[wi][lane + 32] : 0.0);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, d));
  peak = fmax(peak, 0.0);
  double* out = bt.thetas + ((long long)f * bt.select_n + r) * kMaxPeaks;
  int* cnt = bt.theta_count + (long long)f * bt.select_n + r;
  if (peak == 0.0) {
    if (lane == 0) { out[0] = 0.0; *cnt = 1; }
    return;
  }
  const double bin_width = kTwoPi / 36;
  int total = 0;
  for (int half = 0; half < 2; ++half) {
    const int b = lane + 32 * half;
    bool is_peak = false;
    double theta = 0.0;
    if (b < 36) {
      const double v = hist[wi][b], l = hist[wi][(b + 35) % 36], rr = hist[wi][(b + 1) % 36];
      if (!(v <= 0.8 * peak || v < l || v < rr)) {
        const double fit = l - 2.0 * v + rr;
        const double delta = fabs(fit) > 1e-12 ? 0.5 * (l - rr) / fit : 0.0;
        theta = wrap_angle((b + delta) * bin_width);
        is_peak = true;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, is_peak);
    if (is_peak) out[total + __popc(bal & ((1u << lane) - 1u))] = theta;
    total += __popc(bal);
  }
  if (lane == 0) {
    if (total == 0) { out[0] = 0.0; total = 1; }
    *cnt = total;
  }
}

// Expands per-point peaks into the oriented list in (point, peak) order
// (descriptor.cpp:252-255). One CTA per frame.
__global__ void __launch_bounds__(1024) k_expand(Batch bt) {
  __shared__ int wsum[33];
  const int f = blockIdx.x;
  const int n = bt.sel_count[f];
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, int(threadIdx.x) * per), hi = min(n, lo + per);
  const int* cnt = bt.theta_count + (long long)f * bt.select_n;
  int c = 0;
  for (int i = lo; i < hi; ++i) c += cnt[i];
  // block exclusive scan
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = c;
  for (int d = 1; d < 32; d <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += x;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int x = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0, xi = x;
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += y;
    }
    wsum[lane] = xi - x;
    if (lane == 31) wsum[32] = xi;
  }
  __syncthreads();
  int pos = wsum[wid] + incl - c;
  const int total = wsum[32];
  Oriented* dst = bt.oriented + (long long)f * bt.cap_or;
  const double* th = bt.thetas + (long long)f * bt.select_n * kMaxPeaks;
  for (int i = lo; i < hi; ++i)
    for (int j = 0; j < cnt[i]; ++j, ++pos)
      if (pos < bt.cap_or) {
        Oriented o;
        o.sel = i;
        o.pad = 0;
        o.theta = th[i * kMaxPeaks + j];
        dst[pos] = o;
      }
  if (threadIdx.x == 0) {
    bt.or_count[f] = total < bt.cap_or ? total : bt.cap_or;
    if (total > bt.cap_or) atomicOr(&bt.status[f], 4);
  }
}

// One WARP per oriented point: description (descriptor.cpp:47-145) +
// compression (transform_coding.cpp:81-217), warp-synchronous (no block
// barriers; the CTA is only a container of independent warps).
//
// The 12-sigma patch is sampled on a samples x samples grid (samples =
// ceil(12 sigma) <= 32) and split into row bands of 16 sample rows — exactly
// the rows of the reference's 16x16 sub-patches. Per band:
//   Phase A: the warp evaluates every sample of the band (bilinear gradient,
//     magnitude, Gaussian weight, orientation bin) with 32 samples in flight
//     and parks (weight, fo, bin0) in shared memory;
//   Phase B: lane (cell c, parity p) owns the four orientation bins of parity
//     p of cell c. Cell coordinates depend on the sample index only, so the
//     samples feeding cell c form a rectangle; the lane walks it in row-major
//     order — the reference's add order — keeping separate partials for the
//     left and right sub-patch of the band, and folds the band's partials into
//     the running total in sub-patch index order (merge_and_normalize).
// Every lane then holds 4 of the 128 bins for normalisation, transform and
// ternary coding.
constexpr int kMaxSamples = 32;  // samples per axis: ceil(12 sigma) for sigma <= 2.66 (radius-8 detector)
constexpr int kBand = 16;        // kSubPatchSide (descriptor.cpp)
constexpr int kDescWarps = 4;

struct DescWarpSmem {
  double w[kBand * kMaxSamples];   // weight; +0 for a skipped sample. Reused as sq / tv after phase B.
  double fo[kBand * kMaxSamples];  // fractional orientation bin
  double u[kMaxSamples];           // (i + 0.5) * step - half (same for rows and columns)
  double wf[2][kMaxSamples];       // [d][i]: 1 - f, f of the cell coordinate
  uint8_t bin[kBand * kMaxSamples];
  int c0[kMaxSamples];             // floor(u * inv_cell + 1.5)
};

__global__ void __launch_bounds__(32 * kDescWarps, 4) k_describe(Batch bt, DetConst dc, Model md, EncodeConst ec) {
  __shared__ DescWarpSmem smem[kDescWarps];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DescWarpSmem& S = smem[wi];
  const int f = blockIdx.y;
  const int n_or = bt.or_count[f];
  const int cell = lane >> 1, parity = lane & 1;
  const int ccx = cell & 3, ccy = cell >> 2;
  for (int idx = blockIdx.x * kDescWarps + wi; idx < n_or; idx += gridDim.x * kDescWarps) {
    const Oriented orp = bt.oriented[(long long)f * bt.cap_or + idx];
    const KP k = bt.sel[(long long)f * bt.select_n + orp.sel];
    const double theta = orp.theta;
    const Frame fr = resolve(bt, dc, f, k);
    // make_geometry (descriptor.cpp:47-58)
    const double half = 6.0 * fr.sigma;
    const int samples = max(1, static_cast<int>(ceil(12.0 * fr.sigma)));
    if (samples > kMaxSamples) {  // outside the supported scale range: flag the frame
      if (lane == 0) atomicOr(&bt.status[f], 8);
      continue;
    }
    const double step = 2.0 * half / samples;
    const int spa = (samples + kBand - 1) / kBand;
    const double cos_t = cos(theta), sin_t = sin(theta);
    const double inv_cell = 1.0 / (3.0 * fr.sigma);
    const double gauss_denom = 2.0 * half * half;
    // Per-axis cell coordinates (descriptor.cpp:89-96): identical for u (i) and v (j).
    int my_c0 = 0x7fff;
    if (lane < samples) {
      const double u = (lane + 0.5) * step - half;
      const double cu = u * inv_cell + 1.5;
      my_c0 = static_cast<int>(floor(cu));
      const double fu = cu - my_c0;
      S.u[lane] = u;
      S.c0[lane] = my_c0;
      S.wf[0][lane] = 1.0 - fu;
      S.wf[1][lane] = fu;
    }
    // This lane's rectangle: indices whose c0 is in {c - 1, c} (c0 is monotone).
    int ia = samples, ib = samples, ja = samples, jb = samples;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const unsigned ge = __ballot_sync(0xffffffffu, lane < samples && my_c0 >= c - 1);
      const unsigned gt = __ballot_sync(0xffffffffu, lane < samples && my_c0 > c);
      const int lo = ge ? __ffs(ge) - 1 : samples, hi = gt ? __ffs(gt) - 1 : samples;
      if (c == ccx) { ia = lo; ib = hi; }
      if (c == ccy) { ja = lo; jb = hi; }
    }
    __syncwarp();
    double tot[4] = {0.0, 0.0, 0.0, 0.0};
    for (int band = 0; band < spa; ++band) {
      const int j0 = band * kBand, j1 = min(samples, j0 + kBand);
      const int n = (j1 - j0) * samples;
      // Phase A (descriptor.cpp:75-88).
      for (int q = lane; q < n; q += 32) {
        const int jr = q / samples, i = q - jr * samples;
        const double v = S.u[j0 + jr];
        const double u = S.u[i];
        const double px = fr.x + u * cos_t - v * sin_t;
        const double py = fr.y + u * sin_t + v * cos_t;
        int bin0 = 0;
        double wgt = 0.0, fo = 0.0;
        if (!(px < 1.0 || px > fr.w - 2.0 || py < 1.0 || py > fr.h - 2.0)) {
          const double gx = 0.5 * (sample_bilinear(fr.lvl, fr.w, px + 1.0, py) - sample_bilinear(fr.lvl, fr.w, px - 1.0, py));
          const double gy = 0.5 * (sample_bilinear(fr.lvl, fr.w, px, py + 1.0) - sample_bilinear(fr.lvl, fr.w, px, py - 1.0));
          const double mag = hypot(gx, gy);
          if (mag != 0.0) {
            wgt = mag * exp(-(u * u + v * v) / gauss_denom);
            const double phi = wrap_angle(atan2(gy, gx) - theta);
            const double obv = phi / kTwoPi * 8 - 0.5;
            const int ob0 = static_cast<int>(floor(obv));
            fo = obv - ob0;
            bin0 = ((ob0 % 8) + 8) % 8;
          }
        }
        S.w[q] = wgt;
        S.fo[q] = fo;
        S.bin[q] = uint8_t(bin0);
      }
      __syncwarp();
      // Phase B (descriptor.cpp:98-116): partials of the band's left (i < 16)
      // and right sub-patch, each in row-major sample order.
      double pa[4] = {0.0, 0.0, 0.0, 0.0}, pb[4] = {0.0, 0.0, 0.0, 0.0};
      const int jlo = max(ja, j0), jhi = min(jb, j1);
      const int ia0 = ia, ib0 = min(ib, kBand), ia1 = max(ia, kBand), ib1 = ib;
      for (int j = jlo; j < jhi; ++j) {
        const double wv = S.wf[ccy - S.c0[j]][j];
        const int row = (j - j0) * samples;
#define CDVZ_VISIT(ACC)                                                   \
  {                                                                       \
    const int q = row + i;                                                \
    const int b0 = S.bin[q];                                              \
    const bool own = (b0 & 1) == parity;                                  \
    const double fo = S.fo[q];                                            \
    const double wo = own ? 1.0 - fo : fo;                                \
    const int slot = (own ? b0 : (b0 + 1) & 7) >> 1;                      \
    const double add = S.w[q] * wv * S.wf[ccx - S.c0[i]][i] * wo;         \
    ACC[0] += slot == 0 ? add : 0.0;                                      \
    ACC[1] += slot == 1 ? add : 0.0;                                      \
    ACC[2] += slot == 2 ? add : 0.0;                                      \
    ACC[3] += slot == 3 ? add : 0.0;                                      \
  }
        for (int i = ia0; i < ib0; ++i) CDVZ_VISIT(pa)
        for (int i = ia1; i < ib1; ++i) CDVZ_VISIT(pb)
#undef CDVZ_VISIT
      }
      // merge_and_normalize's ordered sum of partials (sub-patch index order).
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        tot[m] = band == 0 ? pa[m] : tot[m] + pa[m];
        if (spa > 1) tot[m] = tot[m] + pb[m];
      }
      __syncwarp();
    }
    // normalize_descriptor (descriptor.cpp:124-145): up to 5 rounds of L2
    // normalise + clamp at 0.2; the norm in the Eigen SSE2 reduction order
    // (four stride-4 running sums, then (s0 + s2) + (s1 + s3)).
    double* sq = S.w;
    double* tv = S.w + 128;
    const int bin_base = cell * 8 + parity;
    for (int round = 0; round < 5; ++round) {
#pragma unroll
      for (int m = 0; m < 4; ++m) sq[bin_base + 2 * m] = tot[m] * tot[m];
      __syncwarp();
      double red = 0.0;
      if (lane < 4) {
        double t[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) t[i] = sq[lane + 4 * i];
        red = t[0];
#pragma unroll
        for (int i = 1; i < 32; ++i) red = red + t[i];
      }
      const double r0 = __shfl_sync(0xffffffffu, red, 0), r1 = __shfl_sync(0xffffffffu, red, 1);
      const double r2 = __shfl_sync(0xffffffffu, red, 2), r3 = __shfl_sync(0xffffffffu, red, 3);
      __syncwarp();
      const double norm = sqrt((r0 + r2) + (r1 + r3));
      if (norm == 0.0) break;
      bool clipped = false;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        tot[m] = tot[m] / norm;
        if (tot[m] > 0.2) { tot[m] = 0.2; clipped = true; }
      }
      if (!__any_sync(0xffffffffu, clipped)) break;
    }
    double* dout = bt.desc + ((long long)f * bt.cap_or + idx) * 128;
#pragma unroll
    for (int m = 0; m < 4; ++m) dout[bin_base + 2 * m] = tot[m];
    // transform_descriptor (transform_coding.cpp:81-91): the cell's 8 values
    // are split between this lane and its parity partner.
    {
      double vec[8];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double other = __shfl_xor_sync(0xffffffffu, tot[m], 1);
        vec[2 * m] = parity ? other : tot[m];
        vec[2 * m + 1] = parity ? tot[m] : other;
      }
      const int which = ((ccx + ccy) & 1) == 0 ? 0 : 1;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int i = parity + 2 * m;
        double s = md.tr[which][i][0] * vec[0];
#pragma unroll
        for (int kk = 1; kk < 8; ++kk) s = s + md.tr[which][i][kk] * vec[kk];
        tv[cell * 8 + i] = md.tr_scale * s;
      }
    }
    __syncwarp();
    // quantize_ternary (transform_coding.cpp:202-217): 00 zero, 01 +1, 10 -1;
    // lane L packs symbols 4L .. 4L+3 into code byte L.
    uint8_t* code = bt.codes + ((long long)f * bt.cap_or + idx) * bt.code_stride;
    if (4 * lane < ec.elements) {
      uint8_t byte = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = 4 * lane + q;
        if (t < ec.elements) {
          const int e = md.priority[t];
          const double val = tv[e];
          const uint8_t sym = val < md.t0[e] ? 2 : (val > md.t1[e] ? 1 : 0);
          byte |= uint8_t(sym << (2 * q));
        }
      }
      code[6 + lane] = byte;
    }
    if (lane == 0) {
      // quantize_coord / quantize_sigma_log / quantize_theta (transform_coding.cpp:173-200)
      const double cxq = fmin(fmax(k.x, 0.0), double(bt.W - 1));
      const double cyq = fmin(fmax(k.y, 0.0), double(bt.H - 1));
      const unsigned xq = (unsigned)llround(cxq / (bt.W - 1) * 65535.0);
      const unsigned yq = (unsigned)llround(cyq / (bt.H - 1) * 65535.0);
      const double sc = fmin(fmax(k.sigma, 0.5), 64.0);
      const double tq = log2(sc / 0.5) / ec.log2_range;
      const unsigned sq8 = (unsigned)llround(tq * 255.0);
      double tt = theta / kTwoPi;
      tt -= floor(tt);
      const unsigned th8 = (unsigned)(llround(tt * 256.0) & 0xFF);
      code[0] = uint8_t(xq & 0xFF);
      code[1] = uint8_t(xq >> 8);
      code[2] = uint8_t(yq & 0xFF);
      code[3] = uint8_t(yq >> 8);
      code[4] = uint8_t(sq8);
      code[5] = uint8_t(th8);
    }
    __syncwarp();
  }
}

cudaError_t launch_describe(const Batch& bt, const DetConst& dc, const Model& md, const EncodeConst& ec, cudaStream_t st) {
  k_orient<<<dim3((bt.select_n + 3) / 4, bt.nframes), 128, 0, st>>>(bt, dc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_expand<<<bt.nframes, 1024, 0, st>>>(bt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_describe<<<dim3(32, bt.nframes), 32 * kDescWarps, 0, st>>>(bt, dc, md, ec);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
