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

__device__ __forceinline__ double wrap_angle(double a) {
  a = fmod(a, kTwoPi);
  return a < 0.0 ? a + kTwoPi : a;
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

// One CTA per oriented point, grid-strided: description
// (descriptor.cpp:47-145) + compression (transform_coding.cpp:81-217).
//
// Phase A: all samples of the patch are evaluated in parallel (bilinear
// gradients, magnitude, Gaussian weight, orientation) and parked in shared
// memory. Phase B: thread (sub-patch s, cell c, parity p) owns the 4
// orientation bins of cell c with parity p for sub-patch s. A sample's cell
// coordinates depend only on its index (cu0 = floor(u(i) / 3sigma + 1.5),
// cv0 likewise in j), so the samples feeding cell c form a rectangle in index
// space; the thread walks it in row-major order, which is exactly the order
// the reference adds them, and each sample adds to exactly one of its bins.
constexpr int kMaxSamples = 32;  // samples per axis: ceil(12 sigma) for sigma <= 2.66 (radius-8 detector)

__global__ void __launch_bounds__(128, 5) k_describe(Batch bt, DetConst dc, Model md, EncodeConst ec) {
  __shared__ double s_w[kMaxSamples * kMaxSamples];       // weight; +0 for a skipped sample
  __shared__ double s_wo[2][kMaxSamples * kMaxSamples];   // wo for the bin of parity 0 / 1
  __shared__ uint8_t s_slot[kMaxSamples * kMaxSamples];   // bin >> 1 for parity 0 (bits 0-1) / 1 (bits 2-3)
  __shared__ double s_wu[2][kMaxSamples], s_wv[2][kMaxSamples];  // [du][i]: 1 - fu, fu
  __shared__ int s_cu[kMaxSamples], s_cv[kMaxSamples];
  __shared__ double part[4][128];  // <= 2x2 sub-patches of 16x16 samples
  __shared__ double sq[128], red[4], tv[128], vec[128];
  __shared__ uint8_t sym[128];
  const int tid = threadIdx.x;
  const int f = blockIdx.y;
  const int n_or = bt.or_count[f];
  for (int idx = blockIdx.x; idx < n_or; idx += gridDim.x) {
    const Oriented orp = bt.oriented[(long long)f * bt.cap_or + idx];
    const KP k = bt.sel[(long long)f * bt.select_n + orp.sel];
    const double theta = orp.theta;
    const Frame fr = resolve(bt, dc, f, k);
    // make_geometry (descriptor.cpp:47-58)
    const double half = 6.0 * fr.sigma;
    const int samples = max(1, static_cast<int>(ceil(12.0 * fr.sigma)));
    const double step = 2.0 * half / samples;
    const int spa = (samples + 15) / 16;
    const double cos_t = cos(theta), sin_t = sin(theta);
    const double inv_cell = 1.0 / (3.0 * fr.sigma);
    const double gauss_denom = 2.0 * half * half;
    const int n_sub = spa * spa;
    if (samples > kMaxSamples) {  // outside the supported scale range: flag the frame
      if (tid == 0) atomicOr(&bt.status[f], 8);
      continue;
    }
    // Per-axis cell coordinates (descriptor.cpp:89-96): cu depends on i only.
    for (int i = tid; i < samples; i += blockDim.x) {
      const double u = (i + 0.5) * step - half;
      const double cu = u * inv_cell + 1.5;
      const int cu0 = static_cast<int>(floor(cu));
      const double fu = cu - cu0;
      s_cu[i] = cu0;
      s_wu[0][i] = 1.0 - fu;
      s_wu[1][i] = fu;
    }
    for (int j = tid; j < samples; j += blockDim.x) {
      const double v = (j + 0.5) * step - half;
      const double cv = v * inv_cell + 1.5;
      const int cv0 = static_cast<int>(floor(cv));
      const double fv = cv - cv0;
      s_cv[j] = cv0;
      s_wv[0][j] = 1.0 - fv;
      s_wv[1][j] = fv;
    }
    // Phase A: every sample (descriptor.cpp:75-88).
    const int ns = samples * samples;
    for (int q = tid; q < ns; q += blockDim.x) {
      const int j = q / samples, i = q - j * samples;
      const double v = (j + 0.5) * step - half;
      const double u = (i + 0.5) * step - half;
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
      // Of the sample's two orientation bins (bin0, bin0 + 1 mod 8), the one
      // of parity p gets wo = 1 - fo if it is bin0, fo otherwise.
      const int odd = bin0 & 1;
      const int b_even = odd ? (bin0 + 1) & 7 : bin0, b_odd = odd ? bin0 : (bin0 + 1) & 7;
      s_w[q] = wgt;
      s_wo[0][q] = odd ? fo : 1.0 - fo;
      s_wo[1][q] = odd ? 1.0 - fo : fo;
      s_slot[q] = uint8_t((b_even >> 1) | ((b_odd >> 1) << 2));
    }
    __syncthreads();
    // Phase B: ordered accumulation (descriptor.cpp:98-116).
    {
      const int sp = tid >> 5, cell = (tid >> 1) & 15, parity = tid & 1;
      const int cx = cell & 3, cy = cell >> 2;
      double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
      if (sp < n_sub) {
        const int i_lo = (sp % spa) * 16, j_lo = (sp / spa) * 16;
        const int i_hi = min(samples, i_lo + 16), j_hi = min(samples, j_lo + 16);
        // Samples with cu0 in {cx-1, cx} (du = 1, 0) and cv0 in {cy-1, cy}.
        int ia = i_lo, ib = i_hi, ja = j_lo, jb = j_hi;
        while (ia < ib && s_cu[ia] < cx - 1) ++ia;
        while (ib > ia && s_cu[ib - 1] > cx) --ib;
        while (ja < jb && s_cv[ja] < cy - 1) ++ja;
        while (jb > ja && s_cv[jb - 1] > cy) --jb;
        const double* wo_p = s_wo[parity];
        const int shift = 2 * parity;
        for (int j = ja; j < jb; ++j) {
          const double wv = s_wv[cy - s_cv[j]][j];
          const int row = j * samples;
#pragma unroll 4
          for (int i = ia; i < ib; ++i) {
            const int q = row + i;
            // A skipped sample has weight +0: the add leaves the (non-negative) sum unchanged.
            const double add = s_w[q] * wv * s_wu[cx - s_cu[i]][i] * wo_p[q];
            const int slot = (s_slot[q] >> shift) & 3;
            acc0 += slot == 0 ? add : 0.0;
            acc1 += slot == 1 ? add : 0.0;
            acc2 += slot == 2 ? add : 0.0;
            acc3 += slot == 3 ? add : 0.0;
          }
        }
        part[sp][cell * 8 + parity] = acc0;
        part[sp][cell * 8 + parity + 2] = acc1;
        part[sp][cell * 8 + parity + 4] = acc2;
        part[sp][cell * 8 + parity + 6] = acc3;
      }
    }
    __syncthreads();
    // merge_and_normalize (descriptor.cpp:124-145): sum partials in order,
    // then up to 5 rounds of L2 normalise + clamp at 0.2; the norm uses the
    // Eigen SSE2 reduction order.
    double v = part[0][tid];
    for (int s = 1; s < n_sub; ++s) v = v + part[s][tid];
    for (int round = 0; round < 5; ++round) {
      sq[tid] = v * v;
      __syncthreads();
      if (tid < 4) {
        double a = sq[tid];
        for (int i = tid + 4; i < 128; i += 4) a = a + sq[i];
        red[tid] = a;
      }
      __syncthreads();
      const double norm = sqrt((red[0] + red[2]) + (red[1] + red[3]));
      if (norm == 0.0) break;
      v = v / norm;
      bool clipped = false;
      if (v > 0.2) { v = 0.2; clipped = true; }
      if (!__syncthreads_or(clipped)) break;
    }
    bt.desc[((long long)f * bt.cap_or + idx) * 128 + tid] = v;
    vec[tid] = v;
    __syncthreads();
    // transform_descriptor (transform_coding.cpp:81-91)
    {
      const int c = tid >> 3, i = tid & 7;
      const int which = (((c % 4) + (c / 4)) & 1) == 0 ? 0 : 1;
      double s = md.tr[which][i][0] * vec[c * 8];
#pragma unroll
      for (int kk = 1; kk < 8; ++kk) s = s + md.tr[which][i][kk] * vec[c * 8 + kk];
      tv[tid] = md.tr_scale * s;
    }
    __syncthreads();
    // quantize_ternary (transform_coding.cpp:202-217): 00 zero, 01 +1, 10 -1
    if (tid < ec.elements) {
      const int e = md.priority[tid];
      const double val = tv[e];
      sym[tid] = val < md.t0[e] ? 2 : (val > md.t1[e] ? 1 : 0);
    }
    __syncthreads();
    uint8_t* code = bt.codes + ((long long)f * bt.cap_or + idx) * bt.code_stride;
    const int nbytes = (ec.elements * 2 + 7) / 8;
    if (tid < nbytes) {
      uint8_t byte = 0;
      for (int q = 0; q < 4; ++q) {
        const int j = tid * 4 + q;
        if (j < ec.elements) byte |= uint8_t(sym[j] << (2 * q));
      }
      code[6 + tid] = byte;
    }
    if (tid == 0) {
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
    __syncthreads();
  }
}

cudaError_t launch_describe(const Batch& bt, const DetConst& dc, const Model& md, const EncodeConst& ec, cudaStream_t st) {
  k_orient<<<dim3((bt.select_n + 3) / 4, bt.nframes), 128, 0, st>>>(bt, dc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_expand<<<bt.nframes, 1024, 0, st>>>(bt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_describe<<<dim3(96, bt.nframes), 128, 0, st>>>(bt, dc, md, ec);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
