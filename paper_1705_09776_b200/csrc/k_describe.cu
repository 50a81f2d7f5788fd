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
#include "dmath.cuh"

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

// sample_bilinear split in two so that a caller can issue the loads of
// several taps before any arithmetic: the tap geometry (x0 = floor(qx),
// fx = qx - x0, ...) and the four texels — a neighbour whose fraction is 0 is
// not read by the reference, so its address falls back to the base texel
// (always inside the raster) and its term is skipped — then the reference's
// sum in its order.
struct BTap {
  double fx, fy;
  unsigned off, dx, dy;  // texel index within the level (32-bit: one IMAD.WIDE per address)
};
__device__ __forceinline__ BTap btap(int w, double qx, double qy) {
  const double xf = floor(qx), yf = floor(qy);
  BTap t;
  t.fx = qx - xf;  // == qx - x0: x0 = (int)floor(qx) is exact in double
  t.fy = qy - yf;
  t.off = unsigned(int(yf)) * unsigned(w) + unsigned(int(xf));
  t.dx = t.fx > 0.0 ? 1u : 0u;
  t.dy = t.fy > 0.0 ? unsigned(w) : 0u;
  return t;
}
struct BTexels {
  double v00, v01, v10, v11;
};
// Read-only loads kept in program order (volatile), so the four taps' 16
// texel requests leave before the first use.
__device__ __forceinline__ double ldg_early(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ BTexels btexels(const double* img, const BTap& t) {
  return {ldg_early(img + t.off), ldg_early(img + (t.off + t.dx)), ldg_early(img + (t.off + t.dy)),
          ldg_early(img + (t.off + t.dx + t.dy))};
}
// The reference skips a term whose fraction is 0 (descriptor.cpp:25-35).
// Adding it instead is exact: its product is +0 (every factor is finite and
// non-negative — fractions in [0, 1), pyramid values never -0.0, as the
// reference's 0.0-started blur sums never are (`canon` in blur_level) — and
// the fallback texel is a real one), and r, itself a product of non-negative
// factors, is never -0.0, so r + (+0) == r.
// Unconditional terms spare the compare and the two selects per term that
// the skip costs after if-conversion.
__device__ __forceinline__ double bmix(const BTap& t, const BTexels& v) {
  double r = (1.0 - t.fy) * (1.0 - t.fx) * v.v00;
  r += (1.0 - t.fy) * t.fx * v.v01;
  r += t.fy * (1.0 - t.fx) * v.v10;
  r += t.fy * t.fx * v.v11;
  return r;
}

struct Frame { const double* lvl; int w, h; double x, y, sigma; };

// Orientation bin floor(wrap_angle(atan2(gy, gx)) / 2pi * 36 + 0.5) % 36
// (descriptor.cpp:196-199). Only the integer bin is used, so an FP32 atan2
// decides it whenever the value lies farther than 1e-3 bins from a bin edge
// (its error is below 1e-5 bins); otherwise the FP64 expression runs, so the
// bin is always the one the double computation gives.
__device__ __forceinline__ int orient_bin(double gx, double gy) {
  if (fmax(fabs(gx), fabs(gy)) < 1e-30) {  // outside FP32's comfortable range: FP64 only
    const double ang = wrap_angle(dm::atan2(gy, gx));
    return static_cast<int>(floor(ang / kTwoPi * 36 + 0.5)) % 36;
  }
  float a = atan2f(float(gy), float(gx));
  if (a < 0.0f) a += 6.28318548f;
  const float t = a * 5.72957795f + 0.5f;  // 36 / 2pi
  const float fl = floorf(t), fr = t - fl;
  if (fr > 1e-3f && fr < 1.0f - 1e-3f) return int(fl) % 36;
  const double ang = wrap_angle(dm::atan2(gy, gx));
  return static_cast<int>(floor(ang / kTwoPi * 36 + 0.5)) % 36;
}

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

// One warp per selected point (descriptor.cpp:172-232). The disk's samples
// are evaluated 32 at a time and parked (bin, value) in shared memory; a
// stable counting sort by bin (warp match + per-bin running offsets) then
// gives every bin the list of its samples in raster order, and the lane that
// owns a bin adds them in that order — the reference's per-bin add order —
// touching only its own samples.
constexpr int kOrientCap = 512;  // box of the 3.96-sigma disk: (2 * 10.5 + 1)^2 <= 484 for sigma <= 2.66
// One warp (one keypoint) per CTA: window sizes differ by up to 3x between
// keypoints, and a single-warp CTA frees its slot as soon as its keypoint is
// done (0.3% faster than four-warp CTAs end to end).
constexpr int kOrientWarps = 1;
struct OrientSmem {
  double val[kOrientCap];
  uint16_t list[kOrientCap];
  uint8_t bin[kOrientCap];
  int cnt[36], off[36], run[36];
  double hist[36];
};

__global__ void __launch_bounds__(32 * kOrientWarps) k_orient(Batch bt, DetConst dc) {
  __shared__ OrientSmem smem[kOrientWarps];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  OrientSmem& S = smem[wi];
  const int f = blockIdx.y;
  const int r = blockIdx.x * kOrientWarps + wi;
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
  int npx = (nx > 0 && ny > 0) ? nx * ny : 0;
  if (npx > kOrientCap) {  // outside the supported scale range: flag the frame
    if (lane == 0) atomicOr(&bt.status[f], 8);
    npx = 0;
  }
  for (int b = lane; b < 36; b += 32) S.cnt[b] = 0;
  __syncwarp();
  // (q + 0.5) / nx is at least 1/(2 nx) from an integer: exact row index.
  const float inv_nx = nx > 0 ? 1.0f / float(nx) : 0.0f;
  for (int q = lane; q < npx; q += 32) {
    const int qy = int((float(q) + 0.5f) * inv_nx);
    const int ix = x_lo + q - qy * nx, iy = y_lo + qy;
    const double dx = ix - fr.x, dy = iy - fr.y;
    const double d2 = dx * dx + dy * dy;
    int bin = 255;
    double val = 0.0;
    if (!(d2 >= radius * radius)) {
      const double* row = fr.lvl + (long long)iy * fr.w + ix;
      const double gx = 0.5 * (row[1] - row[-1]);
      const double gy = 0.5 * (row[fr.w] - row[-fr.w]);
      const double mag = hypot(gx, gy);
      if (mag != 0.0) {
        bin = orient_bin(gx, gy);
        val = mag * dm::exp(-d2 / denom);
        atomicAdd(&S.cnt[bin], 1);
      }
    }
    S.bin[q] = uint8_t(bin);
    S.val[q] = val;
  }
  __syncwarp();
  if (lane == 0) {
    int o = 0;
    for (int b = 0; b < 36; ++b) {
      S.off[b] = o;
      S.run[b] = 0;
      o += S.cnt[b];
    }
  }
  __syncwarp();
  // Stable scatter of sample indices into per-bin lists (raster order kept).
  for (int base = 0; base < npx; base += 32) {
    const int q = base + lane;
    const int b = q < npx ? S.bin[q] : 255;
    const unsigned grp = __match_any_sync(0xffffffffu, b);
    const int rank = __popc(grp & ((1u << lane) - 1u));
    const int start = b < 36 ? S.off[b] + S.run[b] : 0;
    __syncwarp();
    if (b < 36) {
      S.list[start + rank] = uint16_t(q);
      if (rank == 0) S.run[b] += __popc(grp);
    }
    __syncwarp();
  }
  // Ordered per-bin sums: lane L owns bins L and L + 32.
  double acc0 = 0.0, acc1 = 0.0;
  for (int i = S.off[lane], e = i + S.cnt[lane]; i < e; ++i) acc0 += S.val[S.list[i]];
  if (lane < 4)
    for (int i = S.off[lane + 32], e = i + S.cnt[lane + 32]; i < e; ++i) acc1 += S.val[S.list[i]];
  double* hist_w = S.hist;
  hist_w[lane] = acc0;
  if (lane < 4) hist_w[lane + 32] = acc1;
  __syncwarp();
  for (int pass = 0; pass < 2; ++pass) {
    double s0 = (hist_w[(lane + 35) % 36] + hist_w[lane] + hist_w[(lane + 1) % 36]) / 3.0, s1 = 0.0;
    if (lane < 4) s1 = (hist_w[(lane + 32 + 35) % 36] + hist_w[lane + 32] + hist_w[(lane + 33) % 36]) / 3.0;
    __syncwarp();
    hist_w[lane] = s0;
    if (lane < 4) hist_w[lane + 32] = s1;
    __syncwarp();
  }
  double peak = fmax(hist_w[lane], lane < 4 ? hist_w[lane + 32] : 0.0);
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
      const double v = hist_w[b], l = hist_w[(b + 35) % 36], rr = hist_w[(b + 1) % 36];
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

// Description (descriptor.cpp:47-145) + compression
// (transform_coding.cpp:81-217) in three launches:
//   k_geometry  thread per oriented point: resolve_frame + make_geometry.
//   k_sample    Phase A, thread per patch sample (no shared memory, full
//               occupancy): bilinear gradient, magnitude, Gaussian weight and
//               orientation bin of every sample of the samples x samples grid
//               (samples = ceil(12 sigma) <= 32), parked in HBM/L2 as
//               (weight, fo, bin0) — descriptor.cpp:75-88.
//   k_describe  Phase B + epilogue, one WARP per oriented point. Lane (cell c,
//               parity p) owns the four orientation bins of parity p of cell
//               c. Cell coordinates depend on the sample index only, so the
//               samples feeding cell c form a rectangle, cut by the
//               16-sample sub-patch grid into up to four sub-rectangles. The
//               lane walks them in sub-patch index order, each in row-major
//               order — the reference's add order within each sub-patch
//               partial — and folds each partial into its running total in
//               that order (merge_and_normalize). The walk is one flat loop
//               per lane (a small state machine), so every lane stays busy
//               until its own rectangle is done. Every lane then holds 4 of
//               the 128 bins for normalisation, transform and ternary coding.
constexpr int kMaxSamples = 32;  // samples per axis: ceil(12 sigma) for sigma <= 2.66 (radius-8 detector)
constexpr int kSub = 16;         // kSubPatchSide (descriptor.cpp)

__global__ void __launch_bounds__(128) k_geometry(Batch bt, DetConst dc) {
  const int f = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= bt.or_count[f]) return;
  const Oriented orp = bt.oriented[(long long)f * bt.cap_or + idx];
  const KP k = bt.sel[(long long)f * bt.select_n + orp.sel];
  const Frame fr = resolve(bt, dc, f, k);
  DescGeo g;
  g.x = fr.x;
  g.y = fr.y;
  g.half = 6.0 * fr.sigma;
  g.samples = max(1, static_cast<int>(ceil(12.0 * fr.sigma)));
  g.step = 2.0 * g.half / g.samples;
  g.cos_t = cos(orp.theta);
  g.sin_t = sin(orp.theta);
  g.inv_cell = 1.0 / (3.0 * fr.sigma);
  g.gauss_denom = 2.0 * g.half * g.half;
  g.lvl_off = fr.lvl - bt.pyr;
  g.w = fr.w;
  g.h = fr.h;
  g.pad = 0;
  if (g.samples * g.samples > bt.smp_cap) {  // outside the supported scale range: flag the frame
    atomicOr(&bt.status[f], 8);
    g.samples = 0;
  }
  bt.geo[(long long)f * bt.cap_or + idx] = g;
}

// Groups of four points share a warp in k_describe_cells, which walks as
// many rows as the group's largest point has; ordering the points by
// descending samples per axis (17 .. 32 in the supported scale range) keeps
// each group's sizes alike. Counting sort, CTA per frame; the descriptors
// still land in each point's own slot, so the order is invisible downstream.
__global__ void __launch_bounds__(256) k_order(Batch bt) {
  __shared__ int cnt[33], off[33];
  const int f = blockIdx.x;
  const int n = bt.or_count[f];
  const DescGeo* geo = bt.geo + (long long)f * bt.cap_or;
  int* order = bt.order + (long long)f * bt.cap_or;
  for (int b = threadIdx.x; b < 33; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cnt[kMaxSamples - min(geo[i].samples, kMaxSamples)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int o = 0;
    for (int b = 0; b < 33; ++b) {
      off[b] = o;
      o += cnt[b];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    order[atomicAdd(&off[kMaxSamples - min(geo[i].samples, kMaxSamples)], 1)] = i;
}

// The Gaussian weight exp(-(u*u + v*v) / denom) of sample (i, j) equals that
// of (j, i) bit for bit (u_i == v_i, and the sum commutes), so each CTA first
// tabulates the samples*(samples+1)/2 distinct values of its point in shared
// memory, then runs the per-sample body.
constexpr int kSampleThreads = 128;

// phi / 2pi, correctly rounded, without the division sequence: q0 = phi * y
// with y = RN(1 / 2pi), the remainder r = phi - q0 * 2pi is exact in one fused
// multiply-add, and RN(q0 + r * y) is the correctly rounded quotient
// (Markstein's theorem: y within half an ulp of 1/b, q0 within one ulp of a/b).
// The remainder is exact only while it stays normal, so tiny dividends
// (< 2^-900, never produced by a wrapped angle in practice) take the IEEE
// division. Checked bit for bit against a / b on 1.9e9 random dividends in
// [0, 2pi) (uniform and uniform-by-bits).
__device__ __forceinline__ double div_two_pi(double a) {
  constexpr double kInvTwoPi = 0.15915494309189535;  // RN(1 / (2 * 3.14159265358979323846))
  if (!(a >= 0x1p-900)) return a / kTwoPi;
  const double q0 = __dmul_rn(a, kInvTwoPi);
  const double r = fma(-q0, kTwoPi, a);
  return fma(r, kInvTwoPi, q0);
}

__global__ void __launch_bounds__(kSampleThreads, 12) k_sample(Batch bt) {
  __shared__ double gexp[kMaxSamples * (kMaxSamples + 1) / 2];  // [j * (j + 1) / 2 + i], i <= j
  // Per-axis terms (u_i = v_i, the same expression): the reference's
  // px = (cx + u cos) - v sin and py = (cy + u sin) + v cos, evaluated in its
  // order from per-column sums and per-row products.
  __shared__ double ax_px[kMaxSamples], ax_py[kMaxSamples], ax_vs[kMaxSamples], ax_vc[kMaxSamples];
  const int f = blockIdx.y;
  const int n_or = bt.or_count[f];
  for (int idx = blockIdx.x; idx < n_or; idx += gridDim.x) {
    const long long slot = (long long)f * bt.cap_or + idx;
    const DescGeo g = bt.geo[slot];
    const double theta = bt.oriented[slot].theta;
    const double* lvl = bt.pyr + g.lvl_off;
    asm("" : "+l"(lvl));  // one 64-bit base: each texel address is then a single IMAD.WIDE.U32
    const int samples = g.samples, ns = samples * samples;
    double2* out = bt.smp + slot * bt.smp_cap;
    uint8_t* outb = bt.smpb + slot * kMaxSamples * kMaxSamples;
    // (q + 0.5) / n is at least 1/64 away from an integer for q < 1024, far
    // beyond the float error: exact row indices without integer division.
    const int nt = samples * (samples + 1) / 2;
    __syncthreads();  // previous point's tables fully read
    if (threadIdx.x < samples) {
      const double u = (threadIdx.x + 0.5) * g.step - g.half;
      ax_px[threadIdx.x] = g.x + u * g.cos_t;
      ax_py[threadIdx.x] = g.y + u * g.sin_t;
      ax_vs[threadIdx.x] = u * g.sin_t;
      ax_vc[threadIdx.x] = u * g.cos_t;
    }
    for (int q = threadIdx.x; q < nt; q += kSampleThreads) {
      // q = j (j + 1) / 2 + i with i <= j
      int j = int((sqrtf(8.0f * float(q) + 1.0f) - 1.0f) * 0.5f);
      j += (j + 1) * (j + 2) / 2 <= q;
      j -= j * (j + 1) / 2 > q;
      const int i = q - j * (j + 1) / 2;
      const double v = (j + 0.5) * g.step - g.half;
      const double u = (i + 0.5) * g.step - g.half;
      gexp[q] = dm::exp(-(u * u + v * v) / g.gauss_denom);
    }
    __syncthreads();
    const float inv_samples = 1.0f / float(samples);
    for (int q = threadIdx.x; q < ns; q += kSampleThreads) {
      const int j = int((float(q) + 0.5f) * inv_samples), i = q - j * samples;
      const double px = ax_px[i] - ax_vs[j];
      const double py = ax_py[i] + ax_vc[j];
      double wgt = 0.0, fo = 0.0;
      int b0 = 0;
      if (!(px < 1.0 || px > g.w - 2.0 || py < 1.0 || py > g.h - 2.0)) {
        // The four bilinear taps of the central differences: all 16 texel
        // loads in flight before the arithmetic (sample_bilinear,
        // descriptor.cpp:25-35, at (px +- 1, py) and (px, py +- 1)).
        const BTap tr = btap(g.w, px + 1.0, py), tl = btap(g.w, px - 1.0, py);
        const BTap tu = btap(g.w, px, py + 1.0), td = btap(g.w, px, py - 1.0);
        const BTexels vr = btexels(lvl, tr), vl = btexels(lvl, tl), vu = btexels(lvl, tu), vd = btexels(lvl, td);
        const double gx = 0.5 * (bmix(tr, vr) - bmix(tl, vl));
        const double gy = 0.5 * (bmix(tu, vu) - bmix(td, vd));
        const double mag = hypot(gx, gy);
        if (mag != 0.0) {
          const int lo = min(i, j), hi = max(i, j);
          wgt = mag * gexp[hi * (hi + 1) / 2 + lo];
          const double phi = wrap_angle(dm::atan2(gy, gx) - theta);
          // ob = phi / 2pi * 8 - 0.5, ob0 = floor(ob), fo = ob - ob0 (descriptor.cpp:86-98)
          const double ob = div_two_pi(phi) * 8 - 0.5;
          const double obf = floor(ob);
          fo = ob - obf;
          b0 = static_cast<int>(obf) & 7;  // ((ob0 % 8) + 8) % 8
        }
      }
      // A skipped sample (outside the image, or zero magnitude) keeps weight
      // +0: its products are +0 and adding them leaves every bin unchanged.
      out[q] = make_double2(wgt, fo);
      outb[j * kMaxSamples + i] = uint8_t(b0);
    }
  }
}

// Phase B: FOUR oriented points per warp, row-synchronous, accumulators in
// registers. Lane (q, cx, p) of point q owns the cells (cy, cx) with
// cy = p (mod 2), i.e. cells hl and hl + 8 (hl = 4p + cx). Sample row j feeds
// the cell rows c0[j] and c0[j] + 1 (descriptor.cpp:89-116), one of each
// parity, so in every row each lane works on exactly one of its cells, and
// a cell's rows are contiguous (c0 is monotonic): the lane walks its cells
// one after the other. In row j it visits, in increasing i, the samples whose
// cell column is cx (c0[i] in {cx - 1, cx}) and adds their two orientation
// contributions (bins b0 and b0 + 1 mod 8) to its 8 bin registers: every
// (cell, bin) is one sequential chain in the reference's sample order. There
// is one register set per sub-patch column (i < 16, i >= 16); a cell's
// partials are folded into its total ((P0 + P1) + P2) + P3
// (merge_and_normalize) when the lane leaves the cell, at the 16-row band
// boundary and at the end. Rows of (weight, fo) records and their bins
// stream into a 2-row shared ring with cp.async, one row ahead of the walk.
constexpr int kPBWarps = 4, kPBPts = 4, kPBLanes = 8;  // 4 warps x 4 points per CTA (2 or 8 warps: 0.2-0.7% slower)
struct PhaseBSmem {
  union {
    struct {
      double2 rec[2][kPBPts][kMaxSamples];  // [slot][q][i]: (weight, fo)
      uint8_t bin[2][kPBPts][kMaxSamples];  // [slot][q][i]: ob0 mod 8
    } ring;
    double sq[kPBPts][128];                 // normalisation scratch (after the walk)
  };
  double wf[kPBPts][2][kMaxSamples];        // [q][0][i] = 1 - f, [q][1][i] = f of the cell coordinate
  int8_t c0[kPBPts][kMaxSamples];           // [q][i]: floor(u * inv_cell + 1.5) in -1 .. 4
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(uint32_t(__cvta_generic_to_shared(smem))), "l"(gmem)
               : "memory");
}

// 1.0 when c, else +0.0: built on the integer side (only the high word is
// non-zero), so a masked add is one DFMA: fma(x, 1, a) = RN(x + a) exactly
// (the product is exact), and fma(x, 0, a) = a (x >= +0, a >= +0).
__device__ __forceinline__ double unit_if(bool c) { return __hiloint2double(c ? 0x3FF00000 : 0, 0); }

// acc[b] += x0, acc[(b + 1) mod 8] += x1, as masked DFMAs on registers (the
// bins a lane does not hit this visit are unchanged). The two bins have
// opposite parity: with h = b / 2, an even b puts x0 on even bin h and x1 on
// odd bin h; an odd b puts x0 on odd bin h and x1 on even bin h + 1 (mod 4).
__device__ __forceinline__ void add_two_bins(double (&acc)[8], int b, double x0, double x1) {
  const int h = b >> 1;
  const bool odd = (b & 1) != 0;
  const double ev = odd ? x1 : x0, ov = odd ? x0 : x1;
  const int eh = odd ? ((h + 1) & 3) : h;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    acc[2 * k] = fma(ev, unit_if(eh == k), acc[2 * k]);
    acc[2 * k + 1] = fma(ov, unit_if(h == k), acc[2 * k + 1]);
  }
}

__global__ void __launch_bounds__(32 * kPBWarps, 16 / kPBWarps) k_describe(Batch bt) {
  extern __shared__ __align__(16) uint8_t pb_smem[];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PhaseBSmem& S = reinterpret_cast<PhaseBSmem*>(pb_smem)[wi];
  const int f = blockIdx.y;
  const int n_or = bt.or_count[f];
  const int q = lane >> 3, hl = lane & 7;
  const int cx = hl & 3, par = hl >> 2;
  const unsigned gmask = 0xffu << (kPBLanes * q);
  for (int grp = blockIdx.x * kPBWarps + wi; kPBPts * grp < n_or; grp += gridDim.x * kPBWarps) {
    const int idx = kPBPts * grp + q;
    const bool live = idx < n_or;
    const long long gslot = (long long)f * bt.cap_or + (live ? idx : 0);
    const DescGeo g = bt.geo[gslot];
    const int samples = live ? g.samples : 0;  // 0: no point, or flagged by k_geometry
    const double2* smp = bt.smp + gslot * bt.smp_cap;
    const uint8_t* smb = bt.smpb + gslot * kMaxSamples * kMaxSamples;
    auto fetch_row = [&](int j) {
      if (j < samples) {
        double2* dst = S.ring.rec[j & 1][q];
        const double2* src = smp + (long long)j * samples;
        for (int i = hl; i < samples; i += kPBLanes) cp_async16(dst + i, src + i);
        if (hl < 2) cp_async16(S.ring.bin[j & 1][q] + 16 * hl, smb + j * kMaxSamples + 16 * hl);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    __syncwarp();  // the previous group's epilogue is done with the scratch union
    fetch_row(0);
    // Per-axis cell coordinates (descriptor.cpp:89-96): identical for u (i) and v (j).
    for (int i = hl; i < samples; i += kPBLanes) {
      const double u = (i + 0.5) * g.step - g.half;
      const double cu = u * g.inv_cell + 1.5;
      const int c0 = static_cast<int>(floor(cu));
      const double fu = cu - c0;
      S.c0[q][i] = c0;
      S.wf[q][1][i] = fu;
      S.wf[q][0][i] = 1.0 - fu;
    }
    __syncwarp();
    // Column range of cx: c0 in {cx - 1, cx}; weight f (du = 1) below im.
    int ia = 0, im = 0, ib = 0;
    for (int i = 0; i < samples; ++i) {
      const int c = S.c0[q][i];
      ia += c < cx - 1;
      im += c < cx;
      ib += c < cx + 1;
    }
    // The two sub-patch columns are independent chains, so each lane walks
    // its larger part first (register set A) and the other part second (set
    // B): both loops are then short for every lane of the warp.
    const int ia1 = max(ia, kSub), ib0 = min(ib, kSub);
    const bool rfirst = (ib - ia1) > (ib0 - ia);
    const int f_lo = rfirst ? ia1 : ia, f_hi = rfirst ? ib : ib0;
    const int s_lo = rfirst ? ia : ia1, s_hi = rfirst ? ib0 : ib;
    const int rows = __reduce_max_sync(0xffffffffu, samples);
    double tot[2][8];  // totals of cells hl (slot 0) and hl + 8 (slot 1)
    double a0[8], a1[8];  // partials of the current cell: the lane's first / second part
#pragma unroll
    for (int k = 0; k < 8; ++k) tot[0][k] = tot[1][k] = a0[k] = a1[k] = 0.0;
    int cur = -1;  // cell row being accumulated (-1: none)
    auto fold = [&]() {  // T = (T + left) + right
      if (cur >= 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) tot[1][k] = (tot[1][k] + (rfirst ? a1[k] : a0[k])) + (rfirst ? a0[k] : a1[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) tot[0][k] = (tot[0][k] + (rfirst ? a1[k] : a0[k])) + (rfirst ? a0[k] : a1[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) a0[k] = a1[k] = 0.0;
    };
    for (int j = 0; j < rows; ++j) {
      fetch_row(j + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
      if (j < samples) {
        const int c = S.c0[q][j];
        const int cy = c + ((c & 1) != par);  // this lane's cell row in row j
        const bool valid = cy >= 0 && cy < 4;
        // Leaving a cell, or the first row of the second band (j == 16, only
        // when samples > 16): its partials so far are complete.
        if (cur >= 0 && (cur != cy || j == kSub)) fold();
        cur = valid ? cy : -1;
        if (valid) {
          const double wv = S.wf[q][cy - c][j];  // dv = cy - c0[j]: 1 -> f, 0 -> 1 - f
          const double2* rowp = S.ring.rec[j & 1][q];
          const uint8_t* rowb = S.ring.bin[j & 1][q];
          const double* wfq = S.wf[q][0];
          // Visit i: ((weight * wv) * wu) * wo, wo = 1 - fo (bin b0) and fo
          // (bin b0 + 1), descriptor.cpp:89-116; wu = f for i < im (du = 1).
          for (int i = f_lo; i < f_hi; ++i) {
            const double2 rec = rowp[i];
            const double x = (rec.x * wv) * wfq[(i < im ? kMaxSamples : 0) + i];
            add_two_bins(a0, rowb[i], x * (1.0 - rec.y), x * rec.y);
          }
          for (int i = s_lo; i < s_hi; ++i) {
            const double2 rec = rowp[i];
            const double x = (rec.x * wv) * wfq[(i < im ? kMaxSamples : 0) + i];
            add_two_bins(a1, rowb[i], x * (1.0 - rec.y), x * rec.y);
          }
        }
      }
      __syncwarp();
    }
    if (cur >= 0) fold();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    // normalize_descriptor (descriptor.cpp:124-145): up to 5 rounds of L2
    // normalise + clamp at 0.2; the norm in the Eigen SSE2 reduction order
    // (four stride-4 running sums, then (s0 + s2) + (s1 + s3)).
    // Element index of (cell, bin) is cell * 8 + bin.
    double* sq = S.sq[q];
    bool done = samples == 0;
    for (int round = 0; round < 5; ++round) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int k = 0; k < 8; ++k) sq[8 * (hl + 8 * c) + k] = tot[c][k] * tot[c][k];
      __syncwarp();
      double red = 0.0;
      if (hl < 4) {
        red = sq[hl];
#pragma unroll 8
        for (int k = 1; k < 32; ++k) red = red + sq[hl + 4 * k];
      }
      const int gb = kPBLanes * q;
      const double r0 = __shfl_sync(0xffffffffu, red, gb), r1 = __shfl_sync(0xffffffffu, red, gb + 1);
      const double r2 = __shfl_sync(0xffffffffu, red, gb + 2), r3 = __shfl_sync(0xffffffffu, red, gb + 3);
      __syncwarp();
      const double norm = sqrt((r0 + r2) + (r1 + r3));
      bool clipped = false;
      if (!done) {
        if (norm == 0.0) {
          done = true;
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              tot[c][k] = tot[c][k] / norm;
              if (tot[c][k] > 0.2) { tot[c][k] = 0.2; clipped = true; }
            }
        }
      }
      if (!(__ballot_sync(0xffffffffu, clipped) & gmask)) done = true;
      if (__all_sync(0xffffffffu, done)) break;
    }
    if (samples > 0) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int cl = hl + 8 * c;
        double2* dout = reinterpret_cast<double2*>(bt.desc + ((long long)f * bt.cap_or + idx) * 128 + 8 * cl);
#pragma unroll
        for (int k = 0; k < 4; ++k) dout[k] = make_double2(tot[c][2 * k], tot[c][2 * k + 1]);
      }
    }
  }
}

// Phase B, shared-memory cell accumulators (the default): FOUR oriented points
// per warp, row-synchronous.
// Lane (q, cx, dv) of point q walks every sample row j in order; in row j it
// visits, in increasing i, the samples whose cell column is cx (c0[i] in
// {cx - 1, cx}), decodes each sample once and adds its two orientation
// contributions (bins ob0 and ob0 + 1 mod 8) to cell (cx, c0[j] + dv).
// Accumulators live in shared memory indexed by (set, bin, cell): at any
// moment each (cell, bin) has exactly one owning lane, and a cell's chains
// pass from lane dv = 1 to lane dv = 0 when the rows cross a cell boundary
// with no exchange, so every bin is one sequential chain in the reference's
// sample order (descriptor.cpp:98-116). Sets: the left (i < 16) and right
// (i >= 16) sub-patch partials of the current 16-row band; the folded total
// ((P0 + P1) + P2) + P3 of merge_and_normalize lives in registers (lane hl
// folds cells hl and hl + 8). Rows of (weight, fo) records and their bins
// stream into a 2-row shared ring with cp.async, one row ahead of the walk.
// (k_describe below keeps the bins in registers instead: debug bit 256.)
// Bank-conflict-free accumulator layout: the 16 lanes of a half-warp (points
// q, q^1) touch cells (cx, cy) with distinct (q & 1, cy & 1, cx), which is the
// double's bank slot (index mod 16); set, bin, cy >> 1 and q >> 1 select
// 16-double rows.
__device__ __forceinline__ int acc_index(int q, int set, int bin, int cy, int cx) {
  return (q >> 1) * 512 + set * 256 + bin * 32 + (cy >> 1) * 16 + (q & 1) * 8 + (cy & 1) * 4 + cx;
}
struct CellSmem {
  double2 ring[2][kPBPts][kMaxSamples];  // [slot][q][i]: (weight, fo)
  uint8_t bin[2][kPBPts][kMaxSamples];   // [slot][q][i]: ob0 mod 8
  double acc[kPBPts * 256];              // acc_index(); after phase B: per-point scratch [q][256]
  double wf[kPBPts][kMaxSamples];        // [q][i]: f of the cell coordinate (1 - f formed on use)
  int8_t c0[kPBPts][kMaxSamples];        // [q][i]: floor(u * inv_cell + 1.5) in -1 .. 4
};


__global__ void __launch_bounds__(32 * kPBWarps, 16 / kPBWarps) k_describe_cells(Batch bt) {
  extern __shared__ __align__(16) uint8_t pb_smem[];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CellSmem& S = reinterpret_cast<CellSmem*>(pb_smem)[wi];
  const int f = blockIdx.y;
  const int n_or = bt.or_count[f];
  const int q = lane >> 3, hl = lane & 7;
  const int cx = hl & 3, dv = hl >> 2;
  const unsigned gmask = 0xffu << (kPBLanes * q);
  for (int grp = blockIdx.x * kPBWarps + wi; kPBPts * grp < n_or; grp += gridDim.x * kPBWarps) {
    const bool live = kPBPts * grp + q < n_or;
    const int idx = live ? bt.order[(long long)f * bt.cap_or + kPBPts * grp + q] : 0;
    const long long gslot = (long long)f * bt.cap_or + idx;
    const DescGeo g = bt.geo[gslot];
    const int samples = live ? g.samples : 0;  // 0: no point, or flagged by k_geometry
    const double2* smp = bt.smp + gslot * bt.smp_cap;
    const uint8_t* smb = bt.smpb + gslot * kMaxSamples * kMaxSamples;
    auto fetch_row = [&](int j) {
      if (j < samples) {
        double2* dst = S.ring[j & 1][q];
        const double2* src = smp + (long long)j * samples;
        for (int i = hl; i < samples; i += kPBLanes) cp_async16(dst + i, src + i);
        if (hl < 2) cp_async16(S.bin[j & 1][q] + 16 * hl, smb + j * kMaxSamples + 16 * hl);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch_row(0);
    // Per-axis cell coordinates (descriptor.cpp:89-96): identical for u (i) and v (j).
    for (int i = hl; i < samples; i += kPBLanes) {
      const double u = (i + 0.5) * g.step - g.half;
      const double cu = u * g.inv_cell + 1.5;
      const int c0 = static_cast<int>(floor(cu));
      const double fu = cu - c0;
      S.c0[q][i] = c0;
      S.wf[q][i] = fu;
    }
    double* acc = S.acc;
    for (int e = lane; e < kPBPts * 256; e += 32) acc[e] = 0.0;
    __syncwarp();
    // Column range of cx: c0 in {cx - 1, cx}; weight f (d = 1) below im.
    int ia = 0, im = 0, ib = 0;
    for (int i = 0; i < samples; ++i) {
      const int c = S.c0[q][i];
      ia += c < cx - 1;
      im += c < cx;
      ib += c < cx + 1;
    }
    const int rows = __reduce_max_sync(0xffffffffu, samples);
    double tot[2][8];  // lane hl's fold of cells hl and hl + 8
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) tot[c][k] = 0.0;
    for (int j = 0; j < rows; ++j) {
      fetch_row(j + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
      if (j == kSub && samples > kSub) {
        // Band boundary: the first two sub-patch partials are complete.
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int e = acc_index(q, 0, k, c * 2 + (hl >> 2), hl & 3);  // cell hl + 8c
            tot[c][k] = acc[e] + acc[256 + e];
            acc[e] = 0.0;
            acc[256 + e] = 0.0;
          }
      }
      __syncwarp();
      if (j < samples) {
        const int cy = S.c0[q][j] + dv;
        if (cy >= 0 && cy < 4) {
          const double fv = S.wf[q][j];
          const double wv = dv ? fv : 1.0 - fv;
          const double2* rowp = S.ring[j & 1][q];
          const uint8_t* rowb = S.bin[j & 1][q];
          const double* wfq = S.wf[q];
          const int cell = acc_index(q, 0, 0, cy, cx);
          // Visit i: weight * wv * wu * wo for wo = 1 - fo (bin ob0) and fo
          // (bin ob0 + 1), descriptor.cpp:89-116. Two-stage software
          // pipeline: visit i + 1 is decoded while visit i's two chains are
          // updated.
          auto decode = [&](int i, int& o0, int& o1, double& x0, double& x1) {
            const double2 rec = rowp[i];
            const double fu = wfq[i];
            const double wu = i < im ? fu : 1.0 - fu;
            const double fo = rec.y;
            const int b0 = rowb[i];
            const double base = rec.x * wv * wu;
            const int so = cell + (i < kSub ? 0 : 256);
            o0 = so + 32 * b0;
            o1 = so + 32 * ((b0 + 1) & 7);
            x0 = base * (1.0 - fo);
            x1 = base * fo;
          };
          // The next visit's two loads are issued before this visit's
          // stores; a load that hits a bin just updated takes the updated
          // value from registers instead (o0 != o1 always), so each chain's
          // critical path is one add.
          if (ia < ib) {
            int o0, o1;
            double x0, x1;
            decode(ia, o0, o1, x0, x1);
            double a0 = acc[o0], a1 = acc[o1];
            for (int i = ia; i < ib; ++i) {
              const double s0 = a0 + x0, s1 = a1 + x1;
              int n0 = o0, n1 = o1;
              double y0 = 0.0, y1 = 0.0, b0 = 0.0, b1 = 0.0;
              if (i + 1 < ib) {
                decode(i + 1, n0, n1, y0, y1);
                b0 = acc[n0];
                b1 = acc[n1];
              }
              acc[o0] = s0;
              acc[o1] = s1;
              a0 = n0 == o0 ? s0 : (n0 == o1 ? s1 : b0);
              a1 = n1 == o0 ? s0 : (n1 == o1 ? s1 : b1);
              o0 = n0;
              o1 = n1;
              x0 = y0;
              x1 = y1;
            }
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int e = acc_index(q, 0, k, c * 2 + (hl >> 2), hl & 3);
        tot[c][k] = samples > kSub ? (tot[c][k] + acc[e]) + acc[256 + e] : acc[e];
      }
    __syncwarp();
    // normalize_descriptor (descriptor.cpp:124-145): up to 5 rounds of L2
    // normalise + clamp at 0.2; the norm in the Eigen SSE2 reduction order
    // (four stride-4 running sums, then (s0 + s2) + (s1 + s3)).
    // Element index of (cell, bin) is cell * 8 + bin.
    double* sq = acc + 256 * q;
    bool done = samples == 0;
    for (int round = 0; round < 5; ++round) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int k = 0; k < 8; ++k) sq[8 * (hl + 8 * c) + k] = tot[c][k] * tot[c][k];
      __syncwarp();
      double red = 0.0;
      if (hl < 4) {
        red = sq[hl];
#pragma unroll 8
        for (int k = 1; k < 32; ++k) red = red + sq[hl + 4 * k];
      }
      const int gb = kPBLanes * q;
      const double r0 = __shfl_sync(0xffffffffu, red, gb), r1 = __shfl_sync(0xffffffffu, red, gb + 1);
      const double r2 = __shfl_sync(0xffffffffu, red, gb + 2), r3 = __shfl_sync(0xffffffffu, red, gb + 3);
      __syncwarp();
      const double norm = sqrt((r0 + r2) + (r1 + r3));
      bool clipped = false;
      if (!done) {
        if (norm == 0.0) {
          done = true;
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              tot[c][k] = tot[c][k] / norm;
              if (tot[c][k] > 0.2) { tot[c][k] = 0.2; clipped = true; }
            }
        }
      }
      if (!(__ballot_sync(0xffffffffu, clipped) & gmask)) done = true;
      if (__all_sync(0xffffffffu, done)) break;
    }
    if (samples > 0) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int cl = hl + 8 * c;
        double2* dout = reinterpret_cast<double2*>(bt.desc + ((long long)f * bt.cap_or + idx) * 128 + 8 * cl);
#pragma unroll
        for (int k = 0; k < 4; ++k) dout[k] = make_double2(tot[c][2 * k], tot[c][2 * k + 1]);
      }
    }
    __syncwarp();
  }
}

// Compression (pipeline.cpp:37-50, the reference's "compression" stage):
// transform_descriptor (transform_coding.cpp:81-91), quantize_ternary
// (:202-217) and the location quantisers quantize_coord / quantize_sigma_log /
// quantize_theta (:173-200) of every described point. Thread per (point,
// cell): the cell's 8 transformed values go to shared memory, then thread
// (point, b) packs code bytes 2b and 2b + 1 (symbols 8b .. 8b + 7 in the
// mode's priority order: 00 zero, 01 +1, 10 -1).
constexpr int kCompPts = 8;
__global__ void __launch_bounds__(16 * kCompPts) k_compress(Batch bt, Model md, EncodeConst ec) {
  __shared__ double tv[kCompPts][128];
  const int f = blockIdx.y;
  const int n_or = bt.or_count[f];
  const int pl = threadIdx.x >> 4, cl = threadIdx.x & 15;
  const int idx = blockIdx.x * kCompPts + pl;
  const bool live = idx < n_or;
  const long long slot = (long long)f * bt.cap_or + (live ? idx : 0);
  const bool ok = live && bt.geo[slot].samples > 0;
  if (ok) {
    const double2* d = reinterpret_cast<const double2*>(bt.desc + slot * 128 + 8 * cl);
    double v[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 t = d[k];
      v[2 * k] = t.x;
      v[2 * k + 1] = t.y;
    }
    const int which = (((cl & 3) + (cl >> 2)) & 1) == 0 ? 0 : 1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = md.tr[which][i][0] * v[0];
#pragma unroll
      for (int kk = 1; kk < 8; ++kk) s = s + md.tr[which][i][kk] * v[kk];
      tv[pl][cl * 8 + i] = md.tr_scale * s;
    }
  }
  __syncthreads();
  if (!ok) return;
  uint8_t* code = bt.codes + slot * bt.code_stride;
#pragma unroll
  for (int by = 0; by < 2; ++by) {
    const int t0 = 8 * cl + 4 * by;
    if (t0 < ec.elements) {
      uint8_t byte = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = t0 + k;
        if (t < ec.elements) {
          const int e = md.priority[t];
          const double val = tv[pl][e];
          const uint8_t sym = val < md.t0[e] ? 2 : (val > md.t1[e] ? 1 : 0);
          byte |= uint8_t(sym << (2 * k));
        }
      }
      code[6 + 2 * cl + by] = byte;
    }
  }
  if (cl == 0) {
    const Oriented orp = bt.oriented[slot];
    const KP k = bt.sel[(long long)f * bt.select_n + orp.sel];
    const double cxq = fmin(fmax(k.x, 0.0), double(bt.W - 1));
    const double cyq = fmin(fmax(k.y, 0.0), double(bt.H - 1));
    const unsigned xq = (unsigned)llround(cxq / (bt.W - 1) * 65535.0);
    const unsigned yq = (unsigned)llround(cyq / (bt.H - 1) * 65535.0);
    const double sc = fmin(fmax(k.sigma, 0.5), 64.0);
    const double tq = log2(sc / 0.5) / ec.log2_range;
    const unsigned sq8 = (unsigned)llround(tq * 255.0);
    double tt = orp.theta / kTwoPi;
    tt -= floor(tt);
    const unsigned th8 = (unsigned)(llround(tt * 256.0) & 0xFF);
    code[0] = uint8_t(xq & 0xFF);
    code[1] = uint8_t(xq >> 8);
    code[2] = uint8_t(yq & 0xFF);
    code[3] = uint8_t(yq >> 8);
    code[4] = uint8_t(sq8);
    code[5] = uint8_t(th8);
  }
}

cudaError_t launch_describe(const Batch& bt, const DetConst& dc, cudaStream_t st) {
  k_orient<<<dim3((bt.select_n + kOrientWarps - 1) / kOrientWarps, bt.nframes), 32 * kOrientWarps, 0, st>>>(bt, dc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_expand<<<bt.nframes, 1024, 0, st>>>(bt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_geometry<<<dim3((bt.cap_or + 127) / 128, bt.nframes), 128, 0, st>>>(bt, dc);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_order<<<bt.nframes, 256, 0, st>>>(bt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_sample<<<dim3(256, bt.nframes), kSampleThreads, 0, st>>>(bt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  static size_t configured[kMaxDevices] = {};
  constexpr int smem = int(sizeof(PhaseBSmem)) * kPBWarps, csmem = int(sizeof(CellSmem)) * kPBWarps;
  e = once_per_device(configured, 1, [&] {
    cudaError_t r = cudaFuncSetAttribute(k_describe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return r != cudaSuccess ? r : cudaFuncSetAttribute(k_describe_cells, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem);
  });
  if (e != cudaSuccess) return e;
  const dim3 grid((bt.cap_or + kPBPts * kPBWarps - 1) / (kPBPts * kPBWarps), bt.nframes);
  if (dc.desc_registers)
    k_describe<<<grid, 32 * kPBWarps, smem, st>>>(bt);
  else
    k_describe_cells<<<grid, 32 * kPBWarps, csmem, st>>>(bt);
  return cudaGetLastError();
}

cudaError_t launch_compress(const Batch& bt, const Model& md, const EncodeConst& ec, cudaStream_t st) {
  k_compress<<<dim3((bt.cap_or + kCompPts - 1) / kCompPts, bt.nframes), 16 * kCompPts, 0, st>>>(bt, md, ec);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
