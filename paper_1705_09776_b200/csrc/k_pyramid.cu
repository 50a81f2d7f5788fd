// K1 — fused octave kernel: separable Gaussian scale space (4 levels, each
// blurred from the octave base), sigma^2-normalised 3x3 Laplacian, ALP cubic
// fit alpha = beta * L, analytic scale extrema with the strict 8-neighbour
// test, and sub-pixel refinement with the edge test — one pass over the base.
//
// Replaces gaussian_blur / laplacian_3x3 (proj/src/image.cpp:177-238),
// build_octave / detect_extrema / refine_candidates
// (proj/src/scale_space.cpp:141-270).
//
// Layout and schedule. One CTA owns a vertical strip of S
// output columns of one frame and walks it top to bottom, one "virtual row"
// v = -R..h-1+R per step (rows outside [0,h) are the mirror-reflected rows the
// reference's y pass reads). Each thread owns one column (plus 2 halo columns
// each side so the Laplacian and the 8-neighbour test stay CTA-local):
//   1. the base row mirror(v) is staged in shared memory (u8 -> b/255 for
//      octave 0; G3 of the previous octave at even coordinates otherwise);
//   2. x pass for all 4 levels from that row into per-level register rings;
//   3. y pass from the rings -> G row v-R, stored to HBM (the descriptor
//      stages read it) and to a 3-row shared ring;
//   4. Laplacian + alpha for row v-R-1 into a 3-row shared ring;
//   5. extrema + refinement for row v-R-2; survivors are appended to the
//      frame's unordered list and flagged in a raster bitmap, from which
//      k_merge_octave recovers the reference's sorted order exactly.
// The only HBM traffic is the base read (1 B/px at octave 0) and the 4 G
// levels written (32 B/px): the L planes, the x-pass temporaries and the
// candidate list of the reference never leave the SM.
//
// Every sum runs in the reference's order (taps j = -r..r, Laplacian
// ((up+down)+left)+right-4c, alpha in column order) with separately rounded
// multiplies and adds (--fmad=false), so G, alpha and every candidate are
// bit-identical to the oracle.
#include <cuda.h>

#include "common.cuh"

namespace cdvz_gpu {

namespace {

__device__ __forceinline__ double poly_at(const double a[4], double s) { return a[0] + s * (a[1] + s * (a[2] + s * a[3])); }

// scale_space.cpp:20-43
__device__ __forceinline__ int derivative_roots(const double a[4], double r[2]) {
  const double qa = 3.0 * a[3], qb = 2.0 * a[2], qc = a[1];
  if (qa == 0.0) {
    if (qb == 0.0) return 0;
    r[0] = -qc / qb;
    return 1;
  }
  const double disc = qb * qb - 4.0 * qa * qc;
  if (disc < 0.0) return 0;
  const double sq = sqrt(disc);
  const double q = -0.5 * (qb + copysign(sq, qb));
  int n = 0;
  if (q != 0.0) {
    r[n++] = q / qa;
    r[n++] = qc / q;
  } else {
    r[n++] = 0.0;
  }
  if (n == 2 && r[0] == r[1]) n = 1;
  return n;
}

// Mirror for indices within one period of the border (|overhang| < n):
// -1 -> 0, n -> n-1 (common.hpp:24-30 restricted to the range the walks use).
__device__ __forceinline__ int mirror_near(int i, int n) { return i < 0 ? -1 - i : (i >= n ? 2 * n - 1 - i : i); }

// Base sources: 0 u8 frames (4-byte aligned rows), 3 u8 frames (unaligned
// rows), 1 resized f64 frames, 2 G3 of the previous octave.
template <int SRC> struct RawT { using type = double; };
template <> struct RawT<0> { using type = uint8_t; };
template <> struct RawT<3> { using type = uint8_t; };

template <int SRC>
__device__ __forceinline__ typename RawT<SRC>::type load_raw(const Batch& bt, int f, int o, int ry, int xx) {
  if constexpr (SRC == 0) return bt.pix8[f * bt.frame_bytes8 + (long long)ry * bt.stride8 + xx];
  else if constexpr (SRC == 1) return bt.pixf[(long long)f * bt.W * bt.H + (long long)ry * bt.W + xx];
  else return bt.pyr[f * bt.frame_doubles + bt.plane_off[o - 1][3] + (long long)(2 * ry) * bt.ow[o - 1] + 2 * xx];
}

template <int SRC>
__device__ __forceinline__ double to_base(typename RawT<SRC>::type v) {
  if constexpr (SRC == 0) return v * (1.0 / 255.0);  // image.cpp:79-87: raw * (1.0 / 255.0)
  else return v;
}

template <int SRC>
__device__ __forceinline__ double load_base(const Batch& bt, int f, int o, int ry, int xx) {
  if constexpr (SRC == 0) {
    const uint8_t b = bt.pix8[f * bt.frame_bytes8 + (long long)ry * bt.stride8 + xx];
    return b * (1.0 / 255.0);  // image.cpp:79-87: raw * (1.0 / 255.0)
  } else if constexpr (SRC == 1) {
    return bt.pixf[(long long)f * bt.W * bt.H + (long long)ry * bt.W + xx];
  } else {  // downsample_half(G3 of octave o-1): image.cpp:147-155
    const double* g3 = bt.pyr + f * bt.frame_doubles + bt.plane_off[o - 1][3];
    return g3[(long long)(2 * ry) * bt.ow[o - 1] + 2 * xx];
  }
}

}  // namespace

// Exact candidate test + refinement for one pixel whose alpha rows are in
// shared memory (scale_space.cpp:172-205 and :221-266). Emits survivors.
__device__ __forceinline__ void exact_detect(const Batch& bt, const DetConst& dc, int f, int o, int w, int yd, int cx,
                                          const double* up, const double* mid, const double* dn, int T, int t,
                                          double oct_scale) {
  const double* arow[3] = {up, mid, dn};
  double a[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = mid[i * T + t];
  double roots[2];
  const int nr = derivative_roots(a, roots);
  for (int ri = 0; ri < nr; ++ri) {
    const double s = roots[ri];
    if (s < dc.s_lo || s > dc.s_hi) continue;
    const double p = poly_at(a, s);
    if (fabs(p) < dc.thr) continue;
    double p3[3][3];
    bool ext = true;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        double an[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) an[i] = arow[dy + 1][i * T + t + dx];
        const double pn = (dx == 0 && dy == 0) ? p : poly_at(an, s);
        p3[dy + 1][dx + 1] = pn;
        if (!(dx == 0 && dy == 0) && (p > 0.0 ? (p <= pn) : (p >= pn))) ext = false;
      }
    if (!ext) continue;
    const double gx = 0.5 * (p3[1][2] - p3[1][0]);
    const double gy = 0.5 * (p3[2][1] - p3[0][1]);
    const double hxx = p3[1][2] + p3[1][0] - 2.0 * p3[1][1];
    const double hyy = p3[2][1] + p3[0][1] - 2.0 * p3[1][1];
    const double hxy = 0.25 * (p3[2][2] - p3[2][0] - p3[0][2] + p3[0][0]);
    const double det = hxx * hyy - hxy * hxy;
    if (det <= 0.0) continue;
    const double rho = (hxx + hyy) * (hxx + hyy) / det;
    if (rho > dc.rho_limit) continue;
    const double ox = -(hyy * gx - hxy * gy) / det;
    const double oy = (hxy * gx - hxx * gy) / det;
    if (fabs(ox) > 0.6 || fabs(oy) > 0.6) continue;
    KP k;
    k.x = (cx + ox) * oct_scale;
    k.y = (yd + oy) * oct_scale;
    k.sigma = s * oct_scale;
    k.p = p;
    k.rho = rho;
    k.pss = 2.0 * a[2] + 6.0 * a[3] * s;
    k.d = 0.0;
    k.octave = o;
    const int slot = (nr == 2 && s > roots[1 - ri]) ? 1 : 0;  // sigma order within the pixel
    k.key = (uint32_t(yd) * uint32_t(w) + uint32_t(cx)) * 2u + uint32_t(slot);
    const int idx = atomicAdd(&bt.raw_count[f * bt.n_oct + o], 1);
    if (idx < bt.cap_oct) {
      bt.raw[((long long)f * bt.n_oct + o) * bt.cap_oct + idx] = k;
      atomicOr(&bt.bitmap[f * bt.bitmap_words + bt.bm_off[o] + (k.key >> 5)], 1u << (k.key & 31u));
    } else {
      atomicOr(&bt.status[f], 4);
    }
  }
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Conservative FP32 screen (FP32 pipe + MUFU, beside the FP64 work) on the
// float copies of alpha (each alpha converted once, when its row is formed):
// a pixel is dropped only when the discriminant is clearly negative (the
// reference's own test is disc < 0: no real root), or no float root lies
// within [s_lo - 0.05, s_hi + 0.05], or no in-range root can reach |p| >= thr
// with a margin of 1e-5 of the coefficient magnitudes, or the up or down
// neighbour is clearly past p — every margin orders of magnitude above the
// float error (the alpha copies are within 6e-8 relative of the exact values;
// fused multiply-adds are fine: this only screens). Near-double roots and
// degenerate cases go to the exact path.
//
// The magnitude bounds are taken at the largest screened scale r_max =
// s_hi + 0.05 (r <= r_max, so they bound the per-root values from above and
// only widen the margins): B(x) = sum |x_i| r_max^i for the pixel's own cubic,
// M(x) = B(x) + sum i |x_i| r_max^(i-1) (value plus slope) for a neighbour's;
// both are formed once per pixel, when its alpha row is made.
__device__ __forceinline__ float mag_bound(const float a[4], float rm) {
  return __fmaf_rn(rm, __fmaf_rn(rm, __fmaf_rn(rm, fabsf(a[3]), fabsf(a[2])), fabsf(a[1])), fabsf(a[0]));
}
__device__ __forceinline__ float nbr_bound(const float a[4], float rm) {
  const float slope = __fmaf_rn(rm, __fmaf_rn(rm, 3.0f * fabsf(a[3]), 2.0f * fabsf(a[2])), fabsf(a[1]));
  return mag_bound(a, rm) + slope;
}

__device__ __forceinline__ bool screen_pixel(const float a[4], float ba, const float up[4], float mu, const float dn[4],
                                              float md, const DetConst& dc) {
  const float fa = 3.0f * a[3], fb = 2.0f * a[2], fc = a[1];
  if (fa == 0.0f) return true;
  const float bb = fb * fb, ac4 = 4.0f * fa * fc;
  const float fd = bb - ac4;
  const float de = 1e-5f * (bb + fabsf(ac4)) + 1e-30f;
  if (fd < -de) return false;         // the reference's disc < 0, by a margin
  if (!(fd > de)) return true;        // near-double root, or not finite: the exact path decides
  const float sq = fd * rsqrt_approx(fd);
  const float q = -0.5f * (fb + copysignf(sq, fb));
  if (!(fabsf(q) > 1e-30f)) return true;
  const float r0 = q * rcp_approx(fa), r1 = fc * rcp_approx(q);
  auto horner = [](float r, const float c[4]) {
    return __fmaf_rn(r, __fmaf_rn(r, __fmaf_rn(r, c[3], c[2]), c[1]), c[0]);
  };
  // The exact test needs p above (p > 0) or below (p < 0) all eight
  // neighbours' cubics at the same scale; drop the root only when the up or
  // down neighbour is clearly past p. The float root is within ~1e-6 s of the
  // exact one and p is stationary there, so a margin of 1e-4 of the
  // magnitudes (values plus slopes) is far beyond the float error.
  const float m = 1e-4f * (ba + mu + md) + 1e-7f;
  const float tmargin = __fmaf_rn(1e-5f, ba, 1e-6f);
  bool any = false;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float r = k ? r1 : r0;
    if (!(r >= dc.scr_lo && r <= dc.scr_hi)) {
      if (!isfinite(r)) any = true;
      continue;
    }
    const float p = horner(r, a);
    if (!(fabsf(p) + tmargin >= dc.scr_thr)) continue;
    const float pu = horner(r, up), pd = horner(r, dn);
    const bool past = p > 0.0f ? (pu >= p + m || pd >= p + m) : (pu <= p - m || pd <= p - m);
    if (!past) any = true;
  }
  return any;
}

// screen_pixel with no early exits: every predicate of the test above is
// evaluated for both roots and combined with bitwise logic, so the walk's
// screen is straight-line predicated code (no divergent branches and
// reconvergence points per pixel). The result is the same function of the
// inputs: where the branchy form returns early, the garbage values computed
// past that point (rsqrt of a negative, rcp of 0) are masked by the same
// predicate.
__device__ __forceinline__ bool screen_pixel_flat(const float a[4], float ba, const float up[4], float mu,
                                                   const float dn[4], float md, const DetConst& dc) {
  const float fa = 3.0f * a[3], fb = 2.0f * a[2], fc = a[1];
  const float bb = fb * fb, ac4 = 4.0f * fa * fc;
  const float fd = bb - ac4;
  const float de = 1e-5f * (bb + fabsf(ac4)) + 1e-30f;
  const float sq = fd * rsqrt_approx(fd);
  const float q = -0.5f * (fb + copysignf(sq, fb));
  const float r0 = q * rcp_approx(fa), r1 = fc * rcp_approx(q);
  const float m = 1e-4f * (ba + mu + md) + 1e-7f;
  const float tmargin = __fmaf_rn(1e-5f, ba, 1e-6f);
  auto horner = [](float r, const float c[4]) {
    return __fmaf_rn(r, __fmaf_rn(r, __fmaf_rn(r, c[3], c[2]), c[1]), c[0]);
  };
  auto root_ok = [&](float r) {
    const bool in = r >= dc.scr_lo && r <= dc.scr_hi;
    const float p = horner(r, a), pu = horner(r, up), pd = horner(r, dn);
    const bool strong = fabsf(p) + tmargin >= dc.scr_thr;
    const bool past = p > 0.0f ? ((pu >= p + m) | (pd >= p + m)) : ((pu <= p - m) | (pd <= p - m));
    return (in & strong & !past) | (!in & !isfinite(r));
  };
  const bool any = root_ok(r0) | root_ok(r1);
  const bool undecided = !(fd > de) | !(fabsf(q) > 1e-30f);  // near-double root, not finite, q ~ 0
  return (fa == 0.0f) | (!(fd < -de) & (undecided | any));
}

__device__ __forceinline__ bool screen_pixel(const double a[4], const double up[4], const double dn[4],
                                              const DetConst& dc) {
  float af[4], uf[4], df[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    af[i] = float(a[i]);
    uf[i] = float(up[i]);
    df[i] = float(dn[i]);
  }
  return screen_pixel(af, mag_bound(af, dc.scr_hi), uf, nbr_bound(uf, dc.scr_hi), df, nbr_bound(df, dc.scr_hi), dc);
}

// ---------------------------------------------------------------- K1a: blur
// One CTA (NT = 64 or 32 threads) = one Gaussian level of a strip of 2 NT
// output columns of one frame; thread t owns the two adjacent
// columns x0 + 2t, x0 + 2t + 1 and walks them top to bottom over the virtual
// rows v = -R .. h-1+R (rows outside [0,h) are the mirror-reflected rows the
// reference's y pass reads, image.cpp:187-210).
//
// x pass (gather): the strip's base row v sits in shared memory; the thread
// reads its 2R+2 inputs with R+1 16-byte loads and forms both columns' sums
// in the reference's tap order.
//
// y pass (scatter with shared products): output row y is
// (((k_R r[y-R] + k_{R-1} r[y-R+1]) + ...) + k_R r[y+R]) and the taps are
// symmetric bit for bit, so the rounded product k_j r[v] serves both output
// rows v - j and v + j. Each new x-pass row v therefore costs R+1 multiplies
// (not 2R+1): its products are added to the 2R+1 pending output rows
// y = v-R .. v+R, each of which receives its terms in increasing v — exactly
// the reference's add sequence, so every G value is bit-identical. The 2R+1
// accumulators rotate through statically named registers: the row loop is
// unrolled by one period (CH = 2R+1 rows).
//
// Base rows stream into a shared ring with cp.async kBlurAhead rows ahead (no
// registers held): f64 sources straight into the staged layout, u8 frames as
// raw 4-byte words, converted (b / 255, mirrored columns) one row ahead into
// a 2-row f64 ring. Octave >= 1 reads G3 of the previous octave at even
// coordinates directly (downsample_half, image.cpp:147-155).
constexpr int kBlurThreadsMax = 64;                    // 64 (octave 0) or 32 threads (smaller octaves)
constexpr int kBlurCols = 2 * kBlurThreadsMax;
constexpr int kMaxBlurR = 8;                           // launch_octave instantiates radii <= 8
constexpr int kBlurAhead = 6;                          // rows in flight
constexpr int kBlurRaw = kBlurAhead + 1;               // raw ring slots
constexpr int kBlurNS = kBlurCols + 2 * kMaxBlurR;     // staged doubles per row (max radius)
constexpr int kBlurRawBytes = kBlurNS + 16;            // u8 raw row: aligned word superset (16-byte multiple)

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(uint32_t(__cvta_generic_to_shared(smem))), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8b(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(uint32_t(__cvta_generic_to_shared(smem))), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

static_assert(kBlurRawBytes * kBlurRaw % 16 == 0 && kBlurNS % 2 == 0, "16-byte aligned staged rows");
struct BlurSmem {
  union {
    double f64[kBlurRaw][kBlurNS];  // f64 sources: the staged rows themselves
    struct {
      uint8_t raw[kBlurRaw][kBlurRawBytes];
      double conv[2][kBlurNS];
    } u8;
  };
};

template <int R, int LVL, int SRC, int NT, bool UNROLL>
__device__ __forceinline__ void blur_level(const Batch& bt, const DetConst& dc, int f, int o, BlurSmem& S) {
  constexpr int CH = 2 * R + 1, NS = 2 * NT + 2 * R;
  static_assert(NS >= 2 * NT && NS <= 3 * NT && NS <= kBlurNS, "staging layout");
  const int w = bt.ow[o], h = bt.oh[o];
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * 2 * NT;
  const int cx = x0 + 2 * t;
  double* G = bt.pyr + f * bt.frame_doubles + bt.plane_off[o][LVL];
  // Staged column sc = t + k * NT holds image column
  // mirror(x0 - R + sc); the thread's own window is sc = 2t .. 2t + 2R + 1.
  const bool third = t + 2 * NT < NS;
  int mc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) mc[k] = mirror_index(x0 - R + min(t + k * NT, NS - 1), w);
  auto src_row = [&](int r) { return min(max(mirror_near(r - R, h), 0), h - 1); };  // rows past h-1+R are never stored
  // ---- row sources
  const uint8_t* s8 = nullptr;
  const double* sf = nullptr;
  long long rstride;
  int lo = 0, nwords = 0;
  if constexpr (SRC == 0 || SRC == 3) {
    s8 = bt.pix8 + f * bt.frame_bytes8;
    rstride = bt.stride8;
    // Bytes [lo, lo + 4 * nwords) cover every mirrored column of the strip.
    const int clo = max(0, x0 - R), chi = min(w - 1, x0 + NS - 1 - R);
    lo = clo & ~3;
    nwords = (chi - lo) / 4 + 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) mc[k] -= lo;
  } else if constexpr (SRC == 1) {
    sf = bt.pixf + (long long)f * bt.W * bt.H;
    rstride = bt.W;
  } else {
    sf = bt.pyr + f * bt.frame_doubles + bt.plane_off[o - 1][3];
    rstride = 2LL * bt.ow[o - 1];
#pragma unroll
    for (int k = 0; k < 3; ++k) mc[k] *= 2;
  }
  auto issue = [&](int r, int slot) {  // base row of virtual row r - R into raw slot r % kBlurRaw
    const long long ro = (long long)src_row(r) * rstride;
    if constexpr (SRC == 0) {
      if (t < nwords) cp_async4(S.u8.raw[slot] + 4 * t, s8 + ro + lo + 4 * t);
    } else if constexpr (SRC == 3) {  // unaligned rows: synchronous byte copies
      for (int b = t; b < 4 * nwords; b += NT)
        if (lo + b < w) S.u8.raw[slot][b] = s8[ro + lo + b];
    } else {
      double* dst = S.f64[slot];
      cp_async8b(dst + t, sf + ro + mc[0]);
      cp_async8b(dst + t + NT, sf + ro + mc[1]);
      if (third) cp_async8b(dst + t + 2 * NT, sf + ro + mc[2]);
    }
    cp_commit();
  };
  auto convert = [&](int r, int slot) {  // u8: raw row r -> f64 ring slot r & 1 (image.cpp:79-87: raw * (1.0 / 255.0))
    if constexpr (SRC == 0 || SRC == 3) {
      const uint8_t* rw = S.u8.raw[slot];
      double* d = S.u8.conv[r & 1];
      d[t] = rw[mc[0]] * (1.0 / 255.0);
      d[t + NT] = rw[mc[1]] * (1.0 / 255.0);
      if (third) d[t + 2 * NT] = rw[mc[2]] * (1.0 / 255.0);
    }
  };
  // Prologue: rows 0 .. kBlurAhead-1 in flight; u8 converts row 0.
#pragma unroll
  for (int r = 0; r < kBlurAhead; ++r) issue(r, r);
  if constexpr (SRC == 0 || SRC == 3) {
    cp_wait<kBlurAhead - 1>();
    __syncthreads();
    convert(0, 0);
  }
  auto next = [](int s) { return s + 1 == kBlurRaw ? 0 : s + 1; };
  int rs = 0, is = kBlurAhead;  // raw slots of rows r and r + kBlurAhead
  const double* tp = dc.taps[LVL] + R;  // tp[j] = tp[-j]: tap of offset j
  double acc0[CH], acc1[CH];
#pragma unroll
  for (int s = 0; s < CH; ++s) acc0[s] = acc1[s] = 0.0;
  const bool col0 = cx < w, col1 = cx + 1 < w;
  double* gcol = G + cx;
  const bool vec = col1 && (w & 1) == 0 && (reinterpret_cast<uintptr_t>(gcol) & 15) == 0;
  const int nrows = h + 2 * R;  // virtual rows r = 0 .. nrows-1 (v = r - R)
  // The reference's sums start from 0.0 (acc = 0.0; acc += ...), ours from
  // the first product: the values are the same except that an all -0.0 sum
  // stays -0.0 here and is +0.0 there. Only f64 base rows can hold -0.0 (a
  // GrayImage of -0.0 pixels passes validate()); their G values take one
  // + 0.0, which maps -0.0 to +0.0 and leaves every other value alone, so the
  // pyramid never holds -0.0 — as the reference's never does.
  auto canon = [](double v) {
    if constexpr (SRC == 1) return __dadd_rn(v, 0.0);
    else return v;
  };
  if constexpr (!UNROLL) {
    // Rolled row loop (a few hundred instructions, resident in the
    // instruction cache): acc[s] holds output row v - R + s; row v adds
    // k_|R-s| x[v] to each pending row, starts row v + R, completes row v - R,
    // and the accumulators shift down by one (register moves, no FP64).
#pragma unroll 1
    for (int r = 0; r < nrows; ++r) {
      const double* row;
      if constexpr (SRC == 0 || SRC == 3) {
        cp_wait<kBlurAhead - 2>();
        __syncthreads();
        issue(r + kBlurAhead, is);
        convert(r + 1, next(rs));
        row = S.u8.conv[r & 1];
      } else {
        cp_wait<kBlurAhead - 1>();
        __syncthreads();
        issue(r + kBlurAhead, is);
        row = S.f64[rs];
      }
      double b[2 * R + 2];
      const double2* sp = reinterpret_cast<const double2*>(row + 2 * t);
#pragma unroll
      for (int k = 0; k <= R; ++k) {
        const double2 q = sp[k];
        b[2 * k] = q.x;
        b[2 * k + 1] = q.y;
      }
      double xa = tp[R] * b[0], xb = tp[R] * b[1];
#pragma unroll
      for (int j = 1; j <= 2 * R; ++j) {
        const double k = tp[j < R ? R - j : j - R];
        xa = xa + k * b[j];
        xb = xb + k * b[j + 1];
      }
      double pa[R + 1], pb[R + 1];
#pragma unroll
      for (int j = 0; j <= R; ++j) {
        pa[j] = tp[j] * xa;
        pb[j] = tp[j] * xb;
      }
#pragma unroll
      for (int s2 = 0; s2 < 2 * R; ++s2) {
        const int j = s2 < R ? R - s2 : s2 - R;
        acc0[s2] = acc0[s2] + pa[j];
        acc1[s2] = acc1[s2] + pb[j];
      }
      acc0[2 * R] = pa[R];  // first term of output row v + R
      acc1[2 * R] = pb[R];
      rs = next(rs);
      is = next(is);
      const int y = r - 2 * R;  // complete: its last term (row y + R) was just added
      if (y >= 0 && y < h) {
        double* gp = gcol + (long long)y * w;
        if (vec) {
          *reinterpret_cast<double2*>(gp) = make_double2(canon(acc0[0]), canon(acc1[0]));
        } else {
          if (col0) gp[0] = canon(acc0[0]);
          if (col1) gp[1] = canon(acc1[0]);
        }
      }
#pragma unroll
      for (int s2 = 0; s2 < 2 * R; ++s2) {
        acc0[s2] = acc0[s2 + 1];
        acc1[s2] = acc1[s2 + 1];
      }
    }
    cp_wait<0>();
    return;
  }
  for (int rc = 0; rc < nrows; rc += CH) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int r = rc + i;
      const double* row;
      if constexpr (SRC == 0 || SRC == 3) {
        cp_wait<kBlurAhead - 2>();  // raw row r + 1 landed (own copies)
        __syncthreads();            // ... everyone's; row r converted; slots of rows <= r - 1 free
        issue(r + kBlurAhead, is);
        convert(r + 1, next(rs));
        row = S.u8.conv[r & 1];
      } else {
        cp_wait<kBlurAhead - 1>();  // row r landed (own copies)
        __syncthreads();            // ... everyone's; slot of row r - 1 free
        issue(r + kBlurAhead, is);
        row = S.f64[rs];
      }
      double b[2 * R + 2];
      const double2* sp = reinterpret_cast<const double2*>(row + 2 * t);
#pragma unroll
      for (int k = 0; k <= R; ++k) {
        const double2 q = sp[k];
        b[2 * k] = q.x;
        b[2 * k + 1] = q.y;
      }
      double xa = tp[R] * b[0], xb = tp[R] * b[1];
#pragma unroll
      for (int j = 1; j <= 2 * R; ++j) {
        const double k = tp[j < R ? R - j : j - R];
        xa = xa + k * b[j];
        xb = xb + k * b[j + 1];
      }
#pragma unroll
      for (int j = 0; j <= R; ++j) {
        const double pa = tp[j] * xa, pb = tp[j] * xb;
        // output rows y = v - j and v + j; slot of output row y is (y + R) mod CH
        const int sm = ((i - j) % CH + CH) % CH, sp_ = (i + j) % CH;
        acc0[sm] = acc0[sm] + pa;
        acc1[sm] = acc1[sm] + pb;
        if (j == R) {
          acc0[sp_] = pa;  // first term of output row v + R
          acc1[sp_] = pb;
        } else if (j > 0) {
          acc0[sp_] = acc0[sp_] + pa;
          acc1[sp_] = acc1[sp_] + pb;
        }
      }
      rs = next(rs);
      is = next(is);
      const int y = r - 2 * R;  // complete: its last term (row y + R) was just added
      if (y >= 0 && y < h) {
        const int so = ((i - R) % CH + CH) % CH;
        double* gp = gcol + (long long)y * w;
        if (vec) {
          *reinterpret_cast<double2*>(gp) = make_double2(canon(acc0[so]), canon(acc1[so]));
        } else {
          if (col0) gp[0] = canon(acc0[so]);
          if (col1) gp[1] = canon(acc1[so]);
        }
      }
    }
  }
  cp_wait<0>();
}

template <int R0, int R1, int R2, int R3, int SRC, int NT, bool UNROLL>
__global__ void __launch_bounds__(NT) k_blur(Batch bt, DetConst dc, int o) {
  __shared__ __align__(16) BlurSmem S;
  // Level-major grid (blockIdx.z = level): the CTAs resident on an SM at any
  // moment mostly share one level's loop in the instruction cache.
  const int f = blockIdx.y;
  switch (blockIdx.z) {
    case 0: blur_level<R0, 0, SRC, NT, UNROLL>(bt, dc, f, o, S); break;
    case 1: blur_level<R1, 1, SRC, NT, UNROLL>(bt, dc, f, o, S); break;
    case 2: blur_level<R2, 2, SRC, NT, UNROLL>(bt, dc, f, o, S); break;
    default: blur_level<R3, 3, SRC, NT, UNROLL>(bt, dc, f, o, S); break;
  }
}

// ---------------------------------------------------------------- K1b: extrema
// One CTA = a kDetW x kDetH tile of the detection window [m, w-m) x [m, h-m)
// of one octave of one frame. G of the tile plus a 2-pixel halo is read back
// (HBM/L2), sigma^2-Laplacians and alpha = beta * L are formed for the tile
// plus a 1-pixel halo in shared memory, every pixel is screened (FP32) and the
// plausible ones run the exact FP64 test + refinement from a dense queue.
constexpr int kDetW = 64, kDetH = 16, kDetThreads = 256;
constexpr int kGW = kDetW + 4, kGH = kDetH + 4;  // G region
constexpr int kAW = kDetW + 2, kAH = kDetH + 2;  // alpha region

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(kDetThreads, 2)
    k_detect(Batch bt, DetConst dc, int o, const __grid_constant__ CUtensorMap tmap, int use_tma) {
  extern __shared__ __align__(128) double dsm[];
  double* Gt = dsm;                      // [4][kGH][kGW]
  double* At = Gt + 4 * kGH * kGW;       // [kAH][4][kAW]
  __shared__ int q_count;
  __shared__ uint16_t queue[kDetW * kDetH];
  __shared__ __align__(8) uint64_t tma_bar;
  const int f = blockIdx.z, tid = threadIdx.x;
  const int w = bt.ow[o], h = bt.oh[o], m = dc.margin;
  const int tx0 = m + blockIdx.x * kDetW, ty0 = m + blockIdx.y * kDetH;
  const double* pyr = bt.pyr + f * bt.frame_doubles;
  if (tid == 0) q_count = 0;
  if (use_tma) {
    // One 4-D TMA box (68 x 20 x 4 levels x 1 frame) brings the tile's G
    // levels into shared memory; rows/columns past the image arrive as zeros
    // and only feed alpha outside the detection window.
    if (tid == 0) {
      const uint32_t bar = smem_u32(&tma_bar);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(sizeof(double) * 4 * kGH * kGW)) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
          ::"r"(smem_u32(Gt)), "l"(&tmap), "r"(tx0 - 2), "r"(ty0 - 2), "r"(0), "r"(f), "r"(bar)
          : "memory");
    }
    __syncthreads();  // barrier initialised before anyone polls it
    const uint32_t bar = smem_u32(&tma_bar);
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done) : "r"(bar) : "memory");
    }
  } else {
    constexpr int N = 4 * kGH * kGW, PER = (N + kDetThreads - 1) / kDetThreads;
    double v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {  // all loads in flight before the first store
      const int q = tid + k * kDetThreads;
      if (q < N) {
        const int lv = q / (kGH * kGW), r = (q / kGW) % kGH, cc = q % kGW;
        const int y = min(ty0 - 2 + r, h - 1), x = min(tx0 - 2 + cc, w - 1);
        v[k] = __ldg(pyr + bt.plane_off[o][lv] + (long long)y * w + x);
      }
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int q = tid + k * kDetThreads;
      if (q < N) Gt[q] = v[k];
    }
    __syncthreads();
  }
  // Laplacian x sigma^2 then alpha, for the tile + 1 halo (scale_space.cpp:148-170);
  // a fixed, unrolled set of positions per thread so loads and the four
  // independent alpha sums of several positions overlap.
  {
    constexpr int N = kAH * kAW, PER = (N + kDetThreads - 1) / kDetThreads;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int q = tid + k * kDetThreads;
      if (q < N) {
        const int r = q / kAW, cc = q - r * kAW;
        double L[4];
#pragma unroll
        for (int lv = 0; lv < 4; ++lv) {
          const double* g = Gt + (lv * kGH + r + 1) * kGW + cc + 1;
          const double lap = fma(-4.0, g[0], g[-kGW] + g[kGW] + g[-1] + g[1]);  // 4c is exact: == s - 4c
          L[lv] = dc.s2[lv] * lap;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double sum = dc.beta[i][0] * L[0];
          sum = sum + dc.beta[i][1] * L[1];
          sum = sum + dc.beta[i][2] * L[2];
          sum = sum + dc.beta[i][3] * L[3];
          At[(r * 4 + i) * kAW + cc] = sum;
        }
      }
    }
  }
  __syncthreads();
  static_assert((kDetW * kDetH) % kDetThreads == 0, "uniform screen loop");
  const int lane = tid & 31;
  for (int q = tid; q < kDetW * kDetH; q += kDetThreads) {
    const int r = q / kDetW, cc = q % kDetW;
    const int yd = ty0 + r, xd = tx0 + cc;
    bool push = false;
    if (yd < h - m && xd < w - m) {
      const double* a = At + ((r + 1) * 4) * kAW + cc + 1;
      const double av[4] = {a[0], a[kAW], a[2 * kAW], a[3 * kAW]};
      const double* au = a - 4 * kAW;
      const double* ad = a + 4 * kAW;
      const double uv[4] = {au[0], au[kAW], au[2 * kAW], au[3 * kAW]};
      const double dv[4] = {ad[0], ad[kAW], ad[2 * kAW], ad[3 * kAW]};
      push = !dc.screen || screen_pixel(av, uv, dv, dc);
    }
    // One shared-memory atomic per warp (queue order is irrelevant: the merge
    // kernel restores raster order from the bitmap).
    const unsigned bal = __ballot_sync(0xffffffffu, push);
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(&q_count, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (push) queue[base + __popc(bal & ((1u << lane) - 1u))] = uint16_t(q);
  }
  __syncthreads();
  const int nq = q_count;
  const double oct_scale = ldexp(1.0, o);
  for (int qi = tid; qi < nq; qi += kDetThreads) {
    const int q = queue[qi];
    const int r = q / kDetW, cc = q % kDetW;
    exact_detect(bt, dc, f, o, w, ty0 + r, tx0 + cc, At + (r * 4) * kAW, At + ((r + 1) * 4) * kAW,
                 At + ((r + 2) * 4) * kAW, kAW, cc + 1, oct_scale);
  }
}

// ------------------------------------------------------- K1b v2: extrema walk
// One WARP = a strip of 30 detection-window columns (lanes 1..30; lanes 0 and
// 31 are the 1-column halo) walking a segment of ~kSegTarget window rows top to
// bottom. Per row the warp reads the four G levels of the next row once
// (coalesced; the edge lanes also read their outer neighbour), slides the
// Laplacian's up/centre/down rows in registers, takes left/right from a
// per-warp row buffer, forms sigma^2 L and alpha = beta * L (the reference's
// order) and parks alpha in a per-warp ring of kRing rows in shared memory.
// Each window pixel is screened (FP32) as soon as its alpha exists; plausible
// pixels are queued and the queue is drained in full-warp passes by the exact
// FP64 test (exact_detect, reading the 3x3 alpha neighbourhood from the ring)
// before the ring can overwrite any row a queued pixel needs.
constexpr int kStripCols = 30, kSegTarget = 96, kRing = 6, kDetWarps = 3, kPrefetch = 2, kGRows = kPrefetch + 2;  // kDetWarps: max warps per CTA
struct alignas(128) DetWarpSmem {
  union {
    double grow[kGRows][4][34];   // cp.async path: G rows in flight [row % kGRows][level][1 + lane], edges at 0 and 33
    double gpair[2][4][2][34];    // TMA path: row pairs [pair % 2][level][row of pair][1 + lane] (one 4-D box each)
  };
  double ring[kRing][4][32];   // alpha rows: [row % kRing][coefficient][lane]
  uint64_t bar[2];             // TMA path: one mbarrier per pair slot
  uint16_t queue[128];         // ((row - y0 + 2) << 5) | lane
};
static_assert(sizeof(double) * 4 * 2 * 34 % 128 == 0, "TMA pair slots stay 128-byte aligned");

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  }
}

// TMA = true: G rows arrive as row pairs, one 4-D TMA box (34 columns x 2 rows
// x 4 levels) per pair issued by lane 0 into a 2-slot ring with an mbarrier
// per slot — one instruction per pair instead of 8-16 cp.async per lane and
// row (needs even widths: 16-byte row strides; the walk map is built in
// plan()). Columns of the box past the image arrive as zeros; they only feed
// alpha outside the detection window, which is never screened or used.
template <bool TMA>
__global__ void __maxnreg__(96) k_detect_walk(Batch bt, DetConst dc, int o, int seg_rows,
                                              const __grid_constant__ CUtensorMap wmap) {
  extern __shared__ __align__(128) uint8_t det_smem[];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DetWarpSmem& S = reinterpret_cast<DetWarpSmem*>(det_smem)[wi];
  const int f = blockIdx.z;
  const int w = bt.ow[o], h = bt.oh[o], m = dc.margin;
  const int xs0 = m + (blockIdx.x * int(blockDim.x >> 5) + wi) * kStripCols;  // first window column of the strip
  const int y0 = m + blockIdx.y * seg_rows, y1 = min(h - m, y0 + seg_rows);
  if (xs0 >= w - m || y0 >= y1) return;  // warp-uniform
  const int x = xs0 - 1 + lane;
  const bool out_col = lane >= 1 && lane <= kStripCols && x < w - m;
  const int xc = min(x, w - 1);
  const bool edge = lane == 0 || lane == 31;
  const int xe = lane == 0 ? x - 1 : min(x + 1, w - 1);  // edge lanes' outer neighbour
  const int eslot = lane == 0 ? 0 : 33;
  // G rows stream into a kGRows-row shared ring with cp.async, kPrefetch
  // rows ahead of the row being differentiated.
  const double* gp[4];
  const long long eoff = (long long)(xe - xc);
  {
    const double* base = bt.pyr + f * bt.frame_doubles + (long long)(y0 - 2) * w;
#pragma unroll
    for (int k = 0; k < 4; ++k) gp[k] = base + bt.plane_off[o][k] + xc;
  }
  int next_row = y0 - 2;
  // TMA path: pair p holds rows y0 - 2 + 2p, y0 - 1 + 2p in slot p & 1 (phase p >> 1).
  const int npairs = (y1 - y0 + 5) >> 1;  // rows y0 - 2 .. y1 + 1
  auto issue_pair = [&](int p) {
    if (lane == 0 && p < npairs) {
      const uint32_t bar = smem_u32(&S.bar[p & 1]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(sizeof(S.gpair[0])))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
          ::"r"(smem_u32(&S.gpair[p & 1][0][0][0])), "l"(&wmap), "r"(xs0 - 2), "r"(y0 - 2 + 2 * p), "r"(0), "r"(f),
          "r"(bar)
          : "memory");
    }
  };
  auto wait_pair = [&](int p) { mbar_wait(smem_u32(&S.bar[p & 1]), uint32_t((p >> 1) & 1)); };
  auto issue = [&]() {  // next G row into its slot (or an empty group past the segment)
    if (next_row <= y1 + 1) {
      double(*dst)[34] = S.grow[unsigned(next_row) % kGRows];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cp_async8(&dst[k][lane + 1], gp[k]);
        if (edge) cp_async8(&dst[k][eslot], gp[k] + eoff);
        gp[k] += w;
      }
    }
    ++next_row;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if constexpr (TMA) {
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.bar[0])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.bar[1])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    issue_pair(0);
    issue_pair(1);
  } else {
#pragma unroll
    for (int i = 0; i < kPrefetch + 2; ++i) issue();  // rows y0 - 2 .. y0 + kPrefetch - 1
  }
  const double oct_scale = ldexp(1.0, o);
  // Float copies of the lane's own alpha (the screen's inputs, each alpha
  // converted once): the previous row (screened one row late) with its
  // magnitude and neighbour bounds, and the row before it with its neighbour
  // bound. Registers, not shared memory: every lane reads only its own column.
  float apf[4] = {0.f, 0.f, 0.f, 0.f}, a2f[4] = {0.f, 0.f, 0.f, 0.f};
  float bp = 0.f, mp = 0.f, m2 = 0.f;
  int qn = 0;
  auto drain = [&]() {
    for (int qi = lane; qi - lane < qn; qi += 32) {
      if (qi < qn) {
        const int ent = S.queue[qi];
        const int t = ent & 31, yd = (ent >> 5) + y0 - 2;
        exact_detect(bt, dc, f, o, w, yd, xs0 - 1 + t, &S.ring[(yd - 1) % kRing][0][0], &S.ring[yd % kRing][0][0],
                     &S.ring[(yd + 1) % kRing][0][0], 32, t, oct_scale);
      }
    }
    qn = 0;
    __syncwarp();
  };
  const int T = y1 - y0 + 2;  // alpha rows y0 - 1 .. y1
  // sigma^2-normalised Laplacian of row ra (image.cpp:220-238,
  // scale_space.cpp:148-151), then alpha = beta * L in column order.
  // Row r of level k, slot column c (0..33): the cp.async ring, or the TMA
  // pair ring (rows y0 - 2 + 2p and y0 - 1 + 2p in slot p & 1).
  auto grow_at = [&](int r, int k) -> const double* {
    if constexpr (TMA) {
      const int d = r - (y0 - 2);
      return &S.gpair[(d >> 1) & 1][k][d & 1][0];
    } else {
      return &S.grow[unsigned(r) % kGRows][k][0];
    }
  };
  auto alpha_row = [&](int ra, double an[4]) {
    double L[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double* rU = grow_at(ra - 1, k);
      const double* rC = grow_at(ra, k);
      const double* rD = grow_at(ra + 1, k);
      // (((up + down) + left) + right) - 4c with one rounding for the last
      // step: 4c is exact, so the fused multiply-add is RN(s - 4c) itself.
      const double lap = fma(-4.0, rC[lane + 1], rU[lane + 1] + rD[lane + 1] + rC[lane] + rC[lane + 2]);
      L[k] = dc.s2[k] * lap;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double sum = dc.beta[i][0] * L[0];
      sum = sum + dc.beta[i][1] * L[1];
      sum = sum + dc.beta[i][2] * L[2];
      sum = sum + dc.beta[i][3] * L[3];
      an[i] = sum;
    }
  };
  auto screen_row = [&](int rs, const float a[4], float ba, const float up[4], float mu, const float dn[4],
                        float md) {  // 3x3 neighbourhood complete
    if (rs >= y0 && rs < y1) {
      const bool push = out_col & (!dc.screen | screen_pixel_flat(a, ba, up, mu, dn, md, dc));
      const unsigned bal = __ballot_sync(0xffffffffu, push);
      if (push) S.queue[qn + __popc(bal & ((1u << lane) - 1u))] = uint16_t(((rs - y0 + 2) << 5) | lane);
      qn += __popc(bal);
    }
  };
  for (int t0 = 0; t0 < T; t0 += 4) {
    // Two alpha rows per step (independent FP64 chains side by side).
#pragma unroll
    for (int ph = 0; ph < 4; ph += 2) {
      const int t = t0 + ph;
      if (t >= T) break;
      const int ra = y0 - 1 + t;
      // Rows ra - 1 .. ra + 2 must have landed: rows up to ra + kPrefetch
      // may still be in flight.
      if constexpr (TMA) {
        wait_pair(t >> 1);
        wait_pair((t >> 1) + 1);
      } else {
        asm volatile("cp.async.wait_group %0;" ::"n"(kPrefetch - 2) : "memory");
        __syncwarp();
      }
      double a0[4], a1[4];
      alpha_row(ra, a0);
      alpha_row(ra + 1, a1);
      const bool second = t + 1 < T;
      const float a0f[4] = {float(a0[0]), float(a0[1]), float(a0[2]), float(a0[3])};
      const float a1f[4] = {float(a1[0]), float(a1[1]), float(a1[2]), float(a1[3])};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        S.ring[unsigned(ra) % kRing][i][lane] = a0[i];
        if (second) S.ring[unsigned(ra + 1) % kRing][i][lane] = a1[i];
      }
      const float b0 = mag_bound(a0f, dc.scr_hi), m0 = nbr_bound(a0f, dc.scr_hi);
      const float b1 = mag_bound(a1f, dc.scr_hi), m1 = nbr_bound(a1f, dc.scr_hi);
      __syncwarp();
      if constexpr (TMA) {
        issue_pair((t >> 1) + 2);  // into the slot of pair t/2 (rows ra - 1, ra), read by every lane above
      } else {
        issue();  // rows ra + kPrefetch + 1, ra + kPrefetch + 2 into the slots of rows ra - 1, ra
        issue();
      }
      screen_row(ra - 1, apf, bp, a2f, m2, a0f, m0);
      if (second) screen_row(ra, a0f, b0, apf, mp, a1f, m1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a2f[i] = a0f[i];
        apf[i] = a1f[i];
      }
      m2 = m0;
      bp = b1;
      mp = m1;
    }
    __syncwarp();
    // Every queued pixel (rows <= the last alpha row - 1) has its
    // neighbourhood in the ring; the ring keeps the 6 rows they need.
    if (qn > 0) drain();
  }
  if constexpr (!TMA) asm volatile("cp.async.wait_group 0;" ::: "memory");
}

constexpr size_t kDetSmem = sizeof(double) * (4 * kGH * kGW + kAH * 4 * kAW);
static_assert((kGW * sizeof(double)) % 16 == 0, "TMA box rows must be 16-byte multiples");

template <int R0, int R1, int R2, int R3>
cudaError_t launch_octave_variant(const Batch& bt, const DetConst& dc, int o, int src, cudaStream_t st) {
  // 128-column strips at octave 0 (640 = 5 strips), 64-column strips (one
  // warp) above, where the planes are narrow.
  const int nt = src == 2 ? 32 : 64;
  dim3 grid((bt.ow[o] + 2 * nt - 1) / (2 * nt), bt.nframes, 4);
  const bool aligned8 = ((reinterpret_cast<uintptr_t>(bt.pix8) | uintptr_t(bt.stride8) | uintptr_t(bt.frame_bytes8)) & 3) == 0;
  const int s = src == 0 ? (aligned8 ? 0 : 3) : src;
#define CDVZ_BLUR(S, N)                                                  \
  do {                                                                   \
    if (dc.blur_unrolled) k_blur<R0, R1, R2, R3, S, N, true><<<grid, N, 0, st>>>(bt, dc, o);   \
    else k_blur<R0, R1, R2, R3, S, N, false><<<grid, N, 0, st>>>(bt, dc, o);                   \
  } while (0)
  if (s == 0) CDVZ_BLUR(0, 64);       // octave 0: u8 frames
  else if (s == 3) CDVZ_BLUR(3, 64);  // octave 0: u8 frames, unaligned rows
  else if (s == 1) CDVZ_BLUR(1, 64);  // octave 0: resized f64 frames
  else CDVZ_BLUR(2, 32);              // octaves >= 1: G3 of the previous octave
#undef CDVZ_BLUR
  return cudaGetLastError();
}

cudaError_t launch_detect(const Batch& bt, const DetConst& dc, int o, const CUtensorMap* tmap, const CUtensorMap* wmap,
                          cudaStream_t st) {
  const int ww = bt.ow[o] - 2 * dc.margin, hh = bt.oh[o] - 2 * dc.margin;
  if (ww <= 0 || hh <= 0) return cudaSuccess;  // detect_extrema: empty window (scale_space.cpp:159)
  static size_t configured[kMaxDevices] = {};
  cudaError_t e0 = once_per_device(configured, 1, [&] {
    return cudaFuncSetAttribute(k_detect, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDetSmem));
  });
  if (e0 != cudaSuccess) return e0;
  if (dc.walk) {
    // Balanced row segments of about kSegTarget rows (each costs 4 extra G
    // rows and 2 extra alpha rows at its ends).
    const int strips = (ww + kStripCols - 1) / kStripCols;
    const int nseg = (hh + kSegTarget - 1) / kSegTarget, seg_rows = (hh + nseg - 1) / nseg;
    // One warp (strip) per CTA: no idle warps at any width, and the finest
    // granularity for the register-limited occupancy (measured 1-2% faster
    // than 2- or 3-warp CTAs).
    const int nw = 1;
    dim3 grid((strips + nw - 1) / nw, nseg, bt.nframes);
    constexpr int smem = int(sizeof(DetWarpSmem)) * kDetWarps;
    static size_t walk_configured[kMaxDevices] = {};
    cudaError_t e = once_per_device(walk_configured, 1, [&] {
      for (auto fn : {k_detect_walk<true>, k_detect_walk<false>}) {
        cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (r != cudaSuccess) return r;
      }
      return cudaSuccess;
    });
    if (e != cudaSuccess) return e;
    if (wmap) {
      k_detect_walk<true><<<grid, 32 * nw, int(sizeof(DetWarpSmem)) * nw, st>>>(bt, dc, o, seg_rows, *wmap);
    } else {
      CUtensorMap none{};
      k_detect_walk<false><<<grid, 32 * nw, int(sizeof(DetWarpSmem)) * nw, st>>>(bt, dc, o, seg_rows, none);
    }
    return cudaGetLastError();
  }
  dim3 grid((ww + kDetW - 1) / kDetW, (hh + kDetH - 1) / kDetH, bt.nframes);
  CUtensorMap none{};
  k_detect<<<grid, kDetThreads, kDetSmem, st>>>(bt, dc, o, tmap ? *tmap : none, tmap ? 1 : 0);
  return cudaGetLastError();
}

// Radii of the default detector (sigma_k = 1.4 * 2^(k/4): taps 11/11/13/17)
// get an exact-fit instantiation; any config with radii <= 8 runs on the
// padded variant (zero taps add exact zeros, so results are unchanged).
cudaError_t launch_octave(const Batch& bt, const DetConst& dc, int o, int src, cudaStream_t st) {
  if (dc.radius[0] == 5 && dc.radius[1] == 5 && dc.radius[2] == 6 && dc.radius[3] == 8)
    return launch_octave_variant<5, 5, 6, 8>(bt, dc, o, src, st);
  return launch_octave_variant<8, 8, 8, 8>(bt, dc, o, src, st);
}

}  // namespace cdvz_gpu
