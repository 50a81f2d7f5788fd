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

template <int R0, int R1, int R2, int R3, int SRC>
__global__ void __launch_bounds__(256, 1) k_octave(Batch bt, DetConst dc, int o, int S) {
  constexpr int RM = R3;
  constexpr int D0 = RM + R0 + 1, D1 = RM + R1 + 1, D2 = RM + R2 + 1, D3 = RM + R3 + 1;
  extern __shared__ double smem[];
  const int T = blockDim.x;
  const int nbrow = S + 4 + 2 * RM;
  double* brow = smem;
  double* Gs = brow + nbrow;  // [3 rows][4 levels][T]
  double* As = Gs + 12 * T;   // [3 rows][4 coefs][T]

  const int f = blockIdx.y, t = threadIdx.x;
  const int w = bt.ow[o], h = bt.oh[o];
  const int x0 = blockIdx.x * S;
  const int cx = x0 - 2 + t;
  const bool active = t < S + 4;
  double* pyr = bt.pyr + f * bt.frame_doubles;
  double* G0 = pyr + bt.plane_off[o][0];
  double* G1 = pyr + bt.plane_off[o][1];
  double* G2 = pyr + bt.plane_off[o][2];
  double* G3 = pyr + bt.plane_off[o][3];
  const bool store_col = t >= 2 && t < S + 2 && cx < w;
  const int m = dc.margin;
  const bool det_col = t >= 2 && t < S + 2 && cx >= m && cx < w - m;
  const bool lap_col = t >= 1 && t <= S + 2;
  const double oct_scale = ldexp(1.0, o);

  double r0[D0], r1[D1], r2[D2], r3[D3];
#pragma unroll
  for (int i = 0; i < D0; ++i) r0[i] = 0.0;
#pragma unroll
  for (int i = 0; i < D1; ++i) r1[i] = 0.0;
#pragma unroll
  for (int i = 0; i < D2; ++i) r2[i] = 0.0;
#pragma unroll
  for (int i = 0; i < D3; ++i) r3[i] = 0.0;

  for (int v = -RM; v <= h - 1 + RM; ++v) {
    // 1. stage base row mirror(v), columns mirror(x0-2-RM+i)
    {
      const int ry = mirror_index(v, h);
      for (int i = t; i < nbrow; i += T) brow[i] = load_base<SRC>(bt, f, o, ry, mirror_index(x0 - 2 - RM + i, w));
    }
    __syncthreads();

    // 2. x pass (image.cpp:187-196): acc over j = -r..r; 0.0 + x == x exactly
    //    for the non-negative products, so the first tap seeds the sum.
    if (active) {
      const double* bp = brow + t + RM;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int j = -RM; j <= RM; ++j) {
        const double val = bp[j];
        if (j >= -R0 && j <= R0) a0 = (j == -R0) ? dc.taps[0][0] * val : a0 + dc.taps[0][j + R0] * val;
        if (j >= -R1 && j <= R1) a1 = (j == -R1) ? dc.taps[1][0] * val : a1 + dc.taps[1][j + R1] * val;
        if (j >= -R2 && j <= R2) a2 = (j == -R2) ? dc.taps[2][0] * val : a2 + dc.taps[2][j + R2] * val;
        a3 = (j == -R3) ? dc.taps[3][0] * val : a3 + dc.taps[3][j + R3] * val;
      }
#pragma unroll
      for (int i = 0; i < D0 - 1; ++i) r0[i] = r0[i + 1];
#pragma unroll
      for (int i = 0; i < D1 - 1; ++i) r1[i] = r1[i + 1];
#pragma unroll
      for (int i = 0; i < D2 - 1; ++i) r2[i] = r2[i + 1];
#pragma unroll
      for (int i = 0; i < D3 - 1; ++i) r3[i] = r3[i + 1];
      r0[D0 - 1] = a0;
      r1[D1 - 1] = a1;
      r2[D2 - 1] = a2;
      r3[D3 - 1] = a3;
    }

    // 3. y pass (image.cpp:201-210) for output row y = v - RM.
    const int y = v - RM;
    if (y >= 0 && active) {
      double g0 = dc.taps[0][0] * r0[0], g1 = dc.taps[1][0] * r1[0], g2 = dc.taps[2][0] * r2[0], g3 = dc.taps[3][0] * r3[0];
#pragma unroll
      for (int i = 1; i <= 2 * R0; ++i) g0 = g0 + dc.taps[0][i] * r0[i];
#pragma unroll
      for (int i = 1; i <= 2 * R1; ++i) g1 = g1 + dc.taps[1][i] * r1[i];
#pragma unroll
      for (int i = 1; i <= 2 * R2; ++i) g2 = g2 + dc.taps[2][i] * r2[i];
#pragma unroll
      for (int i = 1; i <= 2 * R3; ++i) g3 = g3 + dc.taps[3][i] * r3[i];
      double* gs = Gs + (y % 3) * 4 * T + t;
      gs[0] = g0;
      gs[T] = g1;
      gs[2 * T] = g2;
      gs[3 * T] = g3;
      if (store_col) {
        const long long off = (long long)y * w + cx;
        G0[off] = g0;
        G1[off] = g1;
        G2[off] = g2;
        G3[off] = g3;
      }
    }
    __syncthreads();

    // 4. Laplacian (image.cpp:220-238) times sigma^2 (scale_space.cpp:150),
    //    then alpha = beta * L (scale_space.cpp:165-170), row yl = y - 1.
    const int yl = y - 1;
    if (yl >= 1 && yl <= h - 2 && lap_col) {
      const double* up = Gs + ((yl - 1) % 3) * 4 * T + t;
      const double* mid = Gs + (yl % 3) * 4 * T + t;
      const double* dn = Gs + ((yl + 1) % 3) * 4 * T + t;
      double L[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double lap = up[k * T] + dn[k * T] + mid[k * T - 1] + mid[k * T + 1] - 4.0 * mid[k * T];
        L[k] = dc.s2[k] * lap;
      }
      double* as = As + (yl % 3) * 4 * T + t;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double s = dc.beta[i][0] * L[0];
        s = s + dc.beta[i][1] * L[1];
        s = s + dc.beta[i][2] * L[2];
        s = s + dc.beta[i][3] * L[3];
        as[i * T] = s;
      }
    }
    __syncthreads();

    // 5. extrema (scale_space.cpp:172-205) + refinement (:221-266), row yd.
    const int yd = y - 2;
    if (det_col && yd >= m && yd < h - m) {
      const double* arow[3] = {As + ((yd - 1) % 3) * 4 * T, As + (yd % 3) * 4 * T, As + ((yd + 1) % 3) * 4 * T};
      double a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = arow[1][i * T + t];
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
        // refine_candidates (scale_space.cpp:221-266)
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
    // The next iteration's stage writes brow only; Gs/As rows it overwrites
    // were last read before this iteration's second barrier.
  }
}

// Launch helper: picks strips so a CTA holds <= 256 threads.
struct OctaveLaunch { int strips, S, T; size_t smem; };

inline OctaveLaunch plan_octave(int w, int rm) {
  OctaveLaunch L;
  L.strips = (w + 251) / 252;
  L.S = (w + L.strips - 1) / L.strips;
  L.T = ((L.S + 4 + 31) / 32) * 32;
  L.smem = sizeof(double) * size_t(L.S + 4 + 2 * rm + 24 * L.T);
  return L;
}

template <int R0, int R1, int R2, int R3>
cudaError_t launch_octave_variant(const Batch& bt, const DetConst& dc, int o, int src, cudaStream_t st) {
  const OctaveLaunch L = plan_octave(bt.ow[o], R3);
  dim3 grid(L.strips, bt.nframes);
  cudaError_t e = cudaSuccess;
  if (src == 0) {
    e = cudaFuncSetAttribute(k_octave<R0, R1, R2, R3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.smem));
    k_octave<R0, R1, R2, R3, 0><<<grid, L.T, L.smem, st>>>(bt, dc, o, L.S);
  } else if (src == 1) {
    e = cudaFuncSetAttribute(k_octave<R0, R1, R2, R3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.smem));
    k_octave<R0, R1, R2, R3, 1><<<grid, L.T, L.smem, st>>>(bt, dc, o, L.S);
  } else {
    e = cudaFuncSetAttribute(k_octave<R0, R1, R2, R3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.smem));
    k_octave<R0, R1, R2, R3, 2><<<grid, L.T, L.smem, st>>>(bt, dc, o, L.S);
  }
  if (e != cudaSuccess) return e;
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
