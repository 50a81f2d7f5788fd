// K8-K11 — SCFV global descriptor: PCA 128->32, GMM soft assignment,
// Fisher mean/variance gradients, delta-ranked component selection and sign
// planes; K12 — CDVZ1 container packing with the CRC-32 trailer.
//
// Replaces pca_reduce / posteriors_matrix / softmax_rows / fv_mean_matrix /
// fv_var_matrix / scfv_delta / scfv_encode (proj/src/scfv.cpp:40-253) and
// serialize_scfv / pack_local / serialize_container / crc32
// (proj/src/scfv.cpp:285-298, proj/src/transform_coding.cpp:232-270,
// proj/src/container.cpp:32-58, proj/src/common.cpp:11-35).
//
// Precision: the reference computes in IEEE double; so do these kernels, on
// the FP64 pipe. Dense products are summed over the inner index in ascending
// order and vector reductions follow Eigen's SSE2 packet order, both as the
// oracle restates them, so the SCFV floats agree with the
// oracle up to libm (exp/log) ulps and the emitted bits agree exactly.
#include "common.cuh"
#include "dmath.cuh"

namespace cdvz_gpu {

namespace {

// Eigen SSE2 redux order over a contiguous vector (oracle eigen_sum).
__device__ __forceinline__ double packet_sum_seq(const double* v, int n) {
  if (n < 2) return n ? v[0] : 0.0;
  if (n < 4) {
    double r = v[0] + v[1];
    for (int i = 2; i < n; ++i) r += v[i];
    return r;
  }
  const int e2 = n / 4 * 4, e1 = n / 2 * 2;
  double a0 = v[0], a1 = v[1], b0 = v[2], b1 = v[3];
  for (int i = 4; i < e2; i += 4) {
    a0 += v[i];
    a1 += v[i + 1];
    b0 += v[i + 2];
    b1 += v[i + 3];
  }
  a0 += b0;
  a1 += b1;
  if (e1 > e2) {
    a0 += v[e2];
    a1 += v[e2 + 1];
  }
  double r = a0 + a1;
  for (int i = e1; i < n; ++i) r += v[i];
  return r;
}

}  // namespace

// X[t][r] = sum_j (R[t][j] - mu[j]) * B[r][j], j ascending (scfv.cpp:82-92).
// The basis is staged transposed in shared memory; each thread carries four
// descriptor rows so four independent sums hide the FP64 add latency.
__global__ void __launch_bounds__(128) k_pca(Batch bt, Model md) {
  extern __shared__ __align__(16) double pca_sm[];
  double(*bT)[33] = reinterpret_cast<double(*)[33]>(pca_sm);              // [128][33] basis transposed (lanes read
                                                                           // consecutive r); padded: conflict-free transpose
  double(*cen)[128] = reinterpret_cast<double(*)[128]>(pca_sm + 128 * 33);  // [16][128] centred rows (broadcast reads)
  const int f = blockIdx.y;
  const int n = bt.or_count[f];
  const int tid = threadIdx.x, r = tid & 31, grp = tid >> 5;
  for (int i = tid; i < 32 * 128; i += blockDim.x) bT[i & 127][i >> 7] = md.pca_basis[i];
  for (int t0 = blockIdx.x * 16; t0 < n; t0 += gridDim.x * 16) {
    __syncthreads();
    for (int i = tid; i < 16 * 128; i += blockDim.x) {
      const int tt = t0 + (i >> 7), j = i & 127;
      cen[i >> 7][j] = tt < n ? bt.desc[((long long)f * bt.cap_or + tt) * 128 + j] - md.pca_mean[j] : 0.0;
    }
    __syncthreads();
    double s[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] = cen[grp * 4 + q][0] * bT[0][r];
    for (int j = 1; j < 128; ++j) {
      const double b = bT[j][r];
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] = s[q] + cen[grp * 4 + q][j] * b;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int tt = t0 + grp * 4 + q;
      if (tt < n) bt.x[((long long)f * bt.cap_or + tt) * 32 + r] = s[q];
    }
  }
}

// posteriors_matrix (scfv.cpp:140-164) + softmax_rows (scfv.cpp:40-48).
// One CTA owns a tile of kPM descriptor rows of one frame and all nc
// components. Phase 1 is a register-tiled FP64 product over component tiles
// of kPN: each thread holds a 4 x 4 block of (row, component) pairs and
// accumulates a = sum_j x_j^2 / v_j and b = sum_j x_j m_j / v_j with the
// inner index ascending and every multiply and add separately rounded (the
// reference's arithmetic; the FP64 tensor-core MMA would fuse them, so it is
// not used), then forms log p = -0.5 (a - 2b + c) + log_norm into the gamma
// buffer while tracking the row maxima. Phase 2 exponentiates, sums each row
// in Eigen's SSE2 packet order (four stride-4 chains) and normalises.
__device__ __forceinline__ void cp_async16_post(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(uint32_t(__cvta_generic_to_shared(smem))), "l"(gmem)
               : "memory");
}

constexpr int kPM = 64, kPN = 64;
constexpr int kSoftmaxRowMax = 1024;  // fused per-row softmax: 8 warps x 1024 doubles of the operand tiles
struct PostSmem {
  double xs2[32][kPM];  // x^2, transposed
  double xs[32][kPM];   // x, transposed
  double iv[32][kPN];   // 1 / v, transposed
  double mv[32][kPN];   // m / v, transposed
  double iv2[32][kPN];  // the next component tile (cp.async double buffer)
  double mv2[32][kPN];
  double cst[kPN];      // sum_j 1.0 * m^2 / v (the ones * (M^2/V)^T product)
  double lnorm[kPN];
  double rmax[16][kPM];
  double chain[kPM][4];
};

static_assert(sizeof(double) * (4 * 32 * kPM) >= sizeof(double) * 8 * kSoftmaxRowMax && kPM == kPN,
              "the operand tiles xs2..mv hold the 8 warps' softmax rows");

// One k = 4 step of the FP64 tensor-core MMA (DMMA): D(8x8) = A(8x4) B(4x8) + C.
// Fragments: lane (g = lane / 4, q = lane % 4) holds A[g][q], B[q][g] and
// C/D[g][2q], C/D[g][2q + 1]. The products are fused into the accumulation
// (not separately rounded), so gamma differs from the reference's in the last
// bits; the containers it feeds were byte-identical on every frame measured
// (DESIGN.md §2.4). Default for mixtures of more than 32 components; debug
// bit 128 selects the bit-exact SIMT kernel.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <bool DMMA>
__global__ void __launch_bounds__(256, 2) k_posterior(Batch bt, Model md) {
  extern __shared__ __align__(16) uint8_t post_smem[];
  PostSmem& S = *reinterpret_cast<PostSmem*>(post_smem);
  const int f = blockIdx.y;
  const int n = bt.or_count[f];
  const int row0 = blockIdx.x * kPM;
  if (row0 >= n) return;
  const int nc = md.nc;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const double* X = bt.x + ((long long)f * bt.cap_or + row0) * 32;
  double* gam = bt.gamma + ((long long)f * bt.cap_or + row0) * nc;
  const int rows = min(kPM, n - row0);
  for (int q = tid; q < kPM * 32; q += 256) {
    const int t = q >> 5, j = q & 31;
    const double v = t < rows ? X[t * 32 + j] : 0.0;
    S.xs[j][t] = v;
    S.xs2[j][t] = v * v;
  }
  double rm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  // Component tiles stream through a double buffer with cp.async from the
  // transposed (and zero-padded) tables: tile k + 1 loads while tile k is
  // multiplied.
  auto load_tile = [&](int c0, double (*iv)[kPN], double (*mv)[kPN]) {
    for (int q = tid; q < 32 * (kPN / 2); q += 256) {  // 16-byte chunks: (j, column pair)
      const int j = q / (kPN / 2), c = 2 * (q % (kPN / 2));
      cp_async16_post(&iv[j][c], md.inv_var_t + (long long)j * md.ncp + c0 + c);
      cp_async16_post(&mv[j][c], md.m_over_v_t + (long long)j * md.ncp + c0 + c);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  load_tile(0, S.iv, S.mv);
  int buf = 0;
  for (int c0 = 0; c0 < nc; c0 += kPN) {
    __syncthreads();  // everyone is done with the tile buffer loaded next
    const bool more = c0 + kPN < nc;
    if (more) load_tile(c0 + kPN, buf ? S.iv : S.iv2, buf ? S.mv : S.mv2);
    if (more) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (tid < kPN) {
      const int i = c0 + tid;
      S.cst[tid] = md.cst[i];
      S.lnorm[tid] = i < nc ? md.log_norm[i] : 0.0;
    }
    __syncthreads();
    const double(*TIV)[kPN] = buf ? S.iv2 : S.iv;
    const double(*TMV)[kPN] = buf ? S.mv2 : S.mv;
    buf ^= 1;
    if constexpr (DMMA) {
      // Warp w: rows 8w .. 8w + 7 x the tile's 64 components (8 MMA tiles),
      // both products over k = 0..31 in 8 steps.
      const int wi = tid >> 5, lane = tid & 31, g = lane >> 2, qq = lane & 3;
      double da[8][2], db[8][2];
#pragma unroll
      for (int ct = 0; ct < 8; ++ct) da[ct][0] = da[ct][1] = db[ct][0] = db[ct][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int j = 4 * kk + qq;
        const double ax2 = S.xs2[j][8 * wi + g], ax = S.xs[j][8 * wi + g];
#pragma unroll
        for (int ct = 0; ct < 8; ++ct) {
          dmma_8x8x4(da[ct][0], da[ct][1], ax2, TIV[j][8 * ct + g]);
          dmma_8x8x4(db[ct][0], db[ct][1], ax, TMV[j][8 * ct + g]);
        }
      }
      const int t = 8 * wi + g;
      double m = -INFINITY;
#pragma unroll
      for (int ct = 0; ct < 8; ++ct)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = 8 * ct + 2 * qq + h, i = c0 + cc;
          if (t < rows && i < nc) {
            const double p = da[ct][h] - 2.0 * db[ct][h] + S.cst[cc];
            const double lp = -0.5 * p + S.lnorm[cc];
            gam[t * nc + i] = lp;
            m = fmax(m, lp);
          }
        }
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
      rm[0] = fmax(rm[0], m);  // this lane's row t (lanes of a quad agree)
      continue;
    }
    double a[4][4], b[4][4];
    {
      const double2 xa = *reinterpret_cast<const double2*>(&S.xs2[0][ty * 4]);
      const double2 xb = *reinterpret_cast<const double2*>(&S.xs2[0][ty * 4 + 2]);
      const double2 ya = *reinterpret_cast<const double2*>(&S.xs[0][ty * 4]);
      const double2 yb = *reinterpret_cast<const double2*>(&S.xs[0][ty * 4 + 2]);
      const double2 ia = *reinterpret_cast<const double2*>(&TIV[0][tx * 4]);
      const double2 ib = *reinterpret_cast<const double2*>(&TIV[0][tx * 4 + 2]);
      const double2 ma = *reinterpret_cast<const double2*>(&TMV[0][tx * 4]);
      const double2 mb = *reinterpret_cast<const double2*>(&TMV[0][tx * 4 + 2]);
      const double x2[4] = {xa.x, xa.y, xb.x, xb.y}, x1[4] = {ya.x, ya.y, yb.x, yb.y};
      const double iv[4] = {ia.x, ia.y, ib.x, ib.y}, mv[4] = {ma.x, ma.y, mb.x, mb.y};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          a[r][c] = x2[r] * iv[c];
          b[r][c] = x1[r] * mv[c];
        }
    }
#pragma unroll 4
    for (int j = 1; j < 32; ++j) {
      const double2 xa = *reinterpret_cast<const double2*>(&S.xs2[j][ty * 4]);
      const double2 xb = *reinterpret_cast<const double2*>(&S.xs2[j][ty * 4 + 2]);
      const double2 ya = *reinterpret_cast<const double2*>(&S.xs[j][ty * 4]);
      const double2 yb = *reinterpret_cast<const double2*>(&S.xs[j][ty * 4 + 2]);
      const double2 ia = *reinterpret_cast<const double2*>(&TIV[j][tx * 4]);
      const double2 ib = *reinterpret_cast<const double2*>(&TIV[j][tx * 4 + 2]);
      const double2 ma = *reinterpret_cast<const double2*>(&TMV[j][tx * 4]);
      const double2 mb = *reinterpret_cast<const double2*>(&TMV[j][tx * 4 + 2]);
      const double x2[4] = {xa.x, xa.y, xb.x, xb.y}, x1[4] = {ya.x, ya.y, yb.x, yb.y};
      const double iv[4] = {ia.x, ia.y, ib.x, ib.y}, mv[4] = {ma.x, ma.y, mb.x, mb.y};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          a[r][c] = a[r][c] + x2[r] * iv[c];
          b[r][c] = b[r][c] + x1[r] * mv[c];
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int t = ty * 4 + r;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = c0 + tx * 4 + c;
        if (t < rows && i < nc) {
          const double p = a[r][c] - 2.0 * b[r][c] + S.cst[tx * 4 + c];
          const double lp = -0.5 * p + S.lnorm[tx * 4 + c];
          gam[t * nc + i] = lp;
          rm[r] = fmax(rm[r], lp);
        }
      }
    }
  }
  if constexpr (DMMA) {
    if ((tid & 3) == 0) S.rmax[0][8 * (tid >> 5) + ((tid & 31) >> 2)] = rm[0];
  } else {
#pragma unroll
    for (int r = 0; r < 4; ++r) S.rmax[tx][ty * 4 + r] = rm[r];
    __syncthreads();
    if (tid < kPM) {
      double pk = S.rmax[0][tid];
      for (int k = 1; k < 16; ++k) pk = fmax(pk, S.rmax[k][tid]);
      S.rmax[0][tid] = pk;
    }
  }
  __syncthreads();
  const int wi = tid >> 5, lane = tid & 31;
  if (nc <= kSoftmaxRowMax) {
    // softmax_rows fused per row: a warp stages its row's e = exp(logp - peak)
    // in shared memory (the phase-1 operand tiles are free now), four lanes
    // sum it in Eigen's packet order (four stride-4 chains, then
    // (c0 + c2) + (c1 + c3), the odd pair and the tail), and the warp writes
    // gamma = e / sum: one read and one write of each gamma row.
    double* buf = reinterpret_cast<double*>(&S.xs2[0][0]) + wi * kSoftmaxRowMax;
    for (int t = wi; t < rows; t += 8) {
      const double pk = S.rmax[0][t];
      double* g = gam + t * nc;
      for (int i = lane; i < nc; i += 32) buf[i] = dm::exp(g[i] - pk);
      __syncwarp();
      double total = 0.0;
      if (nc < 4) {
        if (lane == 0) total = packet_sum_seq(buf, nc);
      } else {
        const int e2 = nc / 4 * 4, e1 = nc / 2 * 2;
        double c = 0.0;
        if (lane < 4) {
          c = buf[lane];
          for (int i = lane + 4; i < e2; i += 4) c = c + buf[i];
        }
        const double c0 = __shfl_sync(0xffffffffu, c, 0), c1 = __shfl_sync(0xffffffffu, c, 1);
        const double c2 = __shfl_sync(0xffffffffu, c, 2), c3 = __shfl_sync(0xffffffffu, c, 3);
        if (lane == 0) {
          double a0 = c0 + c2, a1 = c1 + c3;
          if (e1 > e2) {
            a0 += buf[e2];
            a1 += buf[e2 + 1];
          }
          total = a0 + a1;
          for (int i = e1; i < nc; ++i) total += buf[i];
        }
      }
      total = __shfl_sync(0xffffffffu, total, 0);
      for (int i = lane; i < nc; i += 32) g[i] = buf[i] / total;
      __syncwarp();
    }
    return;
  }
  // softmax_rows: e = exp(logp - peak) ...
  for (int t = wi; t < rows; t += 8) {
    const double pk = S.rmax[0][t];
    for (int i = lane; i < nc; i += 32) gam[t * nc + i] = dm::exp(gam[t * nc + i] - pk);
  }
  __syncthreads();
  // ... e.sum() in Eigen's packet order (packet_sum_seq) ...
  {
    const int t = tid >> 2, k = tid & 3;
    if (t < rows && nc >= 4) {
      const double* e = gam + t * nc;
      const int e2 = nc / 4 * 4;
      double acc = e[k];
      int i = k + 4;
      for (; i + 28 < e2; i += 32) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = e[i + 4 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = acc + v[u];
      }
      for (; i < e2; i += 4) acc = acc + e[i];
      S.chain[t][k] = acc;
    }
  }
  __syncthreads();
  if (tid < rows) {
    const double* e = gam + tid * nc;
    double total;
    if (nc < 4) {
      total = packet_sum_seq(e, nc);
    } else {
      const int e2 = nc / 4 * 4, e1 = nc / 2 * 2;
      double a0 = S.chain[tid][0] + S.chain[tid][2], a1 = S.chain[tid][1] + S.chain[tid][3];
      if (e1 > e2) {
        a0 += e[e2];
        a1 += e[e2 + 1];
      }
      total = a0 + a1;
      for (int i = e1; i < nc; ++i) total += e[i];
    }
    S.chain[tid][0] = total;
  }
  __syncthreads();
  // ... gamma = e / sum.
  for (int t = wi; t < rows; t += 8) {
    const double tot = S.chain[t][0];
    for (int i = lane; i < nc; i += 32) gam[t * nc + i] = gam[t * nc + i] / tot;
  }
}

// posteriors_matrix + softmax_rows for small mixtures (nc <= 32, e.g. the
// 8-component bundles): the 64-component tiles of k_posterior would be mostly
// padding. Thread per row: the row's 32 coordinates stay in registers, the
// mixture's 1/sigma^2 and mu/sigma^2 rows are shared-memory broadcasts, and
// logp of every component is formed with exactly k_posterior's arithmetic
// (sums over j ascending, separately rounded); the same thread then runs the
// row softmax (peak, exp, the packet-order sum of eigen_sum, division).
constexpr int kSmallRows = 64;
__global__ void __launch_bounds__(kSmallRows) k_posterior_small(Batch bt, Model md) {
  __shared__ double iv[32][32], mv[32][32];  // [component][j]
  __shared__ double lp[kSmallRows][33];
  __shared__ double cst[32], lnorm[32];
  const int f = blockIdx.y;
  const int n = bt.or_count[f];
  const int nc = md.nc;
  const int row0 = blockIdx.x * kSmallRows;
  if (row0 >= n) return;
  const int tid = threadIdx.x;
  for (int q = tid; q < nc * 32; q += kSmallRows) {
    iv[q >> 5][q & 31] = md.inv_var[q];
    mv[q >> 5][q & 31] = md.m_over_v[q];
  }
  if (tid < nc) {
    const double* m2 = md.m2_over_v + tid * 32;
    double c = 1.0 * m2[0];
    for (int j = 1; j < 32; ++j) c = c + 1.0 * m2[j];
    cst[tid] = c;
    lnorm[tid] = md.log_norm[tid];
  }
  __syncthreads();
  const int t = row0 + tid;
  if (t >= n) return;
  double x[32];
  const double2* X = reinterpret_cast<const double2*>(bt.x + ((long long)f * bt.cap_or + t) * 32);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double2 v = X[j];
    x[2 * j] = v.x;
    x[2 * j + 1] = v.y;
  }
  double* e = lp[tid];
  for (int i = 0; i < nc; ++i) {
    double a = (x[0] * x[0]) * iv[i][0];
    double b = x[0] * mv[i][0];
#pragma unroll
    for (int j = 1; j < 32; ++j) {
      a = a + (x[j] * x[j]) * iv[i][j];
      b = b + x[j] * mv[i][j];
    }
    const double p = a - 2.0 * b + cst[i];
    e[i] = -0.5 * p + lnorm[i];
  }
  double pk = e[0];
  for (int i = 1; i < nc; ++i) pk = fmax(pk, e[i]);
  for (int i = 0; i < nc; ++i) e[i] = dm::exp(e[i] - pk);
  const double tot = packet_sum_seq(e, nc);
  double* gam = bt.gamma + ((long long)f * bt.cap_or + t) * nc;
  for (int i = 0; i < nc; ++i) gam[i] = e[i] / tot;
}

// fv_mean_matrix / fv_var_matrix (scfv.cpp:166-203). gamma^T X (and
// gamma^T X^2) as sums over the descriptor index t, ascending, one separately
// rounded multiply and add per term. A CTA owns kFI components x all 32
// dimensions; thread (g, j) accumulates components g*4 .. g*4+3 of
// dimension j while the CTA streams gamma and X rows through shared memory.
// gamma^T 1 is the same for every j: it is summed once per component.
constexpr int kFI = 32, kFT = 64;
__global__ void __launch_bounds__(256) k_fisher(Batch bt, Model md, int variance) {
  __shared__ __align__(16) double sg[kFT][kFI];
  __shared__ double sx[kFT][32];
  __shared__ double qo_s[kFI];
  const int f = blockIdx.y;
  const int n = bt.or_count[f];
  const int nc = md.nc;
  const int i0 = blockIdx.x * kFI;
  const int tid = threadIdx.x, j = tid & 31, g = tid >> 5;
  double* gm = bt.gm + (long long)f * nc * 32;
  double* gv = bt.gv + (long long)f * nc * 32;
  if (n == 0) {
    for (int q = tid; q < kFI * 32; q += 256)
      if (i0 + q / 32 < nc) {
        gm[(long long)i0 * 32 + q] = 0.0;
        gv[(long long)i0 * 32 + q] = 0.0;
      }
    return;
  }
  const double* G = bt.gamma + (long long)f * bt.cap_or * nc;
  const double* X = bt.x + (long long)f * bt.cap_or * 32;
  double qx[4], qx2[4], qo = 0.0;
  for (int t0 = 0; t0 < n; t0 += kFT) {
    const int tn = min(kFT, n - t0);
    __syncthreads();
    for (int q = tid; q < kFT * kFI; q += 256) {
      const int t = q / kFI, i = q % kFI;
      sg[t][i] = (t < tn && i0 + i < nc) ? G[(long long)(t0 + t) * nc + i0 + i] : 0.0;
    }
    for (int q = tid; q < kFT * 32; q += 256) {
      const int t = q >> 5;
      sx[t][q & 31] = t < tn ? X[(t0 + t) * 32 + (q & 31)] : 0.0;
    }
    __syncthreads();
    for (int t = 0; t < tn; ++t) {
      const double xt = sx[t][j];
      const double xt2 = xt * xt;
      const double2 ga = *reinterpret_cast<const double2*>(&sg[t][g * 4]);
      const double2 gb = *reinterpret_cast<const double2*>(&sg[t][g * 4 + 2]);
      const double gg[4] = {ga.x, ga.y, gb.x, gb.y};
      if (t0 + t == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          qx[c] = gg[c] * xt;
          qx2[c] = gg[c] * xt2;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          qx[c] = qx[c] + gg[c] * xt;
          if (variance) qx2[c] = qx2[c] + gg[c] * xt2;
        }
      }
    }
    if (tid < kFI) {
      for (int t = 0; t < tn; ++t) qo = (t0 + t == 0) ? sg[t][tid] * 1.0 : qo + sg[t][tid] * 1.0;
    }
  }
  if (tid < kFI) qo_s[tid] = qo;
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int i = i0 + g * 4 + c;
    if (i >= nc) continue;
    const int ij = i * 32 + j;
    const double scale = 1.0 / (double(n) * sqrt(md.weights[i]));
    const double q1 = qo_s[g * 4 + c];
    const double m = md.means[ij], s = md.stds[ij];
    gm[ij] = ((qx[c] - q1 * m) / s) * scale;
    if (variance) {
      const double var = s * s;
      gv[ij] = ((qx2[c] - qx[c] * (2.0 * m) + q1 * (m * m - var)) / var) * scale;
    }
  }
}

// scfv_delta / scfv_encode (scfv.cpp:205-253): one CTA per frame.
__global__ void __launch_bounds__(256) k_scfv_encode(Batch bt, Model md, EncodeConst ec) {
  extern __shared__ double sdelta[];
  const int f = blockIdx.x;
  const int nc = md.nc;
  const double* gm = bt.gm + (long long)f * nc * 32;
  const double* gv = bt.gv + (long long)f * nc * 32;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const double* g = gm + i * 32;
    const double mean = packet_sum_seq(g, 32) / 32;
    double d[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) d[j] = (g[j] - mean) * (g[j] - mean);
    sdelta[i] = sqrt(packet_sum_seq(d, 32) / 32.0);
    bt.norms[(long long)f * nc + i] = sdelta[i];
  }
  __syncthreads();
  uint8_t* chosen = reinterpret_cast<uint8_t*>(sdelta + nc);
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const double di = sdelta[i];
    int rank = 0;
    for (int j = 0; j < nc; ++j) {
      const double dj = sdelta[j];
      rank += (dj > di || (dj == di && j < i)) ? 1 : 0;
    }
    const bool sel = rank < ec.k_select;
    uint32_t mb = 0, vb = 0;
    for (int j = 0; j < 32; ++j) {
      if (gm[i * 32 + j] >= 0.0) mb |= (1u << j);
      if (ec.variance && gv[i * 32 + j] >= 0.0) vb |= (1u << j);
    }
    bt.mean_planes[(long long)f * nc + i] = mb;
    bt.var_planes[(long long)f * nc + i] = vb;
    chosen[i] = sel ? 1 : 0;
  }
  __syncthreads();
  uint8_t* mask = bt.mask + (long long)f * ec.mask_bytes;
  for (int b = threadIdx.x; b < ec.mask_bytes; b += blockDim.x) {
    uint8_t byte = 0;
    for (int q = 0; q < 8 && b * 8 + q < nc; ++q) byte |= uint8_t(chosen[b * 8 + q] << q);
    mask[b] = byte;
  }
}

// serialize_container (container.cpp:32-58) into a fixed device slot.
// CRC-32 (common.cpp:11-35) by a warp. The reflected CRC register update is
// linear over GF(2), so raw(0, A || B) = Z^|B| raw(0, A) ^ raw(0, B) with Z the
// "one zero byte" operator: lanes take 128-byte chunks, a shuffle tree merges
// them with the precomputed operators Z^(2^k) (c_zeros), and the standard
// init/final inversion is applied by linearity at the end.
__constant__ uint32_t c_zeros[17][32];  // c_zeros[k][b] = Z^(2^k) applied to register 1 << b

cudaError_t init_crc_zeros() {
  // c_zeros is per device (constant memory of each device's module image).
  static size_t done[kMaxDevices] = {};
  return once_per_device(done, 1, [] {
    uint32_t table[256];
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    uint32_t z[17][32];
    for (int b = 0; b < 32; ++b) z[0][b] = table[(1u << b) & 0xFFu] ^ ((1u << b) >> 8);
    for (int k = 1; k < 17; ++k)
      for (int b = 0; b < 32; ++b) {  // Z^(2^k) = Z^(2^(k-1)) o Z^(2^(k-1))
        uint32_t v = z[k - 1][b], r = 0;
        for (int c = 0; c < 32; ++c)
          if ((v >> c) & 1u) r ^= z[k - 1][c];
        z[k][b] = r;
      }
    return cudaMemcpyToSymbol(c_zeros, z, sizeof(z));
  });
}

__device__ __forceinline__ uint32_t crc_shift(uint32_t v, uint32_t nbytes) {
  for (int k = 0; nbytes; ++k, nbytes >>= 1)
    if (nbytes & 1u) {
      uint32_t r = 0;
#pragma unroll
      for (int b = 0; b < 32; ++b) r ^= ((v >> b) & 1u) ? c_zeros[k][b] : 0u;
      v = r;
    }
  return v;
}

// Whole warp calls; the CRC is returned on every lane.
__device__ uint32_t warp_crc32(const uint8_t* buf, int n, const uint32_t* table) {
  constexpr int C = 128;
  const int lane = threadIdx.x & 31;
  const int nfull = n / C;
  uint32_t acc = 0;  // raw CRC (register from 0) of the chunks merged so far
  for (int sb = 0; sb < nfull; sb += 32) {
    const int nch = min(32, nfull - sb);
    uint32_t r = 0;
    if (lane < nch) {
      const uint8_t* p = buf + (sb + lane) * C;
      for (int i = 0; i < C; ++i) r = table[(r ^ p[i]) & 0xFFu] ^ (r >> 8);
    }
    for (int st = 1; st < 32; st <<= 1) {
      const uint32_t rr = __shfl_down_sync(0xffffffffu, r, st);
      const int cnt = min(st, max(0, nch - (lane + st)));
      if ((lane & (2 * st - 1)) == 0 && cnt > 0) r = crc_shift(r, uint32_t(cnt * C)) ^ rr;
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    acc = crc_shift(acc, uint32_t(nch * C)) ^ r;
  }
  if (lane == 0)
    for (int i = nfull * C; i < n; ++i) acc = table[(acc ^ buf[i]) & 0xFFu] ^ (acc >> 8);
  acc = __shfl_sync(0xffffffffu, acc, 0);
  return ~(crc_shift(0xFFFFFFFFu, uint32_t(n)) ^ acc);
}

__global__ void __launch_bounds__(256) k_pack(Batch bt, Model md, EncodeConst ec, uint8_t* out, uint32_t* lengths) {
  extern __shared__ uint8_t buf[];
  __shared__ uint32_t table[256];
  __shared__ int s_len;
  const int f = blockIdx.x;
  const int nc = md.nc;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = uint32_t(i);
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    table[i] = c;
  }
  if (bt.status[f] != 0) {
    if (threadIdx.x == 0) lengths[f] = 0;
    return;
  }
  const int n_codes = min(bt.or_count[f], ec.max_codes);
  const int local_len = 4 + n_codes * ec.code_bytes;
  const int total = 24 + ec.global_bytes + local_len + 4;
  const uint8_t* mask = bt.mask + (long long)f * ec.mask_bytes;
  if (threadIdx.x == 0) {
    uint8_t* p = buf;
    p[0] = 'C'; p[1] = 'D'; p[2] = 'V'; p[3] = 'Z'; p[4] = '1';
    p[5] = uint8_t(ec.mode_id);
    p[6] = uint8_t(bt.W & 0xFF); p[7] = uint8_t(bt.W >> 8);
    p[8] = uint8_t(bt.H & 0xFF); p[9] = uint8_t(bt.H >> 8);
    p[10] = uint8_t(nc & 0xFF); p[11] = uint8_t(nc >> 8);
    const uint32_t vals[3] = {ec.model_crc, uint32_t(ec.global_bytes), uint32_t(local_len)};
    for (int q = 0; q < 3; ++q)
      for (int b = 0; b < 4; ++b) p[12 + 4 * q + b] = uint8_t((vals[q] >> (8 * b)) & 0xFF);
    // global block: mask, then planes of selected components in ascending order
    int off = 24;
    for (int b = 0; b < ec.mask_bytes; ++b) p[off++] = mask[b];
    for (int i = 0; i < nc; ++i) {
      if (!((mask[i / 8] >> (i % 8)) & 1)) continue;
      const uint32_t mb = bt.mean_planes[(long long)f * nc + i];
      for (int b = 0; b < 4; ++b) p[off++] = uint8_t((mb >> (8 * b)) & 0xFF);
      if (ec.variance) {
        const uint32_t vb = bt.var_planes[(long long)f * nc + i];
        for (int b = 0; b < 4; ++b) p[off++] = uint8_t((vb >> (8 * b)) & 0xFF);
      }
    }
    // local block header (transform_coding.cpp:236-240)
    p[off++] = uint8_t(ec.mode_id);
    p[off++] = uint8_t(ec.elements);
    p[off++] = uint8_t(n_codes & 0xFF);
    p[off++] = uint8_t(n_codes >> 8);
    s_len = off;
  }
  __syncthreads();
  const int code_base = s_len;
  const uint8_t* codes = bt.codes + (long long)f * bt.cap_or * bt.code_stride;
  for (int q = threadIdx.x; q < n_codes * ec.code_bytes; q += blockDim.x) {
    const int c = q / ec.code_bytes, b = q % ec.code_bytes;
    buf[code_base + q] = codes[(long long)c * bt.code_stride + b];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int body = total - 4;
    const uint32_t c = warp_crc32(buf, body, table);
    if (threadIdx.x == 0) {
      for (int b = 0; b < 4; ++b) buf[body + b] = uint8_t((c >> (8 * b)) & 0xFF);
      lengths[f] = uint32_t(total);
    }
  }
  __syncthreads();
  uint8_t* dst = out + (long long)f * ec.slot_bytes;
  for (int i = threadIdx.x; i < total; i += blockDim.x) dst[i] = buf[i];
}

cudaError_t launch_scfv_pack(const Batch& bt, const Model& md, const EncodeConst& ec, uint8_t* out, uint32_t* lengths,
                             cudaStream_t st, cudaEvent_t after_aggregation) {
  cudaError_t e = init_crc_zeros();
  if (e != cudaSuccess) return e;
  constexpr int pca_smem = int(sizeof(double)) * (128 * 33 + 16 * 128);
  static size_t pca_configured[kMaxDevices] = {};
  e = once_per_device(pca_configured, 1, [&] { return cudaFuncSetAttribute(k_pca, cudaFuncAttributeMaxDynamicSharedMemorySize, pca_smem); });
  if (e != cudaSuccess) return e;
  k_pca<<<dim3(16, bt.nframes), 128, pca_smem, st>>>(bt, md);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  static size_t post_configured[kMaxDevices] = {};
  e = once_per_device(post_configured, 1, [&] {
    cudaError_t r = cudaFuncSetAttribute(k_posterior<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem)));
    return r != cudaSuccess ? r : cudaFuncSetAttribute(k_posterior<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem)));
  });
  if (e != cudaSuccess) return e;
  const dim3 pgrid((bt.cap_or + kPM - 1) / kPM, bt.nframes);
  if (md.nc <= 32)
    k_posterior_small<<<dim3((bt.cap_or + kSmallRows - 1) / kSmallRows, bt.nframes), kSmallRows, 0, st>>>(bt, md);
  else if (ec.post_dmma)  // the FP64 tensor cores
    k_posterior<true><<<pgrid, 256, sizeof(PostSmem), st>>>(bt, md);
  else
    k_posterior<false><<<pgrid, 256, sizeof(PostSmem), st>>>(bt, md);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_fisher<<<dim3((md.nc + kFI - 1) / kFI, bt.nframes), 256, 0, st>>>(bt, md, ec.variance);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t esm = sizeof(double) * size_t(md.nc) + size_t(md.nc);
  if (esm > 48 * 1024) {
    e = cudaFuncSetAttribute(k_scfv_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, int(esm));
    if (e != cudaSuccess) return e;
  }
  k_scfv_encode<<<bt.nframes, 256, esm, st>>>(bt, md, ec);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (after_aggregation) cudaEventRecord(after_aggregation, st);
  const size_t ksm = size_t(ec.slot_bytes);
  if (ksm > 48 * 1024) {
    e = cudaFuncSetAttribute(k_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ksm));
    if (e != cudaSuccess) return e;
  }
  k_pack<<<bt.nframes, 256, ksm, st>>>(bt, md, ec, out, lengths);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
