// Shared device definitions for the B200 extractor kernels.
//
// Arithmetic contract: every file is compiled with --fmad=false so each
// multiply and add rounds separately, in the same order as the reference's
// double-precision code (and the oracle that restates it). Bit-level parity
// with the oracle follows wherever no libm call intervenes.
#pragma once

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace cdvz_gpu {

constexpr int kMaxOctaves = 8;
constexpr int kMaxTapRadius = 16;

// Keypoint record shared by every list on the device (64 bytes).
// Mirrors InterestPoint (proj/include/cdvz/scale_space.hpp:56-64).
struct KP {
  double x, y, sigma, p, rho, pss, d;
  int octave;
  uint32_t key;  // octave-local raster key (y*w + x)*2 + root slot, order of detection
};
static_assert(sizeof(KP) == 64, "KP layout");

struct Oriented { int sel; int pad; double theta; };

// Sampling geometry of one oriented point (make_geometry + resolve_frame,
// descriptor.cpp:47-58,149-170), shared by the sample and histogram kernels.
struct DescGeo {
  double x, y, cos_t, sin_t, step, half, inv_cell, gauss_denom;
  long long lvl_off;   // doubles from the batch pyramid base to the level plane
  int w, h, samples, pad;
};
static_assert(sizeof(DescGeo) == 88, "DescGeo layout");

// Detector constants (ScaleSpaceConfig + derived; scale_space.hpp:16-27).
struct DetConst {
  double taps[4][2 * kMaxTapRadius + 1];
  int radius[4];
  double sigmas[4];
  double s2[4];        // sigma_k * sigma_k (scale_space.cpp:150)
  double beta[4][4];
  double thr, rho_limit, s_lo, s_hi;
  int margin;
  int screen;          // 1: FP32 pre-screen before the exact test; 0: exact test on every pixel
  float scr_lo, scr_hi, scr_thr;  // screen constants: s_lo - 0.05, s_hi + 0.05, thr (FP32)
  int walk;            // 1: warp column-walk extrema kernel; 0: TMA tile kernel
  int blur_unrolled;   // 1: k_blur's y pass unrolled by one accumulator period; 0: rolled (shifted accumulators)
  int desc_registers;  // 1: k_describe with register bins; 0: k_describe_cells (shared-memory cell accumulators)
};

// Per-batch geometry and buffer map (device pointers). One instance lives in
// global memory per batch; kernels receive it by value (fits the 4 KB limit).
struct Batch {
  int nframes;
  int W, H;                       // prepared (resized) size
  int n_oct;
  int ow[kMaxOctaves], oh[kMaxOctaves];
  long long plane_off[kMaxOctaves][4];  // doubles, within a frame's pyramid
  long long frame_doubles;              // pyramid doubles per frame
  double* pyr;                          // [frame][...]
  // Octave-0 input: either u8 frames (pix8) or resized f64 frames (pixf).
  const uint8_t* pix8; long long stride8; long long frame_bytes8;
  const double* pixf;
  // Detection lists.
  int cap_oct;                         // survivors per (frame, octave)
  KP* raw;                             // [frame][octave][cap_oct] unordered survivors
  int* raw_count;                      // [frame][octave]
  int* oct_count;                      // [frame][octave] survivors per octave (after ordering)
  uint32_t* bitmap;                    // [frame][bitmap_words]
  int* bm_prefix;                      // [frame][bitmap_words] word prefix counts when they exceed shared memory
  int merge_cell;                      // dedup grid cell side in px (8, doubled until the grid fits shared memory)
  long long bm_off[kMaxOctaves];       // word offset of each octave's bitmap in a frame
  long long bitmap_words;              // per frame
  int cap_acc;
  KP* acc[2];                          // [frame][cap_acc] ping-pong accumulated lists
  int* acc_count;                      // [frame][2]
  KP* cur;                             // [frame][cap_acc] scratch (sorted current octave)
  int* scratch_idx;                    // [frame][cap_acc]
  uint8_t* flags;                      // [frame][2*cap_acc]
  double* scratch_d;                   // [frame][cap_acc]
  int* status;                         // [frame] 0 ok, 3 internal (capacity)
  // Selection / orientation / description.
  int select_n;
  KP* sel;                             // [frame][select_n]
  int* sel_count;                      // [frame]
  double* thetas;                      // [frame][select_n][36]
  int* theta_count;                    // [frame][select_n]
  int cap_or;
  Oriented* oriented;                  // [frame][cap_or]
  int* or_count;                       // [frame]
  DescGeo* geo;                        // [frame][cap_or]
  int* order;                          // [frame][cap_or]: oriented points by descending samples per axis (k_order)
  int smp_cap;                         // samples per oriented point (max samples^2)
  double2* smp;                        // [frame][cap_or][smp_cap] {weight (+0: skipped), fo}, row stride samples
  uint8_t* smpb;                       // [frame][cap_or][32][32] orientation bin ob0 mod 8 of each sample
  double* desc;                        // [frame][cap_or][128]
  uint8_t* codes;                      // [frame][cap_or][code_stride]
  int code_stride;
  // SCFV.
  int nc;
  double* x;                           // [frame][cap_or][32]
  double* gamma;                       // [frame][cap_or][nc]
  double* gm;                          // [frame][nc][32]
  double* gv;                          // [frame][nc][32]
  uint8_t* mask;                       // [frame][mask_bytes] (selected components)
  uint32_t* mean_planes;               // [frame][nc] by component index
  uint32_t* var_planes;                // [frame][nc]
  double* norms;                       // [frame][nc] scfv_delta of every component (SCFVDescriptor::norms)
};

// Model tables in global memory.
struct Model {
  const double* rel_edges[5];
  const double* rel_vals[5];
  int rel_nb[5];
  double tr[2][8][8];
  double tr_scale;
  const double* t0;
  const double* t1;
  const int* priority;
  const double* pca_mean;   // 128
  const double* pca_basis;  // 32 x 128
  int nc;
  const double* inv_var;    // nc x 32  1/(s*s)
  const double* m_over_v;   // nc x 32  m/(s*s)
  const double* m2_over_v;  // nc x 32  (m*m)/(s*s)
  const double* inv_var_t;  // 32 x ncp  transposed, rows padded to ncp = nc rounded up to 64 (zeros)
  const double* m_over_v_t; // 32 x ncp
  const double* cst;        // ncp      sum_j 1.0 * m2_over_v[i][j], j ascending (0 past nc)
  int ncp;
  const double* log_norm;   // nc       log w - sum log s - 16 log 2pi
  const double* means;      // nc x 32
  const double* stds;       // nc x 32
  const double* weights;    // nc
};

// Encoding parameters of one call.
struct EncodeConst {
  int mode_id, elements, variance;
  int k_select;                 // SCFV components kept
  int max_codes;
  int code_bytes;
  int mask_bytes;
  int global_bytes;
  int slot_bytes;               // container slot
  uint32_t model_crc;
  double half_diag, cx, cy;     // fill_center_distance constants
  double log2_range;            // log2(64 / 0.5)
  int post_dmma;                // 1: posteriors of mixtures > 32 components on the FP64 tensor cores
};

__host__ __device__ inline int mirror_index(int i, int n) {
  if (n <= 1) return 0;
  const int period = 2 * n;
  int m = i % period;
  if (m < 0) m += period;
  return m < n ? m : period - 1 - m;
}

// Host-side setup that must happen once per device (kernel attributes,
// __constant__ tables): runs `f` unless the current device has already been
// set up with a value >= v (e.g. a dynamic shared-memory size). Thread-safe.
constexpr int kMaxDevices = 64;
inline std::mutex& device_setup_mutex() {
  static std::mutex m;
  return m;
}
template <class F>
cudaError_t once_per_device(size_t (&seen)[kMaxDevices], size_t v, F&& f) {
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return e;
  if (d < 0 || d >= kMaxDevices) return f();
  std::lock_guard<std::mutex> g(device_setup_mutex());
  if (seen[d] >= v) return cudaSuccess;
  e = f();
  if (e == cudaSuccess) seen[d] = v;
  return e;
}

#define CDVZ_CUDA_CHECK(expr)                                                              \
  do {                                                                                     \
    cudaError_t e__ = (expr);                                                              \
    if (e__ != cudaSuccess) throw std::runtime_error(std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

}  // namespace cdvz_gpu
