// K0 — ingest: PPM RGB -> grey conversion (load_image, proj/src/image.cpp:79-87),
// bilinear resize of u8 or f64 grey frames to the prepared raster
// (resize_max_side / rescale_bilinear, proj/src/image.cpp:107-145), and the
// deterministic synthetic frame generator used by the benchmarks
// (synth_image / synth_corpus, proj/src/synthetic.cpp:11-61).
#include <algorithm>

#include "common.cuh"
#include "dmath.cuh"

namespace cdvz_gpu {

// One thread per output pixel; frames along grid.z. Source values are u8
// bytes read as b / 255 (load_image of a PGM) or an f64 grey plane (a
// converted PPM).
template <class T>
__device__ __forceinline__ double src_value(const T* row, int x) {
  if constexpr (sizeof(T) == 1) return row[x] * (1.0 / 255.0);  // image.cpp:79-87
  else return row[x];
}

template <class T>
__global__ void k_resize(const T* pix, long long stride, long long frame_elems, int w_in, int h_in, double* out,
                         int w_out, int h_out, double sx, double sy) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int f = blockIdx.z;
  if (x >= w_out) return;
  const T* img = pix + f * frame_elems;
  double src_y = (y + 0.5) * sy - 0.5;
  src_y = fmin(fmax(src_y, 0.0), double(h_in - 1));
  const int y0 = static_cast<int>(src_y);
  const int y1 = min(y0 + 1, h_in - 1);
  const double fy = src_y - y0;
  double src_x = (x + 0.5) * sx - 0.5;
  src_x = fmin(fmax(src_x, 0.0), double(w_in - 1));
  const int x0 = static_cast<int>(src_x);
  const int x1 = min(x0 + 1, w_in - 1);
  const double fx = src_x - x0;
  const T* r0 = img + (long long)y0 * stride;
  const T* r1 = img + (long long)y1 * stride;
  const double p00 = src_value(r0, x0), p01 = src_value(r0, x1);
  const double p10 = src_value(r1, x0), p11 = src_value(r1, x1);
  out[(long long)f * w_out * h_out + (long long)y * w_out + x] =
      (1.0 - fy) * ((1.0 - fx) * p00 + fx * p01) + fy * ((1.0 - fx) * p10 + fx * p11);
}

cudaError_t launch_resize(const uint8_t* pix, long long stride, long long frame_bytes, int w_in, int h_in, double* out,
                          int w_out, int h_out, int frames, cudaStream_t st) {
  const double sx = static_cast<double>(w_in) / w_out, sy = static_cast<double>(h_in) / h_out;
  dim3 grid((w_out + 127) / 128, h_out, frames);
  k_resize<uint8_t><<<grid, 128, 0, st>>>(pix, stride, frame_bytes, w_in, h_in, out, w_out, h_out, sx, sy);
  return cudaGetLastError();
}

cudaError_t launch_resize_f64(const double* grey, int w_in, int h_in, double* out, int w_out, int h_out, int frames,
                              cudaStream_t st) {
  const double sx = static_cast<double>(w_in) / w_out, sy = static_cast<double>(h_in) / h_out;
  dim3 grid((w_out + 127) / 128, h_out, frames);
  k_resize<double><<<grid, 128, 0, st>>>(grey, w_in, (long long)w_in * h_in, w_in, h_in, out, w_out, h_out, sx, sy);
  return cudaGetLastError();
}

// validate (image.cpp:46-51) for f64 grey frames handed in by the caller:
// a frame with a non-finite value or one outside [0, 1] gets status 2 (the
// reference's DataError) and its raster is zeroed in the staging buffer, so
// the rest of the pipeline runs on a harmless plane and k_pack emits nothing
// for it. Grid (row blocks, frames); a second launch scrubs flagged frames.
__global__ void k_validate_f64(const double* pix, long long frame_elems, long long n, int* status) {
  const int f = blockIdx.y;
  const double* p = pix + f * frame_elems;
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = p[i];
    bad |= !(v >= 0.0 && v <= 1.0);  // NaN fails both comparisons; +-inf fails one
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&status[f], 2);
}

__global__ void k_scrub_f64(double* pix, long long frame_elems, long long n, const int* status) {
  const int f = blockIdx.y;
  if (status[f] == 0) return;
  double* p = pix + f * frame_elems;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

cudaError_t launch_validate_f64(double* pix, int w, int h, int frames, int* status, cudaStream_t st) {
  const long long n = (long long)w * h;
  const dim3 grid(unsigned(std::min<long long>(64, (n + 255) / 256)), frames);
  k_validate_f64<<<grid, 256, 0, st>>>(pix, n, n, status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_scrub_f64<<<grid, 256, 0, st>>>(pix, n, n, status);
  return cudaGetLastError();
}

// PPM ingest: interleaved 8-bit RGB -> grey f64, (0.299 r + 0.587 g + 0.114 b)
// * (1 / 255) in this order (load_image, image.cpp:82-86). One thread per
// pixel, frames along grid.z; `out` is a dense w x h plane per frame.
__global__ void k_grey_rgb(const uint8_t* rgb, long long stride, long long frame_bytes, int w, int h, double* out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int f = blockIdx.z;
  if (x >= w) return;
  const uint8_t* p = rgb + f * frame_bytes + (long long)y * stride + 3LL * x;
  const double inv = 1.0 / 255.0;
  out[(long long)f * w * h + (long long)y * w + x] = (0.299 * p[0] + 0.587 * p[1] + 0.114 * p[2]) * inv;
}

cudaError_t launch_grey_rgb(const uint8_t* rgb, long long stride, long long frame_bytes, int w, int h, double* out,
                            int frames, cudaStream_t st) {
  dim3 grid((w + 127) / 128, h, frames);
  k_grey_rgb<<<grid, 128, 0, st>>>(rgb, stride, frame_bytes, w, h, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- synthetic frames

struct SynthParams {
  int n_blobs;
  double blob[14][4];  // cx, cy, amp, denom
  double wave[5][4];   // fx, fy, phase, amp
};

// canvas(y, x): blobs in draw order, then the five waves (synthetic.cpp:19-44).
__global__ void k_synth_canvas(const SynthParams* params, int w, int h, double* canvas, double* bmin, double* bmax) {
  __shared__ double smin[256], smax[256];
  const int f = blockIdx.y;
  const SynthParams& p = params[f];
  double lo = INFINITY, hi = -INFINITY;
  const long long n = (long long)w * h;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int x = int(i % w), y = int(i / w);
    double c = 0.0;
    for (int b = 0; b < p.n_blobs; ++b) {
      const double dx = x - p.blob[b][0], dy = y - p.blob[b][1];
      c += p.blob[b][2] * dm::exp(-(dx * dx + dy * dy) / p.blob[b][3]);
    }
    for (int k = 0; k < 5; ++k)
      c += p.wave[k][3] * sin(2.0 * 3.14159265358979323846 * (p.wave[k][0] * x + p.wave[k][1] * y) + p.wave[k][2]);
    canvas[(long long)f * n + i] = c;
    lo = fmin(lo, c);
    hi = fmax(hi, c);
  }
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bmin[f * gridDim.x + blockIdx.x] = smin[0];
    bmax[f * gridDim.x + blockIdx.x] = smax[0];
  }
}

// img = 0.02 + 0.96 (canvas - lo) / (hi - lo), bytes = lround(img * 255)
// (synthetic.cpp:46-52, image.cpp:101-102).
__global__ void k_synth_quantize(const double* canvas, int w, int h, const double* bmin, const double* bmax, int nblk,
                                 uint8_t* out) {
  const int f = blockIdx.y;
  double lo = INFINITY, hi = -INFINITY;
  for (int b = 0; b < nblk; ++b) {
    lo = fmin(lo, bmin[f * nblk + b]);
    hi = fmax(hi, bmax[f * nblk + b]);
  }
  const long long n = (long long)w * h;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = hi > lo ? 0.02 + 0.96 * (canvas[(long long)f * n + i] - lo) / (hi - lo) : 0.5;
    out[(long long)f * n + i] = uint8_t(llround(v * 255.0));
  }
}

cudaError_t launch_synth(const SynthParams* d_params, int frames, int w, int h, double* canvas, double* bmin,
                         double* bmax, int nblk, uint8_t* out, cudaStream_t st) {
  k_synth_canvas<<<dim3(nblk, frames), 256, 0, st>>>(d_params, w, h, canvas, bmin, bmax);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_synth_quantize<<<dim3(nblk, frames), 256, 0, st>>>(canvas, w, h, bmin, bmax, nblk, out);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
