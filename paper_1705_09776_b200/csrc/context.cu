// Host runtime behind include/cdvz_gpu.h: context (device, stream, model
// tables), batch buffer planning, the per-batch launch sequence and the C ABI.
//
// One context drives one device on one stream. A batch of frames flows
// through ~20 launches with no host round trip: K0 resize (if needed),
// K1 fused octave + K2/K3 merge per octave, K4 selection, K5 orientation,
// K6/K7 description + coding, K8-K11 SCFV, K12 container pack. Per-frame
// failures (capacity overflow) are flagged on the device and surface as
// status 3 for that frame only.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/cdvz_gpu.h"
#include "bundle.hpp"
#include "common.cuh"
#include "train_host.hpp"

namespace cdvz_gpu {
cudaError_t launch_octave(const Batch& bt, const DetConst& dc, int o, int src, cudaStream_t st);
cudaError_t launch_detect(const Batch& bt, const DetConst& dc, int o, const CUtensorMap* tmap, const CUtensorMap* wmap,
                          cudaStream_t st);
cudaError_t launch_merge(const Batch& bt, int o, cudaStream_t st);
int merge_cell_px(int W, int H);
cudaError_t launch_select(const Batch& bt, const Model& md, const EncodeConst& ec, cudaStream_t st);
cudaError_t launch_describe(const Batch& bt, const DetConst& dc, cudaStream_t st);
cudaError_t launch_compress(const Batch& bt, const Model& md, const EncodeConst& ec, cudaStream_t st);
cudaError_t launch_scfv_pack(const Batch& bt, const Model& md, const EncodeConst& ec, uint8_t* out, uint32_t* lengths,
                             cudaStream_t st, cudaEvent_t after_aggregation);
cudaError_t launch_resize_f64(const double* grey, int w_in, int h_in, double* out, int w_out, int h_out, int frames,
                              cudaStream_t st);
cudaError_t launch_grey_rgb(const uint8_t* rgb, long long stride, long long frame_bytes, int w, int h, double* out,
                            int frames, cudaStream_t st);
cudaError_t launch_validate_f64(double* pix, int w, int h, int frames, int* status, cudaStream_t st);
cudaError_t launch_resize(const uint8_t* pix, long long stride, long long frame_bytes, int w_in, int h_in, double* out,
                          int w_out, int h_out, int frames, cudaStream_t st);
struct SynthParams {
  int n_blobs;
  double blob[14][4];
  double wave[5][4];
};
cudaError_t launch_synth(const SynthParams* d_params, int frames, int w, int h, double* canvas, double* bmin,
                         double* bmax, int nblk, uint8_t* out, cudaStream_t st);
}  // namespace cdvz_gpu

using namespace cdvz_gpu;

namespace {

thread_local std::string g_create_error;

// NVTX ranges (header-only nvtx3: no-ops unless a profiler injects itself) name
// the host side of a call in an Nsight / ncu --nvtx timeline: the public
// entry, each device shard's thread, and each chunk's enqueue.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DeviceBuffer {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    CDVZ_CUDA_CHECK(cudaMalloc(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Prepared size per resize_max_side (image.cpp:131-145).
void prepared_dims(int w, int h, int limit, int& pw, int& ph) {
  if (limit < 8) throw DataError("max-side limit must be at least 8");
  const int longer = std::max(w, h);
  pw = w;
  ph = h;
  if (longer <= limit) return;
  const double scale = static_cast<double>(limit) / longer;
  if (w >= h) {
    pw = limit;
    ph = std::max(8, static_cast<int>(std::lround(h * scale)));
  } else {
    ph = limit;
    pw = std::max(8, static_cast<int>(std::lround(w * scale)));
  }
}

}  // namespace

// One in-flight batch: its device buffers, two streams (A: the Gaussian
// blurs, which chain octave to octave; B: extrema, merge, selection,
// description, SCFV, pack) and the events that order and time them. Two
// lanes alternate over a call's chunks, so chunk c's description/SCFV runs
// beside chunk c+1's pyramid.
struct Lane {
  Batch bt{};
  std::vector<DeviceBuffer> bufs;
  DeviceBuffer dbg_oct;
  int geo_w = 0, geo_h = 0, geo_frames = 0;
  bool geo_resize = false, geo_debug = false;
  long long geo_grey = 0;  // doubles of the original-size grey plane buffer (RGB input + resize)
  double* grey = nullptr;  // [frame][h][w] grey plane of RGB frames before resize
  cudaStream_t sA = nullptr, sB = nullptr;
  cudaEvent_t start = nullptr, done = nullptr;
  cudaEvent_t stage[6] = {};
  cudaEvent_t blur[2 * kMaxOctaves] = {}, det[2 * kMaxOctaves] = {};
  CUtensorMap tmap[kMaxOctaves];   // 4-D view (x, y, level, frame) of each octave's G planes (k_detect tiles)
  CUtensorMap wmap[kMaxOctaves];   // the same view with k_detect_walk's box: 34 columns x 2 rows x 4 levels
  bool tmap_ok[kMaxOctaves] = {};
  bool pending = false;   // events of an enqueued chunk not yet folded into the stats
  long long pending_call = 0;  // the call that enqueued it
  int pending_oct = 0;
  double pending_bytes = 0.0;
  bool geo_boost = false;      // planned with the maximal capacities (capacity retry)
  bool geo_tiny = false;

  void init() {
    // The pyramid stream (A) gets the higher priority: its blur CTAs are
    // dispatched ahead of stream B's when both lanes have work, so the next
    // octave's / chunk's blur starts while the extrema, merge and description
    // kernels fill the remaining SM slots (+0.7% over equal priorities; a
    // per-lane priority split measured 8% slower).
    int least = 0, greatest = 0;
    CDVZ_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CDVZ_CUDA_CHECK(cudaStreamCreateWithPriority(&sA, cudaStreamNonBlocking, greatest));
    CDVZ_CUDA_CHECK(cudaStreamCreateWithPriority(&sB, cudaStreamNonBlocking, least));
    CDVZ_CUDA_CHECK(cudaEventCreate(&start));
    CDVZ_CUDA_CHECK(cudaEventCreate(&done));
    for (auto& e : stage) CDVZ_CUDA_CHECK(cudaEventCreate(&e));
    for (auto& e : blur) CDVZ_CUDA_CHECK(cudaEventCreate(&e));
    for (auto& e : det) CDVZ_CUDA_CHECK(cudaEventCreate(&e));
  }
  void release() {
    for (auto& b : bufs) b.release();
    bufs.clear();
    dbg_oct.release();
    geo_w = geo_h = geo_frames = 0;
    geo_boost = false;
  }
  void destroy() {
    release();
    for (auto* e : {&start, &done}) if (*e) cudaEventDestroy(*e);
    for (auto& e : stage) if (e) cudaEventDestroy(e);
    for (auto& e : blur) if (e) cudaEventDestroy(e);
    for (auto& e : det) if (e) cudaEventDestroy(e);
    if (sA) cudaStreamDestroy(sA);
    if (sB) cudaStreamDestroy(sB);
  }
};

struct cdvz_gpu_ctx {
  int device = 0;
  int max_batch = 256;
  int next_lane = 0;      // lane of the next call's first chunk
  size_t device_mem = 0;  // total device memory (queried once)
  cudaStream_t st = nullptr;
  cudaStream_t copy_st = nullptr;          // host->device frame copies (encode_batch)
  std::vector<cudaEvent_t> copy_ev;        // one per chunk of a call
  std::string err;
  Bundle bundle;
  DetConst dc{};
  Model md{};
  std::vector<DeviceBuffer> model_bufs;
  bool debug = false;
  bool serial = false;
  bool tma_disabled = false;
  bool post_simt = false;  // debug bit 128: SCFV posteriors of large mixtures on FP64 SIMT (bit-exact gamma)
  bool cap_boost = false;  // plan the maximal survivor / orientation capacities (capacity retry of single frames)
  bool tiny_caps = false;  // debug bit 5: tiny batch capacities, so ordinary frames exercise the capacity retry
  // A multi-device context (cdvz_gpu_create_multi) owns one single-device
  // context per device and shards host batches across them.
  std::vector<std::unique_ptr<cdvz_gpu_ctx>> shards;

  static constexpr int kLanes = 2;  // chunks in flight (each lane: its own streams and batch buffers; 4 measured no faster)
  Lane lanes[kLanes];
  int last_lane = 0;
  // Staging of one host-frame call (encode_batch*): device input / output
  // slots, pinned container slots and the per-chunk "containers are in host
  // memory" events. Two of them, so a submitted call can be in flight while
  // the next one is enqueued (cdvz_gpu_encode_batch_submit / _wait).
  struct HostSlot {
    DeviceBuffer stage_in, stage_out, stage_len;
    uint8_t* pin_out = nullptr;    // pinned container slots (D2H target)
    uint32_t* pin_len = nullptr;
    int* pin_status = nullptr;     // per-frame device status (2 data error, 4 capacity, 8 unsupported scale)
    size_t pin_out_bytes = 0, pin_len_count = 0;
    std::vector<cudaEvent_t> out_ev;
    std::vector<int> cb;           // chunk boundaries of the call in flight
    bool ramp = true;              // geometric chunk ramp (one call at a time); full chunks when streaming
    // the call in flight (submit -> wait)
    bool busy = false;
    unsigned long long ticket = 0;
    const uint8_t* pixels = nullptr;
    int width = 0, height = 0, count = 0, mode_id = 0, max_side = 0, kind = 1;
    size_t stride = 0, out_cap = 0;
    uint8_t* out = nullptr;
    size_t* offsets = nullptr;
    int* status = nullptr;

    void ensure_pinned_out(size_t bytes, size_t count_) {
      if (bytes > pin_out_bytes) {
        if (pin_out) cudaFreeHost(pin_out);
        pin_out = nullptr;
        CDVZ_CUDA_CHECK(cudaMallocHost(&pin_out, bytes));
        pin_out_bytes = bytes;
      }
      if (count_ > pin_len_count) {
        if (pin_len) cudaFreeHost(pin_len);
        if (pin_status) cudaFreeHost(pin_status);
        pin_len = nullptr;
        pin_status = nullptr;
        CDVZ_CUDA_CHECK(cudaMallocHost(&pin_len, count_ * sizeof(uint32_t)));
        CDVZ_CUDA_CHECK(cudaMallocHost(&pin_status, count_ * sizeof(int)));
        pin_len_count = count_;
      }
    }
    void release() {
      stage_in.release();
      stage_out.release();
      stage_len.release();
      if (pin_out) cudaFreeHost(pin_out);
      if (pin_len) cudaFreeHost(pin_len);
      if (pin_status) cudaFreeHost(pin_status);
      pin_out = nullptr;
      pin_len = nullptr;
      pin_status = nullptr;
      pin_out_bytes = pin_len_count = 0;
      for (auto& e : out_ev) cudaEventDestroy(e);
      out_ev.clear();
    }
  };
  HostSlot hslot[2];
  unsigned long long next_ticket = 1;
  struct Finished {
    unsigned long long ticket;
    int rc;
    std::string err;
  };
  std::vector<Finished> finished;  // submitted calls finished before their wait (result held for it)
  // A multi-device context's submitted calls: each shard's share runs through
  // that shard's own submit / wait (two in flight per shard), and the wait
  // gathers the shards' containers in frame order.
  struct MultiCall {
    unsigned long long ticket = 0;
    std::vector<uint64_t> shard_ticket;
    std::vector<int> start;
    std::vector<std::vector<size_t>> off;
    uint8_t* out = nullptr;
    size_t out_cap = 0;
    size_t* offsets = nullptr;
    int* status = nullptr;
    size_t slot = 0;
  };
  std::vector<MultiCall> multi_calls;
  int last_frames = 0, last_mode = -1;

  cudaEvent_t ev[6] = {};
  cudaEvent_t user_ev[4] = {};
  cudaEvent_t evp[2 * kMaxOctaves] = {};
  // Statistics are folded from each chunk's events lazily (when its lane is
  // reused, or when a caller asks for them), so encode_device returns as soon
  // as its work is enqueued. `stats` is the last call whose chunks have all
  // been folded; `open` holds calls with chunks still pending.
  struct Stats {
    double stage_ms[5] = {0, 0, 0, 0, 0};
    double pyr_ms = 0.0, pyr_bytes = 0.0;
    int chunks = 0;  // chunks not yet folded
  };
  long long call_seq = 0, stats_call = -1;
  std::map<long long, Stats> open;
  Stats stats;
  int launches = 0;  // kernel launches of the last enqueued call (host-side count)

  ~cdvz_gpu_ctx() {
    for (auto& b : model_bufs) b.release();
    for (auto& l : lanes) l.destroy();
    for (auto& h : hslot) h.release();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : evp)
      if (e) cudaEventDestroy(e);
    for (auto& e : user_ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : copy_ev) cudaEventDestroy(e);
    if (copy_st) cudaStreamDestroy(copy_st);
    if (st) cudaStreamDestroy(st);
  }

  template <class T>
  const T* upload(const T* host, size_t n) {
    model_bufs.emplace_back();
    model_bufs.back().ensure(std::max<size_t>(1, n * sizeof(T)));
    CDVZ_CUDA_CHECK(cudaMemcpy(model_bufs.back().p, host, n * sizeof(T), cudaMemcpyHostToDevice));
    return model_bufs.back().as<T>();
  }

  void setup_model() {
    const Bundle& b = bundle;
    // Detector constants; taps laid out for the kernel variant that runs them
    // (exact fit for radii 5/5/6/8, zero-padded to radius 8 otherwise).
    const bool exact = b.radius[0] == 5 && b.radius[1] == 5 && b.radius[2] == 6 && b.radius[3] == 8;
    for (int k = 0; k < 4; ++k) {
      if (b.radius[k] > 8) throw UsageError("detector scales need a Gaussian radius <= 8 (sigma <= 2.66)");
      const int R = exact ? b.radius[k] : 8;
      for (int j = 0; j < 2 * kMaxTapRadius + 1; ++j) dc.taps[k][j] = 0.0;
      for (int j = -b.radius[k]; j <= b.radius[k]; ++j) dc.taps[k][j + R] = b.taps[k][std::size_t(j + b.radius[k])];
      dc.radius[k] = b.radius[k];
      dc.sigmas[k] = b.sigmas[std::size_t(k)];
      dc.s2[k] = b.sigmas[std::size_t(k)] * b.sigmas[std::size_t(k)];
      for (int i = 0; i < 4; ++i) dc.beta[k][i] = b.beta[k][i];
    }
    dc.thr = b.response_threshold;
    dc.rho_limit = b.rho_limit;
    dc.s_lo = b.sigmas[0];
    dc.s_hi = b.sigmas[3];
    dc.scr_lo = float(dc.s_lo) - 0.05f;
    dc.scr_hi = float(dc.s_hi) + 0.05f;
    dc.scr_thr = float(b.response_threshold);
    dc.margin = b.margin;
    dc.screen = 1;
    dc.walk = 1;
    dc.blur_unrolled = 0;
    dc.desc_registers = 0;

    for (int c = 0; c < 5; ++c) {
      md.rel_edges[c] = upload(b.relevance[std::size_t(c)].edges.data(), b.relevance[std::size_t(c)].edges.size());
      md.rel_vals[c] = upload(b.relevance[std::size_t(c)].values.data(), b.relevance[std::size_t(c)].values.size());
      md.rel_nb[c] = int(b.relevance[std::size_t(c)].values.size());
    }
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        md.tr[0][i][j] = b.tr_a[i][j];
        md.tr[1][i][j] = b.tr_b[i][j];
      }
    md.tr_scale = b.tr_scale;
    md.t0 = upload(b.t0, 128);
    md.t1 = upload(b.t1, 128);
    md.priority = upload(b.priority, 128);
    md.pca_mean = upload(b.pca_mean, 128);
    md.pca_basis = upload(b.pca_basis.data(), b.pca_basis.size());
    md.nc = b.nc;
    // posteriors_matrix's derived tables (scfv.cpp:146-160), computed once on the host.
    std::vector<double> iv(std::size_t(b.nc) * 32), mv(iv.size()), m2(iv.size()), ln(std::size_t(b.nc));
    for (int i = 0; i < b.nc; ++i) {
      double s = 0.0;
      for (int j = 0; j < 32; ++j) {
        const double sd = b.stds[std::size_t(i) * 32 + j], mu = b.means[std::size_t(i) * 32 + j];
        const double var = sd * sd;
        iv[std::size_t(i) * 32 + j] = 1.0 / var;
        mv[std::size_t(i) * 32 + j] = mu / var;
        m2[std::size_t(i) * 32 + j] = (mu * mu) / var;
        s += std::log(sd);
      }
      ln[std::size_t(i)] = std::log(b.weights[std::size_t(i)]) - s - 16.0 * 1.8378770664093453;
    }
    md.inv_var = upload(iv.data(), iv.size());
    md.m_over_v = upload(mv.data(), mv.size());
    md.m2_over_v = upload(m2.data(), m2.size());
    // Transposed copies for k_posterior's cp.async tile loads, and the
    // ones * (M^2/V)^T column (sum_j 1.0 * m2, j ascending, separately rounded).
    md.ncp = (b.nc + 63) / 64 * 64;
    std::vector<double> ivt(std::size_t(md.ncp) * 32, 0.0), mvt(ivt.size(), 0.0), cst(std::size_t(md.ncp), 0.0);
    for (int i = 0; i < b.nc; ++i) {
      double c = 1.0 * m2[std::size_t(i) * 32];
      for (int j = 1; j < 32; ++j) c = c + 1.0 * m2[std::size_t(i) * 32 + j];
      cst[std::size_t(i)] = c;
      for (int j = 0; j < 32; ++j) {
        ivt[std::size_t(j) * md.ncp + i] = iv[std::size_t(i) * 32 + j];
        mvt[std::size_t(j) * md.ncp + i] = mv[std::size_t(i) * 32 + j];
      }
    }
    md.inv_var_t = upload(ivt.data(), ivt.size());
    md.m_over_v_t = upload(mvt.data(), mvt.size());
    md.cst = upload(cst.data(), cst.size());
    md.log_norm = upload(ln.data(), ln.size());
    md.means = upload(b.means.data(), b.means.size());
    md.stds = upload(b.stds.data(), b.stds.size());
    md.weights = upload(b.weights.data(), b.weights.size());
  }

  // Sizes every per-batch buffer for `frames` frames of prepared size W x H.
  // need_resize: octave 0 reads an f64 plane (pixf) of the prepared size,
  // because the frames are resized or RGB. grey_px: pixels of an
  // original-size grey plane per frame (RGB frames that are also resized), or 0.
  void plan(Lane& L, int W, int H, int frames, bool need_resize, long long grey_px = 0) {
    if (W == L.geo_w && H == L.geo_h && frames <= L.geo_frames && (!need_resize || L.geo_resize) && L.geo_debug == debug &&
        grey_px * frames <= L.geo_grey && L.geo_boost == cap_boost && L.geo_tiny == tiny_caps)
      return;
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(L.sA));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(L.sB));
    L.release();
    Batch nb{};
    nb.W = W;
    nb.H = H;
    int n_oct = 0, w = W, h = H;
    long long pd = 0, bw = 0;
    while (n_oct < bundle.num_octaves && n_oct < kMaxOctaves && w >= 16 && h >= 16) {
      nb.ow[n_oct] = w;
      nb.oh[n_oct] = h;
      for (int k = 0; k < 4; ++k) nb.plane_off[n_oct][k] = pd + (long long)k * w * h;
      pd += 4LL * w * h;
      nb.bm_off[n_oct] = bw;
      bw += ((2LL * w * h + 31) / 32 + 3) & ~3LL;  // 16-byte aligned octave bitmaps (k_merge_octave's uint4 passes)
      ++n_oct;
      w /= 2;
      h /= 2;
    }
    // detect_keypoints would keep halving (scale_space.cpp:304-326): refuse
    // rather than silently drop octaves the reference computes.
    if (n_oct == kMaxOctaves && n_oct < bundle.num_octaves && w >= 16 && h >= 16)
      throw UsageError("the bundle asks for more than " + std::to_string(kMaxOctaves) +
                       " octaves on a raster this large; the GPU kernels support at most " + std::to_string(kMaxOctaves));
    nb.n_oct = n_oct;
    nb.frame_doubles = std::max<long long>(pd, 1);
    nb.bitmap_words = std::max<long long>(bw, 4);
    // Survivor capacities per frame: a synthetic 1080p octave keeps ~1% of its
    // pixels (21k); 1/16 of the prepared raster leaves 6x headroom.
    nb.cap_oct = std::max(32768, int(std::min<long long>(1LL << 26, (long long)W * H / 16)));
    nb.cap_acc = nb.cap_oct;
    nb.select_n = bundle.select_n;
    nb.cap_or = std::max(64, bundle.select_n * 4);
    if (tiny_caps && !cap_boost) {
      nb.cap_oct = nb.cap_acc = 256;
      nb.cap_or = 64;
    }
    if (cap_boost) {
      // Capacity retry: the largest counts the reference can produce. At most
      // two candidates per pixel (two roots of the derivative), the
      // accumulated list is bounded by the sum over octaves, and a point has at
      // most 36 orientation peaks (one per histogram bin).
      long long px_sum = 0;
      for (int o = 0; o < n_oct; ++o) px_sum += (long long)nb.ow[o] * nb.oh[o];
      nb.cap_oct = int(std::min<long long>(1LL << 28, 2LL * W * H + 64));
      nb.cap_acc = int(std::min<long long>(1LL << 28, 2LL * px_sum + 64));
      nb.cap_or = std::max(64, bundle.select_n * 36);
    }
    nb.code_stride = 40;
    nb.nc = bundle.nc;
    const long long F = frames;
    auto alloc = [&](size_t bytes) {
      L.bufs.emplace_back();
      L.bufs.back().ensure(std::max<size_t>(bytes, 16));
      return L.bufs.back().p;
    };
    nb.pyr = static_cast<double*>(alloc(sizeof(double) * F * nb.frame_doubles));
    nb.pixf = need_resize ? static_cast<double*>(alloc(sizeof(double) * F * W * H)) : nullptr;
    L.grey = grey_px ? static_cast<double*>(alloc(sizeof(double) * F * grey_px)) : nullptr;
    nb.raw = static_cast<KP*>(alloc(sizeof(KP) * F * std::max(1, n_oct) * nb.cap_oct));
    nb.raw_count = static_cast<int*>(alloc(sizeof(int) * F * std::max(1, n_oct)));
    nb.oct_count = static_cast<int*>(alloc(sizeof(int) * F * std::max(1, n_oct)));
    nb.bitmap = static_cast<uint32_t*>(alloc(sizeof(uint32_t) * F * nb.bitmap_words));
    nb.bm_prefix = static_cast<int*>(alloc(sizeof(int) * F * nb.bitmap_words));
    nb.merge_cell = merge_cell_px(W, H);
    nb.acc[0] = static_cast<KP*>(alloc(sizeof(KP) * F * nb.cap_acc));
    nb.acc[1] = static_cast<KP*>(alloc(sizeof(KP) * F * nb.cap_acc));
    nb.acc_count = static_cast<int*>(alloc(sizeof(int) * F * 2));
    nb.cur = static_cast<KP*>(alloc(sizeof(KP) * F * nb.cap_acc));
    nb.scratch_idx = static_cast<int*>(alloc(sizeof(int) * F * nb.cap_acc));
    nb.flags = static_cast<uint8_t*>(alloc(F * 2 * nb.cap_acc));
    nb.scratch_d = static_cast<double*>(alloc(sizeof(double) * F * nb.cap_acc));
    nb.status = static_cast<int*>(alloc(sizeof(int) * F));
    nb.sel = static_cast<KP*>(alloc(sizeof(KP) * F * nb.select_n));
    nb.sel_count = static_cast<int*>(alloc(sizeof(int) * F));
    nb.thetas = static_cast<double*>(alloc(sizeof(double) * F * nb.select_n * 36));
    nb.theta_count = static_cast<int*>(alloc(sizeof(int) * F * nb.select_n));
    nb.oriented = static_cast<Oriented*>(alloc(sizeof(Oriented) * F * nb.cap_or));
    nb.or_count = static_cast<int*>(alloc(sizeof(int) * F));
    nb.geo = static_cast<DescGeo*>(alloc(sizeof(DescGeo) * F * nb.cap_or));
    nb.order = static_cast<int*>(alloc(sizeof(int) * F * nb.cap_or));
    {
      // samples per axis = ceil(12 sigma) with sigma <= sigma_3 (roots are
      // clamped to [sigma_0, sigma_3]); larger patches are flagged per frame.
      const int smax = std::min(32, std::max(1, static_cast<int>(std::ceil(12.0 * bundle.sigmas[3]))));
      nb.smp_cap = smax * smax;
    }
    nb.smp = static_cast<double2*>(alloc(sizeof(double2) * F * nb.cap_or * nb.smp_cap));
    nb.smpb = static_cast<uint8_t*>(alloc(size_t(F) * nb.cap_or * 32 * 32));
    nb.desc = static_cast<double*>(alloc(sizeof(double) * F * nb.cap_or * 128));
    nb.codes = static_cast<uint8_t*>(alloc(F * nb.cap_or * nb.code_stride));
    nb.x = static_cast<double*>(alloc(sizeof(double) * F * nb.cap_or * 32));
    nb.gamma = static_cast<double*>(alloc(sizeof(double) * F * nb.cap_or * nb.nc));
    nb.gm = static_cast<double*>(alloc(sizeof(double) * F * nb.nc * 32));
    nb.gv = static_cast<double*>(alloc(sizeof(double) * F * nb.nc * 32));
    nb.mask = static_cast<uint8_t*>(alloc(F * ((nb.nc + 7) / 8)));
    nb.mean_planes = static_cast<uint32_t*>(alloc(sizeof(uint32_t) * F * nb.nc));
    nb.var_planes = static_cast<uint32_t*>(alloc(sizeof(uint32_t) * F * nb.nc));
    nb.norms = static_cast<double*>(alloc(sizeof(double) * F * nb.nc));
    CDVZ_CUDA_CHECK(cudaMemset(nb.raw_count, 0, sizeof(int) * F * std::max(1, n_oct)));
    CDVZ_CUDA_CHECK(cudaMemset(nb.bitmap, 0, sizeof(uint32_t) * F * nb.bitmap_words));
    CDVZ_CUDA_CHECK(cudaMemset(nb.acc_count, 0, sizeof(int) * F * 2));
    if (debug) L.dbg_oct.ensure(sizeof(KP) * F * std::max(1, n_oct) * nb.cap_acc);
    // TMA views of the pyramid for k_detect: needs 16-byte row strides (even
    // widths); other sizes use the plain load path.
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    for (int o = 0; o < n_oct; ++o) {
      L.tmap_ok[o] = false;
      if (!encode || (nb.ow[o] & 1) || tma_disabled) continue;
      const cuuint64_t dims[4] = {cuuint64_t(nb.ow[o]), cuuint64_t(nb.oh[o]), 4, cuuint64_t(frames)};
      const cuuint64_t strides[3] = {cuuint64_t(nb.ow[o]) * 8, cuuint64_t(nb.ow[o]) * nb.oh[o] * 8,
                                     cuuint64_t(nb.frame_doubles) * 8};
      const cuuint32_t box[4] = {68, 20, 4, 1}, estr[4] = {1, 1, 1, 1};
      const CUresult r = encode(&L.tmap[o], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, nb.pyr + nb.plane_off[o][0], dims, strides,
                                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const cuuint32_t wbox[4] = {34, 2, 4, 1};
      const CUresult rw = encode(&L.wmap[o], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, nb.pyr + nb.plane_off[o][0], dims, strides,
                                 wbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      L.tmap_ok[o] = (r == CUDA_SUCCESS) && (rw == CUDA_SUCCESS);
    }
    L.bt = nb;
    L.geo_w = W;
    L.geo_h = H;
    L.geo_frames = frames;
    L.geo_resize = need_resize;
    L.geo_grey = grey_px * F;
    L.geo_debug = debug;
    L.geo_boost = cap_boost;
    L.geo_tiny = tiny_caps;
  }

  EncodeConst encode_const(int mode_id) const {
    const Mode& m = mode_by_id(mode_id);
    const Budget bu = budget_for(m, bundle.nc);
    EncodeConst ec{};
    ec.mode_id = m.id;
    ec.elements = m.elements;
    ec.variance = m.variance ? 1 : 0;
    ec.k_select = bu.k;
    ec.max_codes = int(bu.max_codes);
    ec.code_bytes = int(bu.code_bytes);
    ec.mask_bytes = (bundle.nc + 7) / 8;
    ec.global_bytes = int(bu.global_bytes);
    ec.slot_bytes = int(m.budget + 28);
    ec.model_crc = bundle.model_crc;
    ec.post_dmma = post_simt ? 0 : 1;
    return ec;
  }

  // Folds a finished chunk's events into its call's statistics (blocks until
  // the chunk is done). Stage labels follow the reference's time_stage calls
  // (pipeline.cpp:19-94): detection, selection, description (orientation +
  // description), compression (k_compress: transform + ternary + location
  // quantisers, pipeline.cpp:37-50), aggregation (PCA + posteriors + Fisher +
  // SCFV coding). The container pack follows, outside the labels, as
  // serialize_container is outside encode_image.
  // CDVZ_TRACE=1: each collected chunk prints its lane, call and device
  // start / end times (ms after the context's first call) to stderr.
  cudaEvent_t trace_base = nullptr;
  bool trace = std::getenv("CDVZ_TRACE") != nullptr;
  void collect(Lane& L) {
    if (!L.pending) return;
    CDVZ_CUDA_CHECK(cudaEventSynchronize(L.done));
    if (trace && trace_base) {
      float a = 0.f, b = 0.f, c = 0.f;
      cudaEventElapsedTime(&a, trace_base, L.start);
      cudaEventElapsedTime(&b, trace_base, L.stage[1]);
      cudaEventElapsedTime(&c, trace_base, L.stage[5]);
      fprintf(stderr, "trace lane %d call %lld start %.3f detect_end %.3f agg_end %.3f\n", int(&L - lanes), L.pending_call,
              a, b, c);
    }
    Stats& st_ = open[L.pending_call];
    float t[5];
    cudaEventElapsedTime(&t[0], L.start, L.stage[1]);
    cudaEventElapsedTime(&t[1], L.stage[1], L.stage[2]);
    cudaEventElapsedTime(&t[2], L.stage[2], L.stage[3]);
    cudaEventElapsedTime(&t[3], L.stage[3], L.stage[4]);
    cudaEventElapsedTime(&t[4], L.stage[4], L.stage[5]);
    for (int i = 0; i < 5; ++i) st_.stage_ms[i] += t[i];
    for (int o = 0; o < L.pending_oct; ++o) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, L.blur[2 * o], L.blur[2 * o + 1]);
      cudaEventElapsedTime(&b, L.det[2 * o], L.det[2 * o + 1]);
      st_.pyr_ms += a + b;  // kernel time of the pair (they may overlap: conservative)
    }
    st_.pyr_bytes += L.pending_bytes;
    L.pending = false;
    if (--st_.chunks == 0) {
      if (L.pending_call > stats_call) {
        stats = st_;
        stats_call = L.pending_call;
      }
      open.erase(L.pending_call);
    }
  }
  void collect_all() {
    for (auto& l : lanes) collect(l);
  }

  // Runs the whole pipeline for `frames` device-resident frames (u8) of size
  // w x h and writes containers into fixed slots of d_out. Ordered after
  // everything already enqueued on the context stream; the context stream
  // waits for the result.
  // With host pointers (h_pix / h_out / h_len), the frames are copied in on a
  // dedicated copy stream ahead of the kernels and each chunk's containers are
  // copied out on its describe stream, overlapping the other lane's kernels.
  // kind: 1 = grey bytes (PGM), 3 = interleaved RGB bytes (PPM), whose
  // grey plane is formed on the device first, 8 = f64 grey values (the
  // reference's GrayImage), validated on the device; `stride` and `h_stride`
  // are in bytes. h_status receives each frame's device status bits.
  void run(const uint8_t* d_pix, int w, int h, long long stride, int frames, int mode_id, int max_side, uint8_t* d_out,
           uint32_t* d_len, const uint8_t* h_pix = nullptr, size_t h_stride = 0, uint8_t* h_out = nullptr,
           uint32_t* h_len = nullptr, int kind = 1, const std::function<void(int, int)>& on_chunk = nullptr,
           int* h_status = nullptr, HostSlot* hs = nullptr) {
    if (w < 8 || h < 8) throw DataError("image smaller than 8 px per side");
    int W, H;
    prepared_dims(w, h, max_side, W, H);
    const bool resize = (W != w || H != h);
    const bool rgb = kind == 3;
    const bool f64 = kind == 8;
    const int channels = rgb ? 3 : 1;
    const size_t elem = f64 ? sizeof(double) : 1;
    if (f64 && stride != (long long)w * 8) throw UsageError("f64 frames must be packed on the device (stride = 8 * width)");
    const bool f64_base = resize || rgb || f64;  // octave 0 reads the f64 plane pixf
    EncodeConst ec = encode_const(mode_id);
    ec.cx = (W - 1) / 2.0;
    ec.cy = (H - 1) / 2.0;
    ec.half_diag = 0.5 * std::hypot(static_cast<double>(W - 1), static_cast<double>(H - 1));
    ec.log2_range = std::log2(64.0 / 0.5);
    int per = std::min(frames, max_batch);
    {
      // Each lane holds its chunk's pyramid (4 levels x 4/3 of the prepared
      // raster, f64), the f64 base planes, the survivor lists (raw per octave,
      // accumulated x2, current) and ~8 MB of descriptor buffers per frame:
      // keep a lane under 35% of the device memory (VGA ~30 MB per frame, a
      // 4K frame ~600 MB).
      if (!device_mem) {
        size_t free_b = 0;
        CDVZ_CUDA_CHECK(cudaMemGetInfo(&free_b, &device_mem));
      }
      const double px = double(W) * H;
      const double cap = std::max(32768.0, px / 16.0);  // survivor capacity (plan())
      const double per_frame = 8.0 * (4.0 * px * 4.0 / 3.0 + (resize || channels == 3 ? px : 0.0) +
                                      (channels == 3 && resize ? double(w) * h : 0.0)) +
                               cap * (64.0 * 7.0 + 14.0) + 8e6;
      per = std::min(per, std::max(1, int(0.35 * double(device_mem) / per_frame)));
    }
    // Host frames much larger than the prepared raster (e.g. 1080p -> 640x360)
    // make the copy the long pole: at least four chunks per call, so each
    // chunk's copy overlaps the previous chunk's kernels.
    if (h_pix && double(w) * h * channels > 2.0 * double(W) * H) per = std::min(per, std::max(32, (frames + 3) / 4));
    // Chunk boundaries. With host frames the chunks ramp up geometrically
    // from 1/16 of a full chunk (1/16, 1/8, 1/4, 1/2, 1, 1, ...): the copies
    // are queued back to back, so the kernels start after the first short
    // copy and each later copy lands while the earlier chunks compute; the
    // last chunk is the remainder, so the call's unoverlapped tail is short.
    // (Round 1 used one 1/16 lead chunk then full chunks: the second chunk's
    // copy — 3 ms for 512 VGA frames — was exposed.)
    std::vector<int> cb{0};
    static const std::vector<int> chunk_env = [] {  // CDVZ_CHUNKS="32,64,...": schedule experiments
      std::vector<int> v;
      if (const char* e = std::getenv("CDVZ_CHUNKS"))
        for (const char* q = e; *q;) {
          char* end = nullptr;
          const long x = std::strtol(q, &end, 10);
          if (end == q) break;
          if (x > 0) v.push_back(int(x));
          q = *end ? end + 1 : end;
        }
      return v;
    }();
    if (h_pix && !chunk_env.empty()) {
      for (size_t k = 0; cb.back() < frames; ++k)
        cb.push_back(std::min(frames, cb.back() + std::min(per, chunk_env[std::min(k, chunk_env.size() - 1)])));
    } else if (h_pix && frames >= 32 && (!hs || hs->ramp)) {
      int c = std::max(1, per / 16);
      while (cb.back() < frames) {
        cb.push_back(std::min(frames, cb.back() + c));
        c = std::min(per, 2 * c);
      }
    } else {
      while (cb.back() < frames) cb.push_back(std::min(frames, cb.back() + per));
    }
    const int chunks = int(cb.size()) - 1;
    const int n_lanes = serial ? 1 : kLanes;
    const long long call = ++call_seq;
    open[call].chunks = chunks;  // folded one by one as lanes are collected
    // Lanes rotate across calls too, so back-to-back asynchronous calls
    // (encode_device) overlap one call's tail with the next call's head.
    const int lane0 = serial ? 0 : next_lane;
    for (int l = 0; l < std::min(chunks, n_lanes); ++l) {
      Lane& L = lanes[(lane0 + l) % kLanes];
      if (!L.sA) L.init();
      plan(L, W, H, per, resize || rgb, rgb && resize ? (long long)w * h : 0);
    }
    launches = 0;
    if (trace && !trace_base) {
      CDVZ_CUDA_CHECK(cudaEventCreate(&trace_base));
      CDVZ_CUDA_CHECK(cudaEventRecord(trace_base, st));
    }
    CDVZ_CUDA_CHECK(cudaEventRecord(ev[0], st));  // everything before this call
    // Host frames: every chunk's copy is queued up front on the copy stream
    // (back to back at full link bandwidth); a chunk's kernels wait only for
    // its own copy, so only the first chunk's copy is exposed.
    if (h_pix) {
      if (!copy_st) CDVZ_CUDA_CHECK(cudaStreamCreateWithFlags(&copy_st, cudaStreamNonBlocking));
      while (int(copy_ev.size()) < chunks) {
        cudaEvent_t e;
        CDVZ_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        copy_ev.push_back(e);
      }
      // Host frames go into the call's own staging slot, free once its
      // previous call was waited for: the copies need not wait for earlier
      // work on the context stream, so they overlap the previous call's
      // kernels (a submitted stream of batches keeps the device busy).
      const size_t row_bytes = size_t(w) * channels * elem;
      const bool contiguous = size_t(stride) == row_bytes && h_stride == row_bytes;
      for (int c = 0; c < chunks; ++c) {
        const int base = cb[size_t(c)], nf = cb[size_t(c) + 1] - base;
        uint8_t* dst = const_cast<uint8_t*>(d_pix) + (long long)base * h * stride;
        const uint8_t* src = h_pix + size_t(base) * h * h_stride;
        if (contiguous)  // one linear transfer (a 2-D copy of 640-byte rows runs well below the link rate)
          CDVZ_CUDA_CHECK(cudaMemcpyAsync(dst, src, row_bytes * h * nf, cudaMemcpyHostToDevice, copy_st));
        else
          CDVZ_CUDA_CHECK(cudaMemcpy2DAsync(dst, size_t(stride), src, h_stride, row_bytes, size_t(h) * nf,
                                            cudaMemcpyHostToDevice, copy_st));
        CDVZ_CUDA_CHECK(cudaEventRecord(copy_ev[size_t(c)], copy_st));
      }
    }
    for (int c = 0; c < chunks; ++c) {
      NvtxRange nv("cdvz chunk enqueue");
      const int base = cb[size_t(c)];
      const int nf = cb[size_t(c) + 1] - base;
      Lane& L = lanes[serial ? 0 : (lane0 + c) % kLanes];
      collect(L);
      // Serial mode (debug bit 2): one stream per lane, so kernels never
      // overlap and their event times are standalone (bench roofline).
      const cudaStream_t sB = serial ? L.sA : L.sB;  // the lane's previous chunk (c - 2) must be done before its buffers are reused
      Batch b = L.bt;
      b.nframes = nf;
      b.pix8 = d_pix + (long long)base * h * stride;
      b.stride8 = stride;
      b.frame_bytes8 = (long long)h * stride;
      if (!h_pix) {  // device frames: ordered after everything already enqueued on the context stream
        CDVZ_CUDA_CHECK(cudaStreamWaitEvent(L.sA, ev[0], 0));
        CDVZ_CUDA_CHECK(cudaStreamWaitEvent(sB, ev[0], 0));
      }
      if (h_pix) CDVZ_CUDA_CHECK(cudaStreamWaitEvent(L.sA, copy_ev[size_t(c)], 0));
      CDVZ_CUDA_CHECK(cudaEventRecord(L.start, L.sA));
      CDVZ_CUDA_CHECK(cudaMemsetAsync(b.status, 0, sizeof(int) * nf, L.sA));
      if (f64) {  // validate (image.cpp:46-51), then resize_max_side on the caller's grey plane
        double* src = reinterpret_cast<double*>(const_cast<uint8_t*>(b.pix8));
        CDVZ_CUDA_CHECK(launch_validate_f64(src, w, h, nf, b.status, L.sA));
        launches += 2;
        if (resize) {
          CDVZ_CUDA_CHECK(launch_resize_f64(src, w, h, const_cast<double*>(b.pixf), W, H, nf, L.sA));
          ++launches;
        } else {
          b.pixf = src;  // octave 0 reads the validated plane in place
        }
      } else if (rgb) {  // load_image's PPM branch, then resize_max_side on the grey plane
        double* grey = resize ? L.grey : const_cast<double*>(b.pixf);
        CDVZ_CUDA_CHECK(launch_grey_rgb(b.pix8, stride, b.frame_bytes8, w, h, grey, nf, L.sA));
        ++launches;
        if (resize) {
          CDVZ_CUDA_CHECK(launch_resize_f64(grey, w, h, const_cast<double*>(b.pixf), W, H, nf, L.sA));
          ++launches;
        }
      } else if (resize) {
        CDVZ_CUDA_CHECK(launch_resize(b.pix8, stride, b.frame_bytes8, w, h, const_cast<double*>(b.pixf), W, H, nf, L.sA));
        ++launches;
      }
      double bytes = 0.0;
      for (int o = 0; o < b.n_oct; ++o) {
        const int src = o == 0 ? (f64_base ? 1 : 0) : 2;
        CDVZ_CUDA_CHECK(cudaEventRecord(L.blur[2 * o], L.sA));
        CDVZ_CUDA_CHECK(launch_octave(b, dc, o, src, L.sA));
        CDVZ_CUDA_CHECK(cudaEventRecord(L.blur[2 * o + 1], L.sA));
        CDVZ_CUDA_CHECK(cudaStreamWaitEvent(sB, L.blur[2 * o + 1], 0));
        CDVZ_CUDA_CHECK(cudaEventRecord(L.det[2 * o], sB));
        CDVZ_CUDA_CHECK(launch_detect(b, dc, o, L.tmap_ok[o] ? &L.tmap[o] : nullptr, L.tmap_ok[o] ? &L.wmap[o] : nullptr, sB));
        CDVZ_CUDA_CHECK(cudaEventRecord(L.det[2 * o + 1], sB));
        CDVZ_CUDA_CHECK(launch_merge(b, o, sB));
        launches += 3;
        if (debug) {
          const KP* srcl = (o == 0) ? b.acc[0] : b.cur;
          CDVZ_CUDA_CHECK(cudaMemcpyAsync(L.dbg_oct.as<KP>() + (long long)o * b.cap_acc * L.geo_frames, srcl,
                                          sizeof(KP) * (long long)nf * b.cap_acc, cudaMemcpyDeviceToDevice, sB));
        }
        // Algorithmic bytes of the split octave pair: K1a reads
        // the base (1 B/px u8 at octave 0, 8 B/px f64 above) and writes 4 G
        // levels (32 B/px); K1b reads the 4 G levels of its window back.
        const double px = double(b.ow[o]) * b.oh[o];
        const double in_b = (o == 0) ? (f64_base ? 8.0 : 1.0) : 8.0;
        const int ww = std::max(0, b.ow[o] - 2 * dc.margin), hh = std::max(0, b.oh[o] - 2 * dc.margin);
        bytes += double(nf) * (px * (in_b + 32.0) + 32.0 * ww * hh);
      }
      // Stream B also waits for the last blur (octaves whose window is empty
      // launch no extrema kernel) before describing from the pyramid.
      CDVZ_CUDA_CHECK(cudaStreamWaitEvent(sB, b.n_oct ? L.blur[2 * b.n_oct - 1] : L.start, 0));
      CDVZ_CUDA_CHECK(cudaEventRecord(L.stage[1], sB));
      CDVZ_CUDA_CHECK(launch_select(b, md, ec, sB));
      CDVZ_CUDA_CHECK(cudaEventRecord(L.stage[2], sB));
      CDVZ_CUDA_CHECK(launch_describe(b, dc, sB));
      CDVZ_CUDA_CHECK(cudaEventRecord(L.stage[3], sB));
      CDVZ_CUDA_CHECK(launch_compress(b, md, ec, sB));
      CDVZ_CUDA_CHECK(cudaEventRecord(L.stage[4], sB));
      // The container pack runs after the aggregation event: the reference
      // serialises outside encode_image's timed stages.
      CDVZ_CUDA_CHECK(launch_scfv_pack(b, md, ec, d_out + (long long)base * ec.slot_bytes, d_len + base, sB, L.stage[5]));
      if (h_out) {
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(h_out + size_t(base) * ec.slot_bytes, d_out + size_t(base) * ec.slot_bytes,
                                        size_t(nf) * ec.slot_bytes, cudaMemcpyDeviceToHost, sB));
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(h_len + base, d_len + base, sizeof(uint32_t) * nf, cudaMemcpyDeviceToHost, sB));
        if (h_status)
          CDVZ_CUDA_CHECK(cudaMemcpyAsync(h_status + base, b.status, sizeof(int) * nf, cudaMemcpyDeviceToHost, sB));
        std::vector<cudaEvent_t>& oev = hs->out_ev;
        while (int(oev.size()) <= c) {
          cudaEvent_t e;
          CDVZ_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          oev.push_back(e);
        }
        CDVZ_CUDA_CHECK(cudaEventRecord(oev[size_t(c)], sB));
      }
      CDVZ_CUDA_CHECK(cudaEventRecord(L.done, sB));
      // The next chunk on this lane's stream A must not overwrite the pyramid
      // before stream B is done with it.
      CDVZ_CUDA_CHECK(cudaStreamWaitEvent(L.sA, L.done, 0));
      launches += 1 + 6 + 1 + 5;  // k_select; k_orient, k_expand, k_geometry, k_order, k_sample, k_describe; k_compress; SCFV + pack
      L.pending = true;
      L.pending_call = call;
      L.pending_oct = b.n_oct;
      L.pending_bytes = bytes;
      last_lane = serial ? 0 : (lane0 + c) % kLanes;
    }
    if (!serial) next_lane = (lane0 + chunks) % kLanes;
    // Host outputs: hand each chunk's containers to the caller in frame order
    // as soon as they land, while later chunks are still on the device.
    if (h_out) hs->cb = cb;
    if (h_out && on_chunk)
      for (int c = 0; c < chunks; ++c) {
        CDVZ_CUDA_CHECK(cudaEventSynchronize(hs->out_ev[size_t(c)]));
        on_chunk(cb[size_t(c)], cb[size_t(c) + 1] - cb[size_t(c)]);
      }
    for (int l = 0; l < kLanes; ++l)
      if (lanes[l].pending) CDVZ_CUDA_CHECK(cudaStreamWaitEvent(st, lanes[l].done, 0));
    // No collect() here: the call returns once its work is enqueued.
    last_frames = cb[size_t(chunks)] - cb[size_t(chunks) - 1];
    last_mode = mode_id;
  }
};

namespace {

template <class F>
int guarded(cdvz_gpu_ctx* ctx, F&& f) {
  try {
    f();
    if (ctx) ctx->err.clear();
    return CDVZ_GPU_OK;
  } catch (const UsageError& e) {
    (ctx ? ctx->err : g_create_error) = e.what();
    return CDVZ_GPU_USAGE;
  } catch (const DataError& e) {
    (ctx ? ctx->err : g_create_error) = e.what();
    return CDVZ_GPU_DATA;
  } catch (const std::exception& e) {
    (ctx ? ctx->err : g_create_error) = e.what();
    return CDVZ_GPU_INTERNAL;
  }
}

// Entry points that act on one device's memory or stream.
void require_single(const cdvz_gpu_ctx* ctx) {
  if (!ctx) throw UsageError("null context");
  if (!ctx->shards.empty()) throw UsageError("this call acts on one device: use a single-device context");
}

}  // namespace

extern "C" {

int cdvz_gpu_create(const char* bundle_text, size_t bundle_len, int device, int max_batch, cdvz_gpu_ctx** out_ctx) {
  return guarded(nullptr, [&] {
    if (!out_ctx || !bundle_text) throw UsageError("null argument");
    *out_ctx = nullptr;
    parse_bundle(std::string(bundle_text, bundle_len));  // data errors before device errors
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw std::runtime_error("no CUDA device available (the extractor has no CPU fallback)");
    if (device < 0 || device >= ndev) throw UsageError("device index out of range");
    cudaDeviceProp prop{};
    CDVZ_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw std::runtime_error(std::string("the kernels are built for sm_100a only; device is ") + prop.name);
    Bundle parsed = parse_bundle(std::string(bundle_text, bundle_len));
    auto ctx = std::make_unique<cdvz_gpu_ctx>();
    ctx->device = device;
    ctx->max_batch = max_batch > 0 ? max_batch : 256;
    CDVZ_CUDA_CHECK(cudaSetDevice(device));
    CDVZ_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking));
    for (auto& e : ctx->ev) CDVZ_CUDA_CHECK(cudaEventCreate(&e));
    for (auto& e : ctx->evp) CDVZ_CUDA_CHECK(cudaEventCreate(&e));
    ctx->bundle = std::move(parsed);
    ctx->setup_model();
    *out_ctx = ctx.release();
  });
}

int cdvz_gpu_create_multi(const char* bundle_text, size_t bundle_len, const int* devices, int ndev, int max_batch,
                          cdvz_gpu_ctx** out_ctx) {
  return guarded(nullptr, [&] {
    if (!out_ctx || !bundle_text || !devices) throw UsageError("null argument");
    *out_ctx = nullptr;
    if (ndev < 1) throw UsageError("at least one device is required");
    Bundle parsed = parse_bundle(std::string(bundle_text, bundle_len));
    auto ctx = std::make_unique<cdvz_gpu_ctx>();
    ctx->device = devices[0];
    ctx->max_batch = max_batch > 0 ? max_batch : 256;
    ctx->bundle = std::move(parsed);
    for (int d = 0; d < ndev; ++d) {
      cdvz_gpu_ctx* sub = nullptr;
      const int rc = cdvz_gpu_create(bundle_text, bundle_len, devices[d], max_batch, &sub);
      if (rc != CDVZ_GPU_OK) {
        const std::string msg = "device " + std::to_string(devices[d]) + ": " + g_create_error;
        if (rc == CDVZ_GPU_USAGE) throw UsageError(msg);
        if (rc == CDVZ_GPU_DATA) throw DataError(msg);
        throw std::runtime_error(msg);
      }
      ctx->shards.emplace_back(sub);
    }
    *out_ctx = ctx.release();
  });
}

int cdvz_gpu_visible_devices(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int cdvz_gpu_device_count(const cdvz_gpu_ctx* ctx, int* devices, int cap) {
  if (!ctx) return -1;
  const int n = ctx->shards.empty() ? 1 : int(ctx->shards.size());
  for (int d = 0; d < n && devices && d < cap; ++d) devices[d] = ctx->shards.empty() ? ctx->device : ctx->shards[size_t(d)]->device;
  return n;
}

void cdvz_gpu_destroy(cdvz_gpu_ctx* ctx) {
  if (!ctx) return;
  if (ctx->shards.empty()) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->st);
  }
  delete ctx;
}

const char* cdvz_gpu_last_error(const cdvz_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

int cdvz_gpu_bundle_check(const char* bundle_text, size_t bundle_len, uint32_t* model_crc, int* components) {
  return guarded(nullptr, [&] {
    if (!bundle_text) throw UsageError("null argument");
    const Bundle b = parse_bundle(std::string(bundle_text, bundle_len));
    if (model_crc) *model_crc = b.model_crc;
    if (components) *components = b.nc;
  });
}

int cdvz_gpu_event_record(cdvz_gpu_ctx* ctx, int slot) {
  return guarded(ctx, [&] {
    require_single(ctx);
    if (slot < 0 || slot >= 4) throw UsageError("event slot out of range");
    if (!ctx->user_ev[slot]) CDVZ_CUDA_CHECK(cudaEventCreate(&ctx->user_ev[slot]));
    CDVZ_CUDA_CHECK(cudaEventRecord(ctx->user_ev[slot], ctx->st));
  });
}

int cdvz_gpu_event_elapsed(cdvz_gpu_ctx* ctx, int a, int b, double* ms) {
  return guarded(ctx, [&] {
    require_single(ctx);
    if (a < 0 || a >= 4 || b < 0 || b >= 4 || !ctx->user_ev[a] || !ctx->user_ev[b]) throw UsageError("event slot not recorded");
    CDVZ_CUDA_CHECK(cudaEventSynchronize(ctx->user_ev[b]));
    float t = 0.f;
    CDVZ_CUDA_CHECK(cudaEventElapsedTime(&t, ctx->user_ev[a], ctx->user_ev[b]));
    *ms = t;
  });
}

int cdvz_gpu_bundle_info(const cdvz_gpu_ctx* ctx, uint32_t* model_crc, int* components, int* select_n) {
  if (!ctx) return CDVZ_GPU_USAGE;
  if (model_crc) *model_crc = ctx->bundle.model_crc;
  if (components) *components = ctx->bundle.nc;
  if (select_n) *select_n = ctx->bundle.select_n;
  return CDVZ_GPU_OK;
}

size_t cdvz_gpu_container_slot(int mode_id) {
  try {
    return mode_by_id(mode_id).budget + 28;
  } catch (...) {
    return 0;
  }
}

int cdvz_gpu_set_debug(cdvz_gpu_ctx* ctx, int on) {
  if (!ctx) return CDVZ_GPU_USAGE;
  for (auto& sh : ctx->shards) cdvz_gpu_set_debug(sh.get(), on);
  ctx->debug = (on & 1) != 0;
  ctx->dc.screen = (on & 2) ? 0 : 1;
  ctx->serial = (on & 4) != 0;
  ctx->dc.walk = (on & 16) ? 0 : 1;
  ctx->tiny_caps = (on & 32) != 0;
  ctx->dc.blur_unrolled = (on & 64) ? 1 : 0;
  ctx->post_simt = (on & 128) != 0;
  ctx->dc.desc_registers = (on & 256) ? 1 : 0;
  if (ctx->tma_disabled != ((on & 8) != 0)) {
    ctx->tma_disabled = (on & 8) != 0;
    for (auto& l : ctx->lanes) l.geo_w = 0;  // rebuild the tensor maps
  }
  return CDVZ_GPU_OK;
}

int cdvz_gpu_encode_device(cdvz_gpu_ctx* ctx, const uint8_t* d_pixels, int width, int height, size_t stride, int count,
                           int mode_id, int max_side, uint8_t* d_out, uint32_t* d_lengths) {
  return guarded(ctx, [&] {
    if (!ctx) throw UsageError("null context");
    if (!ctx->shards.empty()) throw UsageError("device-resident frames belong to one device: use a single-device context");
    if (count < 0) throw UsageError("negative frame count");
    if (count == 0) return;
    mode_by_id(mode_id);
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    ctx->run(d_pixels, width, height, (long long)stride, count, mode_id, max_side, d_out, d_lengths);
  });
}

int cdvz_gpu_trim(cdvz_gpu_ctx* ctx) {
  return guarded(ctx, [&] {
    if (!ctx) throw UsageError("null context");
    if (!ctx->shards.empty()) {
      for (auto& sh : ctx->shards)
        if (cdvz_gpu_trim(sh.get()) != CDVZ_GPU_OK) throw std::runtime_error(sh->err);
      return;
    }
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
    for (auto& l : ctx->lanes) {
      if (l.sA) CDVZ_CUDA_CHECK(cudaStreamSynchronize(l.sA));
      if (l.sB) CDVZ_CUDA_CHECK(cudaStreamSynchronize(l.sB));
      l.release();
    }
    for (auto& h : ctx->hslot) {
      if (h.busy) throw UsageError("a submitted batch is in flight: wait for it before trimming");
      h.stage_in.release();
      h.stage_out.release();
      h.stage_len.release();
    }
  });
}

int cdvz_gpu_sync(cdvz_gpu_ctx* ctx) {
  return guarded(ctx, [&] {
    if (!ctx) throw UsageError("null context");
    for (auto& sh : ctx->shards)
      if (cdvz_gpu_sync(sh.get()) != CDVZ_GPU_OK) throw std::runtime_error(sh->err);
    if (ctx->shards.empty()) {
      CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
      CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
    }
  });
}

}  // extern "C"

namespace {

int encode_host_batch(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride, int count,
                      int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets, int* status, int kind);

// Frame-sharded host batch on a multi-device context: contiguous frame ranges,
// one host thread per device (the GPU analogue of the reference's
// run_indexed fan-out, parallel.cpp:40-78), containers gathered in frame
// order. The lowest-index failing device's error wins, as in run_indexed.
// Gathers per-shard container regions (shard d wrote frames start[d] ..
// start[d+1] with local offsets off[d]) into `out` in frame order.
void gather_multi(const std::vector<int>& start, const std::vector<std::vector<size_t>>& off, bool in_place,
                  const std::vector<std::vector<uint8_t>>& scratch, uint8_t* out, size_t out_cap, size_t* offsets,
                  int* status, size_t slot) {
  const int nd = int(start.size()) - 1;
  // Gather in frame order. In place, shard d's bytes move left (to the end of
  // shard d-1's), so a forward memmove per shard is safe.
  size_t written = 0;
  offsets[0] = 0;
  for (int d = 0; d < nd; ++d) {
    const int n = start[size_t(d) + 1] - start[size_t(d)];
    const size_t bytes = off[size_t(d)][size_t(n)];
    const uint8_t* src = in_place ? out + size_t(start[size_t(d)]) * slot : scratch[size_t(d)].data();
    if (!in_place && written + bytes > out_cap) {
      // Frame-level overflow accounting, as the single-device path does it.
      for (int i = 0; i < n; ++i) {
        const size_t len = off[size_t(d)][size_t(i) + 1] - off[size_t(d)][size_t(i)];
        const int fi = start[size_t(d)] + i;
        if (status[fi] == CDVZ_GPU_OK) {
          if (written + len > out_cap) {
            status[fi] = CDVZ_GPU_USAGE;
          } else {
            std::memcpy(out + written, src + off[size_t(d)][size_t(i)], len);
            written += len;
          }
        }
        offsets[fi + 1] = written;
      }
      continue;
    }
    if (bytes && out + written != src) std::memmove(out + written, src, bytes);
    for (int i = 0; i < n; ++i) offsets[start[size_t(d)] + i + 1] = written + off[size_t(d)][size_t(i) + 1];
    written += bytes;
  }
}

void fold_multi_stats(cdvz_gpu_ctx* ctx) {
  cdvz_gpu_ctx::Stats sum;
  int launches = 0;
  for (auto& sh : ctx->shards) {
    for (int i = 0; i < 5; ++i) sum.stage_ms[i] += sh->stats.stage_ms[i];
    sum.pyr_ms += sh->stats.pyr_ms;
    sum.pyr_bytes += sh->stats.pyr_bytes;
    launches += sh->launches;
  }
  ctx->stats = sum;
  ctx->launches = launches;
}

void encode_multi(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride, int count,
                  int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets, int* status, int kind) {
  const int nd = int(ctx->shards.size());
  const size_t slot = mode_by_id(mode_id).budget + 28;
  std::vector<int> start(static_cast<size_t>(nd) + 1);
  for (int d = 0; d <= nd; ++d) start[size_t(d)] = int((long long)count * d / nd);
  // Each shard writes into its own region: in place in `out` when the caller
  // left room for every frame at full slot size, else in a scratch buffer.
  const bool in_place = out_cap >= size_t(count) * slot;
  std::vector<std::vector<uint8_t>> scratch(in_place ? 0 : static_cast<size_t>(nd));
  std::vector<std::vector<size_t>> off(static_cast<size_t>(nd));
  std::vector<int> rc(static_cast<size_t>(nd), int(CDVZ_GPU_OK));
  std::vector<std::thread> th;
  for (int d = 0; d < nd; ++d) {
    const int n = start[size_t(d) + 1] - start[size_t(d)];
    off[size_t(d)].assign(size_t(n) + 1, 0);
    uint8_t* region = nullptr;
    if (in_place) {
      region = out + size_t(start[size_t(d)]) * slot;
    } else {
      scratch[size_t(d)].resize(std::max<size_t>(1, size_t(n) * slot));
      region = scratch[size_t(d)].data();
    }
    const uint8_t* src = pixels + size_t(start[size_t(d)]) * height * stride;
    th.emplace_back([&, d, n, region, src] {
      if (n == 0) return;
      NvtxRange r("cdvz_gpu shard");
      rc[size_t(d)] = encode_host_batch(ctx->shards[size_t(d)].get(), src, width, height, stride, n, mode_id, max_side,
                                        region, size_t(n) * slot, off[size_t(d)].data(), status + start[size_t(d)], kind);
    });
  }
  for (auto& t : th) t.join();
  for (int d = 0; d < nd; ++d)
    if (rc[size_t(d)] != CDVZ_GPU_OK) {
      const std::string msg = "device " + std::to_string(ctx->shards[size_t(d)]->device) + ": " + ctx->shards[size_t(d)]->err;
      if (rc[size_t(d)] == CDVZ_GPU_USAGE) throw UsageError(msg);
      if (rc[size_t(d)] == CDVZ_GPU_DATA) throw DataError(msg);
      throw std::runtime_error(msg);
    }
  gather_multi(start, off, in_place, scratch, out, out_cap, offsets, status, slot);
  fold_multi_stats(ctx);
}

// Host-frame batch encode of grey (kind 1) or RGB (kind 3) byte rasters, or
// f64 grey rasters (kind 8; `stride` in bytes).
// Frames per host-frame group: bounded so the device staging stays < 4 GB.
int host_group_frames(size_t frame_bytes, int count) {
  return int(std::max<size_t>(1, std::min<size_t>(size_t(count), (size_t(4) << 30) / frame_bytes)));
}

// Enqueues frames [base, base + nf) of the slot's call: the copies, every
// kernel and the container copies back, with no host wait.
void host_begin(cdvz_gpu_ctx* ctx, cdvz_gpu_ctx::HostSlot& hs, int base, int nf) {
  const int channels = hs.kind == 3 ? 3 : 1;
  const size_t elem = hs.kind == 8 ? sizeof(double) : 1;
  const size_t row_bytes = size_t(hs.width) * channels * elem;
  const size_t frame_bytes = row_bytes * hs.height;
  const size_t slot = mode_by_id(hs.mode_id).budget + 28;
  hs.stage_in.ensure(frame_bytes * nf);
  hs.stage_out.ensure(slot * nf);
  hs.stage_len.ensure(sizeof(uint32_t) * nf);
  hs.ensure_pinned_out(slot * nf, nf);
  ctx->run(hs.stage_in.as<uint8_t>(), hs.width, hs.height, (long long)row_bytes, nf, hs.mode_id, hs.max_side,
           hs.stage_out.as<uint8_t>(), hs.stage_len.as<uint32_t>(), hs.pixels + size_t(base) * hs.height * hs.stride,
           hs.stride, hs.pin_out, hs.pin_len, hs.kind, nullptr, hs.pin_status, &hs);
}

// Waits for the group enqueued by host_begin and hands its containers to the
// caller in frame order (chunk by chunk, as they land), with per-frame status;
// frames whose lists overflowed a batch capacity are re-encoded alone with the
// maximal capacities and spliced in. `written` is the caller's output cursor.
// With fold_now false (submitted calls), only this call's chunk events are
// waited on: a later submitted call may already be queued behind it, and its
// statistics are folded lazily (stage_times) instead of draining the device.
void host_finish(cdvz_gpu_ctx* ctx, cdvz_gpu_ctx::HostSlot& hs, int base, int nf, size_t& written,
                 cdvz_gpu_ctx::Stats& acc, int& acc_launches, bool fold_now = true) {
  const size_t slot = mode_by_id(hs.mode_id).budget + 28;
  const int channels = hs.kind == 3 ? 3 : 1;
  const size_t elem = hs.kind == 8 ? sizeof(double) : 1;
  const size_t row_bytes = size_t(hs.width) * channels * elem;
  const size_t frame_bytes = row_bytes * hs.height;
  uint8_t* out = hs.out;
  size_t* offsets = hs.offsets;
  int* status = hs.status;
  auto fold = [&] {
    ctx->collect_all();
    for (int i = 0; i < 5; ++i) acc.stage_ms[i] += ctx->stats.stage_ms[i];
    acc.pyr_ms += ctx->stats.pyr_ms;
    acc.pyr_bytes += ctx->stats.pyr_bytes;
    acc_launches += ctx->launches;
  };
  std::vector<int> retry;                    // frames of this group that overflowed a capacity
  std::vector<size_t> start(size_t(nf), 0);  // byte offset of each written container in `out`
  for (size_t c = 0; c + 1 < hs.cb.size(); ++c) {
    CDVZ_CUDA_CHECK(cudaEventSynchronize(hs.out_ev[c]));
    for (int i = hs.cb[c]; i < hs.cb[c + 1]; ++i) {
      const size_t len = hs.pin_len[size_t(i)];
      const int dev_status = hs.pin_status[size_t(i)];
      const int fi = base + i;
      start[size_t(i)] = written;
      if (len == 0) {
        if (dev_status & 2) {
          status[fi] = CDVZ_GPU_DATA;  // validate(): non-finite or outside [0, 1]
        } else if (dev_status == 4) {
          status[fi] = CDVZ_GPU_OK;    // capacity only: re-encoded below with the maximal capacities
          retry.push_back(i);
        } else {
          status[fi] = CDVZ_GPU_INTERNAL;
        }
      } else if (written + len > hs.out_cap) {
        status[fi] = CDVZ_GPU_USAGE;
      } else {
        std::memcpy(out + written, hs.pin_out + size_t(i) * slot, len);
        written += len;
        status[fi] = CDVZ_GPU_OK;
      }
      offsets[fi + 1] = written;
    }
  }
  if (fold_now) {
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
    fold();
  }
  if (retry.empty()) return;
  // Capacity retry: a frame whose survivor or orientation lists outgrew the
  // batch capacities (adversarial content) is encoded again on its own with
  // the largest counts the reference can produce, so it never fails where
  // the reference succeeds. Its container is then spliced in frame order.
  std::vector<std::vector<uint8_t>> redo(retry.size());
  ctx->cap_boost = true;
  try {
    for (size_t r = 0; r < retry.size(); ++r) {
      const int i = retry[r];
      ctx->run(hs.stage_in.as<uint8_t>() + size_t(i) * frame_bytes, hs.width, hs.height, (long long)row_bytes, 1,
               hs.mode_id, hs.max_side, hs.stage_out.as<uint8_t>(), hs.stage_len.as<uint32_t>(), nullptr, 0, nullptr,
               nullptr, hs.kind);
      CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
      fold();
      uint32_t len = 0;
      int dev_status = 0;
      CDVZ_CUDA_CHECK(cudaMemcpy(&len, hs.stage_len.as<uint32_t>(), sizeof(len), cudaMemcpyDeviceToHost));
      const Lane& L = ctx->lanes[ctx->last_lane];
      CDVZ_CUDA_CHECK(cudaMemcpy(&dev_status, L.bt.status, sizeof(int), cudaMemcpyDeviceToHost));
      if (len == 0) {
        status[base + i] = (dev_status & 2) ? CDVZ_GPU_DATA : CDVZ_GPU_INTERNAL;
        continue;
      }
      redo[r].resize(len);
      CDVZ_CUDA_CHECK(cudaMemcpy(redo[r].data(), hs.stage_out.as<uint8_t>(), len, cudaMemcpyDeviceToHost));
    }
  } catch (...) {
    ctx->cap_boost = false;
    throw;
  }
  ctx->cap_boost = false;
  size_t grow = 0;
  for (const auto& v : redo) grow += v.size();
  if (written + grow > hs.out_cap) {  // no room: the re-encoded frames are reported like any overflow
    for (size_t q = 0; q < retry.size(); ++q)
      if (!redo[q].empty()) status[base + retry[q]] = CDVZ_GPU_USAGE;
    return;
  }
  // Rebuild this group's section back to front: containers only move right.
  size_t end = written + grow;
  size_t r = retry.size();
  for (int i = nf - 1; i >= 0; --i) {
    const int fi = base + i;
    const size_t old_len = size_t(offsets[fi + 1]) - start[size_t(i)];
    const std::vector<uint8_t>* ins = (r > 0 && retry[r - 1] == i) ? &redo[--r] : nullptr;
    const size_t len = ins ? ins->size() : old_len;
    const size_t pos = end - len;
    if (ins) {
      if (len) std::memcpy(out + pos, ins->data(), len);
    } else if (len && pos != start[size_t(i)]) {
      std::memmove(out + pos, out + start[size_t(i)], len);
    }
    offsets[fi + 1] = end;
    end = pos;
  }
  written += grow;
}

// Argument checks shared by the synchronous and the submitted host batch.
// Returns false when there is nothing to enqueue (count 0; frames below 8 px,
// which also throws DataError after filling the per-frame outputs).
bool host_args(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride, int count,
               size_t* offsets, int* status, int kind) {
  const int channels = kind == 3 ? 3 : 1;
  const size_t elem = kind == 8 ? sizeof(double) : 1;
  if (!ctx || (!pixels && count > 0) || !offsets || !status) throw UsageError("null argument");
  if (count < 0) throw UsageError("negative frame count");
  if (stride < size_t(width) * channels * elem) throw UsageError("row stride shorter than a row");
  offsets[0] = 0;
  if (count == 0) return false;
  if (width < 8 || height < 8) {
    for (int i = 0; i < count; ++i) {
      status[i] = CDVZ_GPU_DATA;
      offsets[i + 1] = 0;
    }
    throw DataError("image smaller than 8 px per side");
  }
  return true;
}

void slot_args(cdvz_gpu_ctx::HostSlot& hs, const uint8_t* pixels, int width, int height, size_t stride, int count,
               int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets, int* status, int kind) {
  hs.pixels = pixels;
  hs.width = width;
  hs.height = height;
  hs.stride = stride;
  hs.count = count;
  hs.mode_id = mode_id;
  hs.max_side = max_side;
  hs.out = out;
  hs.out_cap = out_cap;
  hs.offsets = offsets;
  hs.status = status;
  hs.kind = kind;
}

// Host-frame batch encode of grey (kind 1) or RGB (kind 3) byte rasters, or
// f64 grey rasters (kind 8; `stride` in bytes): groups of frames through
// host_begin + host_finish, one after the other.
int encode_host_batch(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride, int count,
                      int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets, int* status, int kind) {
  NvtxRange nv("cdvz_gpu_encode_batch");
  return guarded(ctx, [&] {
    if (!host_args(ctx, pixels, width, height, stride, count, offsets, status, kind)) return;
    mode_by_id(mode_id);
    if (!ctx->shards.empty()) {
      encode_multi(ctx, pixels, width, height, stride, count, mode_id, max_side, out, out_cap, offsets, status, kind);
      return;
    }
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    for (auto& h : ctx->hslot)  // submitted calls finish first (their results stay with their tickets)
      if (h.busy) throw UsageError("a submitted batch is in flight: wait for it before a synchronous call");
    const int channels = kind == 3 ? 3 : 1;
    const size_t elem = kind == 8 ? sizeof(double) : 1;
    const size_t frame_bytes = size_t(width) * channels * elem * height;
    const int group = host_group_frames(frame_bytes, count);
    auto& hs = ctx->hslot[0];
    slot_args(hs, pixels, width, height, stride, count, mode_id, max_side, out, out_cap, offsets, status, kind);
    hs.ramp = true;
    size_t written = 0;
    cdvz_gpu_ctx::Stats acc;
    int acc_launches = 0;
    for (int base = 0; base < count; base += group) {
      const int nf = std::min(group, count - base);
      host_begin(ctx, hs, base, nf);
      host_finish(ctx, hs, base, nf, written, acc, acc_launches);
    }
    ctx->stats = acc;
    ctx->launches = acc_launches;
  });
}

}  // namespace

extern "C" {

// load_image's header parse (proj/src/image.cpp:53-77; read_pnm_token
// :17-36) on an in-memory file.
int cdvz_gpu_pnm_parse(const uint8_t* file, size_t len, int* width, int* height, int* channels, size_t* raster_offset) {
  return guarded(nullptr, [&] {
    if (!file || !width || !height || !channels || !raster_offset) throw UsageError("null argument");
    size_t pos = 0;
    if (len < 2 || file[0] != 'P' || (file[1] != '5' && file[1] != '6'))
      throw DataError("unsupported image format (expected binary PGM/PPM)");
    const bool color = file[1] == '6';
    pos = 2;
    auto token = [&](const char* what) {
      for (;;) {  // whitespace and '#' comments (to the end of the line)
        if (pos >= len) throw DataError(std::string("truncated header while reading ") + what);
        const int c = file[pos];
        if (std::isspace(c)) {
          ++pos;
          continue;
        }
        if (c == '#') {
          while (pos < len && file[pos] != '\n') ++pos;
          if (pos < len) ++pos;
          continue;
        }
        break;
      }
      // operator>>(int): optional sign, then at least one digit, no overflow.
      size_t p = pos;
      bool neg = false;
      if (file[p] == '+' || file[p] == '-') neg = file[p++] == '-';
      long long v = 0;
      size_t digits = 0;
      while (p < len && file[p] >= '0' && file[p] <= '9') {
        v = v * 10 + (file[p++] - '0');
        if (v > 2147483647LL) throw DataError(std::string("invalid header field: ") + what);
        ++digits;
      }
      if (digits == 0 || (neg && v > 0)) throw DataError(std::string("invalid header field: ") + what);
      pos = p;
      return int(v);
    };
    const int w = token("width");
    const int h = token("height");
    const int maxval = token("maxval");
    if (maxval != 255) throw DataError("only maxval 255 is supported");
    if (w < 8 || h < 8) throw DataError("image smaller than 8 px per side");
    ++pos;  // the single whitespace byte before the raster
    const size_t ch = color ? 3 : 1;
    if (pos > len || len - pos < size_t(w) * size_t(h) * ch) throw DataError("truncated raster data");
    *width = w;
    *height = h;
    *channels = int(ch);
    *raster_offset = pos;
  });
}

// Submitted host batches (cdvz_gpu.h): at most two in flight per context, each
// with its own staging slot. A submit that finds both slots taken first
// finishes the older call into its caller's buffers (its wait then returns
// the stored result).
namespace {
void finish_slot(cdvz_gpu_ctx* ctx, cdvz_gpu_ctx::HostSlot& hs) {
  const int rc = guarded(ctx, [&] {
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    size_t written = 0;
    cdvz_gpu_ctx::Stats acc;
    int acc_launches = 0;
    host_finish(ctx, hs, 0, hs.count, written, acc, acc_launches, false);
  });
  ctx->finished.push_back({hs.ticket, rc, rc == CDVZ_GPU_OK ? std::string() : ctx->err});
  hs.busy = false;
  hs.ticket = 0;
}
}  // namespace

// Waits for every shard of the multi-device call multi_calls[i], gathers its
// containers in frame order and drops the record; the call's return code.
static int finish_multi(cdvz_gpu_ctx* ctx, size_t i, std::string& err) {
  cdvz_gpu_ctx::MultiCall mc = std::move(ctx->multi_calls[i]);
  ctx->multi_calls.erase(ctx->multi_calls.begin() + long(i));
  int rc = CDVZ_GPU_OK;
  for (size_t d = 0; d < mc.shard_ticket.size(); ++d) {
    cdvz_gpu_ctx* sh = ctx->shards[d].get();
    const int r = cdvz_gpu_encode_batch_wait(sh, mc.shard_ticket[d]);
    if (r != CDVZ_GPU_OK && rc == CDVZ_GPU_OK) {
      rc = r;
      err = "device " + std::to_string(sh->device) + ": " + sh->err;
    }
  }
  if (rc != CDVZ_GPU_OK) return rc;
  return guarded(ctx, [&] {
    gather_multi(mc.start, mc.off, true, {}, mc.out, mc.out_cap, mc.offsets, mc.status, mc.slot);
    fold_multi_stats(ctx);
  });
}

int cdvz_gpu_encode_batch_submit(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride,
                                 int count, int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets,
                                 int* status, uint64_t* ticket) {
  NvtxRange nv("cdvz_gpu_encode_batch_submit");
  return guarded(ctx, [&] {
    if (!ticket) throw UsageError("null ticket");
    *ticket = 0;  // 0: the call completed inside submit (nothing to wait for)
    if (!host_args(ctx, pixels, width, height, stride, count, offsets, status, 1)) return;
    mode_by_id(mode_id);
    const bool one_group = size_t(count) <= size_t(host_group_frames(size_t(width) * height, count));
    const size_t slot_bytes = mode_by_id(mode_id).budget + 28;
    if (!ctx->shards.empty() && out_cap >= size_t(count) * slot_bytes) {
      // Multi-device: each shard's share through the shard's own submit (its
      // copies and kernels enqueued, nothing waited for); the wait gathers.
      while (ctx->multi_calls.size() >= 2) {  // two calls in flight: finish the oldest now
        const unsigned long long t = ctx->multi_calls.front().ticket;
        std::string err;
        const int rc = finish_multi(ctx, 0, err);
        ctx->finished.push_back({t, rc, err});
      }
      const int nd = int(ctx->shards.size());
      cdvz_gpu_ctx::MultiCall mc;
      mc.start.resize(size_t(nd) + 1);
      for (int d = 0; d <= nd; ++d) mc.start[size_t(d)] = int((long long)count * d / nd);
      mc.off.resize(size_t(nd));
      mc.shard_ticket.assign(size_t(nd), 0);
      mc.out = out;
      mc.out_cap = out_cap;
      mc.offsets = offsets;
      mc.status = status;
      mc.slot = slot_bytes;
      for (int d = 0; d < nd; ++d) {
        const int n = mc.start[size_t(d) + 1] - mc.start[size_t(d)];
        mc.off[size_t(d)].assign(size_t(n) + 1, 0);
        if (n == 0) continue;
        cdvz_gpu_ctx* sh = ctx->shards[size_t(d)].get();
        const int rc = cdvz_gpu_encode_batch_submit(sh, pixels + size_t(mc.start[size_t(d)]) * height * stride, width,
                                                    height, stride, n, mode_id, max_side,
                                                    out + size_t(mc.start[size_t(d)]) * slot_bytes, size_t(n) * slot_bytes,
                                                    mc.off[size_t(d)].data(), status + mc.start[size_t(d)],
                                                    &mc.shard_ticket[size_t(d)]);
        if (rc != CDVZ_GPU_OK) {
          const std::string msg = "device " + std::to_string(sh->device) + ": " + sh->err;
          for (int e = 0; e < d; ++e) cdvz_gpu_encode_batch_wait(ctx->shards[size_t(e)].get(), mc.shard_ticket[size_t(e)]);
          if (rc == CDVZ_GPU_USAGE) throw UsageError(msg);
          if (rc == CDVZ_GPU_DATA) throw DataError(msg);
          throw std::runtime_error(msg);
        }
      }
      mc.ticket = ctx->next_ticket++;
      *ticket = mc.ticket;
      ctx->multi_calls.push_back(std::move(mc));
      return;
    }
    if (!ctx->shards.empty() || !one_group) {  // multi-device without room in place, or > 4 GB of frames: synchronous
      for (auto& h : ctx->hslot)
        if (h.busy) finish_slot(ctx, h);
      if (encode_host_batch(ctx, pixels, width, height, stride, count, mode_id, max_side, out, out_cap, offsets, status,
                            1) != CDVZ_GPU_OK)
        throw std::runtime_error(ctx->err);
      return;
    }
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    cdvz_gpu_ctx::HostSlot* hs = nullptr;
    for (auto& h : ctx->hslot)
      if (!h.busy) hs = &h;
    if (!hs) {  // both in flight: finish the older one now (its wait returns the held result)
      hs = ctx->hslot[0].ticket < ctx->hslot[1].ticket ? &ctx->hslot[0] : &ctx->hslot[1];
      finish_slot(ctx, *hs);
    }
    slot_args(*hs, pixels, width, height, stride, count, mode_id, max_side, out, out_cap, offsets, status, 1);
    hs->ramp = false;  // streamed calls overlap each other: full chunks, like encode_device
    hs->ticket = ctx->next_ticket++;
    hs->busy = true;
    try {
      host_begin(ctx, *hs, 0, count);
    } catch (...) {
      hs->busy = false;
      hs->ticket = 0;
      throw;
    }
    *ticket = hs->ticket;
  });
}

int cdvz_gpu_encode_batch_wait(cdvz_gpu_ctx* ctx, uint64_t ticket) {
  if (!ctx) return guarded(ctx, [] { throw UsageError("null context"); });
  if (ticket == 0) return CDVZ_GPU_OK;
  for (size_t i = 0; i < ctx->multi_calls.size(); ++i) {
    if (ctx->multi_calls[i].ticket != ticket) continue;
    std::string err;
    const int rc = finish_multi(ctx, i, err);
    if (rc != CDVZ_GPU_OK) ctx->err = err;
    return rc;
  }
  for (auto& h : ctx->hslot)
    if (h.busy && h.ticket == ticket) finish_slot(ctx, h);
  for (size_t i = 0; i < ctx->finished.size(); ++i) {
    if (ctx->finished[i].ticket != ticket) continue;
    const int rc = ctx->finished[i].rc;
    if (rc != CDVZ_GPU_OK) ctx->err = ctx->finished[i].err;
    ctx->finished.erase(ctx->finished.begin() + long(i));
    return rc;
  }
  return guarded(ctx, [] { throw UsageError("unknown or already waited ticket"); });
}

int cdvz_gpu_encode_batch(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride, int count,
                          int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets, int* status) {
  return encode_host_batch(ctx, pixels, width, height, stride, count, mode_id, max_side, out, out_cap, offsets, status, 1);
}

int cdvz_gpu_encode_batch_rgb(cdvz_gpu_ctx* ctx, const uint8_t* rgb, int width, int height, size_t stride, int count,
                              int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets, int* status) {
  return encode_host_batch(ctx, rgb, width, height, stride, count, mode_id, max_side, out, out_cap, offsets, status, 3);
}

int cdvz_gpu_encode_batch_f64(cdvz_gpu_ctx* ctx, const double* pixels, int width, int height, size_t stride, int count,
                              int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets, int* status) {
  if (stride > (size_t(-1) >> 4)) return CDVZ_GPU_USAGE;
  return encode_host_batch(ctx, reinterpret_cast<const uint8_t*>(pixels), width, height, stride * sizeof(double), count,
                           mode_id, max_side, out, out_cap, offsets, status, 8);
}

int cdvz_gpu_stage_times(cdvz_gpu_ctx* ctx, double ms[5]) {
  if (!ctx || !ms) return CDVZ_GPU_USAGE;
  return guarded(ctx, [&] {
    if (ctx->shards.empty()) {
      CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
      ctx->collect_all();
    }
    for (int i = 0; i < 5; ++i) ms[i] = ctx->stats.stage_ms[i];
  });
}

int cdvz_gpu_kernel_stats(cdvz_gpu_ctx* ctx, int* launches, double* pyramid_ms, double* pyramid_bytes) {
  if (!ctx) return CDVZ_GPU_USAGE;
  if (launches) *launches = ctx->launches;
  if (!pyramid_ms && !pyramid_bytes) return CDVZ_GPU_OK;  // the launch count needs no synchronisation
  return guarded(ctx, [&] {
    if (ctx->shards.empty()) {
      CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
      ctx->collect_all();
    }
    if (pyramid_ms) *pyramid_ms = ctx->stats.pyr_ms;
    if (pyramid_bytes) *pyramid_bytes = ctx->stats.pyr_bytes;
  });
}

int cdvz_gpu_debug_get(cdvz_gpu_ctx* ctx, const char* name, int frame, double* dst, size_t cap, size_t* n) {
  return guarded(ctx, [&] {
    if (!ctx || !name || !n) throw UsageError("null argument");
    if (!ctx->shards.empty()) throw UsageError("debug arrays live on one device: use a single-device context");
    if (frame < 0 || frame >= ctx->last_frames) throw UsageError("frame index outside the last batch");
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
    const Lane& lane = ctx->lanes[ctx->last_lane];
    const Batch& b = lane.bt;
    const std::string s(name);
    std::vector<double> v;
    auto get_int = [&](const int* p) {
      int x = 0;
      CDVZ_CUDA_CHECK(cudaMemcpy(&x, p, sizeof(int), cudaMemcpyDeviceToHost));
      return x;
    };
    auto get_kps = [&](const KP* p, int count) {
      std::vector<KP> k(std::size_t(std::max(0, count)));
      if (count > 0) CDVZ_CUDA_CHECK(cudaMemcpy(k.data(), p, sizeof(KP) * count, cudaMemcpyDeviceToHost));
      return k;
    };
    auto put_kp = [&](const KP& k) { v.insert(v.end(), {k.x, k.y, k.sigma, double(k.octave), k.p, k.rho, k.pss, k.d}); };
    auto get_d = [&](const double* p, long long count) {
      std::vector<double> d(std::size_t(std::max(0LL, count)));
      if (count > 0) CDVZ_CUDA_CHECK(cudaMemcpy(d.data(), p, sizeof(double) * count, cudaMemcpyDeviceToHost));
      return d;
    };
    const int last = (b.n_oct - 1) & 1;
    const int n_acc = b.n_oct > 0 ? get_int(b.acc_count + frame * 2 + last) : 0;
    const int n_or = get_int(b.or_count + frame);
    if (s.rfind("refined:", 0) == 0) {
      if (!ctx->debug) throw UsageError("per-octave lists need cdvz_gpu_set_debug(ctx, 1) before the batch");
      const int o = std::stoi(s.substr(8));
      if (o < b.n_oct) {
        const KP* base = lane.dbg_oct.as<KP>() + (long long)o * b.cap_acc * lane.geo_frames + (long long)frame * b.cap_acc;
        for (const KP& k : get_kps(base, get_int(b.oct_count + frame * b.n_oct + o))) put_kp(k);
      }
    } else if (s == "keypoints") {
      for (const KP& k : get_kps(b.acc[last] + (long long)frame * b.cap_acc, n_acc)) put_kp(k);
    } else if (s == "selected") {
      const int ns = get_int(b.sel_count + frame);
      for (const KP& k : get_kps(b.sel + (long long)frame * b.select_n, ns)) put_kp(k);
    } else if (s == "oriented") {
      const int ns = get_int(b.sel_count + frame);
      const auto sel = get_kps(b.sel + (long long)frame * b.select_n, ns);
      std::vector<Oriented> o(static_cast<std::size_t>(n_or));
      if (n_or > 0) CDVZ_CUDA_CHECK(cudaMemcpy(o.data(), b.oriented + (long long)frame * b.cap_or, sizeof(Oriented) * n_or, cudaMemcpyDeviceToHost));
      for (const auto& e : o) {
        put_kp(sel[std::size_t(e.sel)]);
        v.push_back(e.theta);
      }
    } else if (s == "descriptors") {
      v = get_d(b.desc + (long long)frame * b.cap_or * 128, (long long)n_or * 128);
    } else if (s == "x") {
      v = get_d(b.x + (long long)frame * b.cap_or * 32, (long long)n_or * 32);
    } else if (s == "gamma") {
      v = get_d(b.gamma + (long long)frame * b.cap_or * b.nc, (long long)n_or * b.nc);
    } else if (s == "gm") {
      v = get_d(b.gm + (long long)frame * b.nc * 32, (long long)b.nc * 32);
    } else if (s == "gv") {
      if (ctx->last_mode >= 0 && mode_by_id(ctx->last_mode).variance) v = get_d(b.gv + (long long)frame * b.nc * 32, (long long)b.nc * 32);
    } else if (s.rfind("gauss:", 0) == 0) {
      const auto c2 = s.find(':', 6);
      const int o = std::stoi(s.substr(6, c2 - 6)), k = std::stoi(s.substr(c2 + 1));
      if (o < b.n_oct && k >= 0 && k < 4)
        v = get_d(b.pyr + (long long)frame * b.frame_doubles + b.plane_off[o][k], (long long)b.ow[o] * b.oh[o]);
    } else if (s == "norms") {
      // SCFVDescriptor::norms: scfv_delta of each selected component, ascending
      // component order (scfv.cpp:240-251).
      const auto all = get_d(b.norms + (long long)frame * b.nc, b.nc);
      std::vector<uint8_t> mask(size_t((b.nc + 7) / 8));
      CDVZ_CUDA_CHECK(cudaMemcpy(mask.data(), b.mask + (long long)frame * mask.size(), mask.size(), cudaMemcpyDeviceToHost));
      for (int i = 0; i < b.nc; ++i)
        if ((mask[size_t(i / 8)] >> (i % 8)) & 1) v.push_back(all[size_t(i)]);
    } else if (s == "status") {
      v = {double(get_int(b.status + frame))};
    } else {
      throw UsageError("unknown debug array '" + s + "'");
    }
    *n = v.size();
    if (dst && cap >= v.size()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
  });
}

int cdvz_gpu_synth_frames(cdvz_gpu_ctx* ctx, uint64_t base_seed, int count, int width, int height, uint8_t* d_out) {
  return guarded(ctx, [&] {
    require_single(ctx);
    if (!d_out) throw UsageError("null argument");
    if (width < 1 || height < 1 || count < 0) throw UsageError("bad synthetic frame geometry");
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    const int chunk = 64;
    const int nblk = 64;
    DeviceBuffer canvas, params, bmin, bmax;
    canvas.ensure(sizeof(double) * size_t(width) * height * std::min(count, chunk));
    params.ensure(sizeof(SynthParams) * std::min(count, chunk));
    bmin.ensure(sizeof(double) * nblk * std::min(count, chunk));
    bmax.ensure(sizeof(double) * nblk * std::min(count, chunk));
    std::vector<SynthParams> hp(std::size_t(std::min(count, chunk)));
    for (int base = 0; base < count; base += chunk) {
      const int nf = std::min(chunk, count - base);
      for (int i = 0; i < nf; ++i) {
        // synthetic.cpp:11-44 draws, in the reference's order.
        std::mt19937_64 rng(base_seed + static_cast<uint64_t>(base + i) * 0x9E3779B97F4A7C15ull);
        std::uniform_real_distribution<double> unit(0.0, 1.0);
        SynthParams& p = hp[std::size_t(i)];
        p.n_blobs = 8 + static_cast<int>(rng() % 7);
        for (int bl = 0; bl < p.n_blobs; ++bl) {
          const double cx = (0.12 + 0.76 * unit(rng)) * width;
          const double cy = (0.12 + 0.76 * unit(rng)) * height;
          const double s = 2.0 + 10.0 * unit(rng);
          const double amp = (unit(rng) < 0.5 ? -1.0 : 1.0) * (0.4 + 0.6 * unit(rng));
          p.blob[bl][0] = cx;
          p.blob[bl][1] = cy;
          p.blob[bl][2] = amp;
          p.blob[bl][3] = 2.0 * s * s;
        }
        for (int wv = 0; wv < 5; ++wv) {
          const double freq = 1.0 / (6.0 + 26.0 * unit(rng));
          const double angle = unit(rng) * 3.14159265358979323846;
          const double phase = unit(rng) * 2.0 * 3.14159265358979323846;
          const double amp = 0.08 + 0.14 * unit(rng);
          p.wave[wv][0] = std::cos(angle) * freq;
          p.wave[wv][1] = std::sin(angle) * freq;
          p.wave[wv][2] = phase;
          p.wave[wv][3] = amp;
        }
      }
      CDVZ_CUDA_CHECK(cudaMemcpyAsync(params.p, hp.data(), sizeof(SynthParams) * nf, cudaMemcpyHostToDevice, ctx->st));
      CDVZ_CUDA_CHECK(launch_synth(params.as<SynthParams>(), nf, width, height, canvas.as<double>(), bmin.as<double>(),
                                   bmax.as<double>(), nblk, d_out + size_t(base) * width * height, ctx->st));
      CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
    }
    canvas.release();
    params.release();
    bmin.release();
    bmax.release();
  });
}

int cdvz_gpu_pyramid_bench(cdvz_gpu_ctx* ctx, const uint8_t* d_pixels, int width, int height, int count, int iters,
                           double* ms_per_iter, double* bytes_per_iter) {
  return guarded(ctx, [&] {
    require_single(ctx);
    if (!d_pixels || !ms_per_iter || !bytes_per_iter) throw UsageError("null argument");
    if (width < 16 || height < 16 || count < 1 || iters < 1) throw UsageError("bad microbenchmark geometry");
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    Lane& L = ctx->lanes[0];
    if (!L.sA) L.init();
    ctx->plan(L, width, height, count, false);
    Batch b = L.bt;
    b.nframes = count;
    b.pix8 = d_pixels;
    b.stride8 = width;
    b.frame_bytes8 = (long long)height * width;
    double bytes = 0.0;
    for (int o = 0; o < b.n_oct; ++o) {
      const double px = double(b.ow[o]) * b.oh[o];
      const int ww = std::max(0, b.ow[o] - 2 * ctx->dc.margin), hh = std::max(0, b.oh[o] - 2 * ctx->dc.margin);
      bytes += double(count) * (px * ((o == 0 ? 1.0 : 8.0) + 32.0) + 32.0 * ww * hh);
    }
    auto pass = [&] {
      CDVZ_CUDA_CHECK(cudaMemsetAsync(b.raw_count, 0, sizeof(int) * count * std::max(1, b.n_oct), L.sA));
      for (int o = 0; o < b.n_oct; ++o) {
        CDVZ_CUDA_CHECK(launch_octave(b, ctx->dc, o, o == 0 ? 0 : 2, L.sA));
        CDVZ_CUDA_CHECK(launch_detect(b, ctx->dc, o, L.tmap_ok[o] ? &L.tmap[o] : nullptr, L.tmap_ok[o] ? &L.wmap[o] : nullptr, L.sA));
      }
    };
    pass();  // warm-up
    CDVZ_CUDA_CHECK(cudaEventRecord(L.start, L.sA));
    for (int i = 0; i < iters; ++i) pass();
    CDVZ_CUDA_CHECK(cudaEventRecord(L.done, L.sA));
    CDVZ_CUDA_CHECK(cudaEventSynchronize(L.done));
    float ms = 0.f;
    CDVZ_CUDA_CHECK(cudaEventElapsedTime(&ms, L.start, L.done));
    *ms_per_iter = double(ms) / iters;
    *bytes_per_iter = bytes;
    L.geo_w = 0;  // the next encode re-plans (raw lists and bitmaps were left dirty)
  });
}

int cdvz_gpu_device_alloc(cdvz_gpu_ctx* ctx, size_t bytes, void** ptr) {
  return guarded(ctx, [&] {
    require_single(ctx);
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    CDVZ_CUDA_CHECK(cudaMalloc(ptr, std::max<size_t>(bytes, 1)));
  });
}

int cdvz_gpu_device_free(cdvz_gpu_ctx* ctx, void* ptr) {
  return guarded(ctx, [&] {
    require_single(ctx);
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    CDVZ_CUDA_CHECK(cudaFree(ptr));
  });
}

int cdvz_gpu_host_alloc(cdvz_gpu_ctx* ctx, size_t bytes, void** ptr) {
  return guarded(ctx, [&] { CDVZ_CUDA_CHECK(cudaMallocHost(ptr, std::max<size_t>(bytes, 1))); });
}

int cdvz_gpu_host_free(cdvz_gpu_ctx* ctx, void* ptr) {
  return guarded(ctx, [&] { CDVZ_CUDA_CHECK(cudaFreeHost(ptr)); });
}

int cdvz_gpu_copy(cdvz_gpu_ctx* ctx, void* dst, const void* src, size_t bytes, int kind) {
  return guarded(ctx, [&] {
    require_single(ctx);
    CDVZ_CUDA_CHECK(cudaSetDevice(ctx->device));
    const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice : kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, k, ctx->st));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
  });
}

}  // extern "C"

// ---------------------------------------------------------------- training
// train_model (proj/src/pipeline.cpp:99-166) with the heavy work on the GPU:
// pass 1 (detection, selection, description of every corpus image) is the
// extractor's own pipeline; the partner images (apply_transform) are built
// and detected on the device; the PCA covariance and projection, the EM
// iterations and the descriptor transform run as the kernels of train.cu;
// the ordered, tiny steps (relevance histograms, k-means++, the 128 x 128
// eigensolver, quantiles) run on the host (train_host.cpp).
namespace cdvz_gpu {
cudaError_t launch_rotate90(const double* in, int w, int h, int k, double* out, cudaStream_t st);
cudaError_t launch_blur_clamp(const double* in, int w, int h, const double* d_taps, int r, double* tmp, double* out,
                              cudaStream_t st);
cudaError_t launch_covariance(const double* centred, long long n, double* cov, cudaStream_t st);
cudaError_t launch_pca_rows(const double* raw, long long n, const double* mean, const double* basis, double* x,
                            cudaStream_t st);
cudaError_t launch_em_step(const double* x, long long n, int nc, const double* means, const double* stds,
                           const double* log_w, const double* log_norm, double* gamma, double* nk, double* mu,
                           double* ex2, cudaStream_t st);
cudaError_t launch_transform_rows(const double* raw, long long n, const double* ta, const double* tb, double scale,
                                  double* out, cudaStream_t st);
}  // namespace cdvz_gpu

namespace {

// Defaults of a fresh bundle (ScaleSpaceConfig::defaults, scale_space.cpp:85-91;
// RelevanceModel::uniform, relevance.cpp:45-52; TransformPair::defaults,
// transform_coding.cpp:59-79) with neutral quantizer / PCA / GMM sections.
Bundle default_training_bundle(int select_n) {
  Bundle b;
  b.num_octaves = 4;
  b.sigmas.resize(4);
  for (int k = 0; k < 4; ++k) b.sigmas[std::size_t(k)] = 1.4 * std::pow(2.0, k / 4.0);
  b.response_threshold = 0.02;
  b.edge_r = 10.0;
  b.select_n = select_n;
  for (auto& t : b.relevance) {
    t.edges = {0.0, 1.0};
    t.values = {1.0};
  }
  double h[8][8] = {};
  h[0][0] = 1.0;
  for (int n = 1; n < 8; n *= 2)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double v = h[i][j];
        h[i][j + n] = v;
        h[i + n][j] = v;
        h[i + n][j + n] = -v;
      }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      b.tr_a[i][j] = h[i][j];
      b.tr_b[i][j] = h[(i + 1) % 8][j];
    }
  b.tr_scale = 1.0 / 8.0;
  for (int e = 0; e < 128; ++e) {
    b.t0[e] = -1.0;
    b.t1[e] = 1.0;
    b.priority[e] = e;
    b.degenerate[e] = 0;
    b.pca_mean[e] = 0.0;
  }
  b.pca_basis.assign(32 * 128, 0.0);
  for (int r = 0; r < 32; ++r) b.pca_basis[std::size_t(r) * 128 + r] = 1.0;
  b.nc = 1;
  b.weights = {1.0};
  b.means.assign(32, 0.0);
  b.stds.assign(32, 1.0);
  return b;
}

struct OwnedBuffer : DeviceBuffer {
  OwnedBuffer() = default;
  OwnedBuffer(const OwnedBuffer&) = delete;
  OwnedBuffer& operator=(const OwnedBuffer&) = delete;
  ~OwnedBuffer() { release(); }
};

struct FrameLists {
  std::vector<TrainPoint> selected, keypoints;
  std::vector<double> desc;  // oriented descriptors, 128 each
  int status = 0;
};

// One pipeline run over `count` device f64 frames (one call's worth) and the
// per-frame lists of its single chunk, read back from the lane.
std::vector<FrameLists> run_lists(cdvz_gpu_ctx* ctx, const double* d_frames, int w, int h, int count, int max_side,
                                  OwnedBuffer& out, OwnedBuffer& len, bool want_desc) {
  if (count > ctx->max_batch) throw UsageError("training run larger than the context's batch");
  const size_t slot = mode_by_id(3).budget + 28;
  out.ensure(slot * count);
  len.ensure(sizeof(uint32_t) * count);
  ctx->run(reinterpret_cast<const uint8_t*>(d_frames), w, h, (long long)w * 8, count, 3, max_side, out.as<uint8_t>(),
           len.as<uint32_t>(), nullptr, 0, nullptr, nullptr, 8);
  CDVZ_CUDA_CHECK(cudaStreamSynchronize(ctx->st));
  ctx->collect_all();
  const Lane& L = ctx->lanes[ctx->last_lane];
  const Batch& b = L.bt;
  auto get_i = [&](const int* p, long long n) {
    std::vector<int> v(std::size_t(std::max(0LL, n)));
    if (n > 0) CDVZ_CUDA_CHECK(cudaMemcpy(v.data(), p, sizeof(int) * n, cudaMemcpyDeviceToHost));
    return v;
  };
  auto to_points = [&](const KP* p, int n) {
    std::vector<KP> k(std::size_t(std::max(0, n)));
    if (n > 0) CDVZ_CUDA_CHECK(cudaMemcpy(k.data(), p, sizeof(KP) * n, cudaMemcpyDeviceToHost));
    std::vector<TrainPoint> out_;
    out_.reserve(k.size());
    for (const KP& q : k) out_.push_back({q.x, q.y, q.sigma, q.p, q.d, q.rho, q.pss});
    return out_;
  };
  const auto status = get_i(b.status, count);
  const auto sel_count = get_i(b.sel_count, count);
  const auto or_count = get_i(b.or_count, count);
  const int last = (b.n_oct - 1) & 1;
  const auto acc_count = get_i(b.acc_count, 2LL * count);
  std::vector<FrameLists> res(static_cast<size_t>(count));
  for (int f = 0; f < count; ++f) {
    FrameLists& r = res[size_t(f)];
    r.status = status[size_t(f)];
    r.selected = to_points(b.sel + (long long)f * b.select_n, sel_count[size_t(f)]);
    r.keypoints = b.n_oct > 0 ? to_points(b.acc[last] + (long long)f * b.cap_acc, acc_count[size_t(f) * 2 + last])
                              : std::vector<TrainPoint>{};
    if (want_desc && or_count[size_t(f)] > 0) {
      r.desc.resize(size_t(or_count[size_t(f)]) * 128);
      CDVZ_CUDA_CHECK(cudaMemcpy(r.desc.data(), b.desc + (long long)f * b.cap_or * 128,
                                 sizeof(double) * r.desc.size(), cudaMemcpyDeviceToHost));
    }
  }
  return res;
}

}  // namespace

extern "C" int cdvz_gpu_train_model(int device, const double* corpus, int count, int width, int height, size_t stride,
                                    uint64_t seed, int gmm_components, int em_iterations, int select_n, int max_side,
                                    int relevance_bins, char* out, size_t out_cap, size_t* out_len) {
  NvtxRange nv("cdvz_gpu_train_model");
  return guarded(nullptr, [&] {
    if (!corpus || !out_len) throw UsageError("null argument");
    if (count < 20) throw DataError("training corpus needs at least 20 images");  // pipeline.cpp:101
    if (width < 8 || height < 8) throw DataError("image smaller than 8 px per side");
    if (stride < size_t(width)) throw UsageError("row stride shorter than a row");
    // Pass-1 context: defaults, the uniform selector, neutral coding sections.
    const std::string text0 = serialize_bundle(default_training_bundle(select_n));
    cdvz_gpu_ctx* raw_ctx = nullptr;
    if (cdvz_gpu_create(text0.data(), text0.size(), device, std::max(count, 1), &raw_ctx) != CDVZ_GPU_OK)
      throw std::runtime_error(cdvz_gpu_last_error(nullptr));
    std::unique_ptr<cdvz_gpu_ctx> ctx(raw_ctx);
    cudaStream_t st = ctx->st;
    OwnedBuffer d_corpus, d_prep, d_out, d_len, d_a, d_b, d_c, d_taps;
    d_corpus.ensure(sizeof(double) * size_t(count) * width * height);
    CDVZ_CUDA_CHECK(cudaMemcpy2D(d_corpus.p, sizeof(double) * width, corpus, sizeof(double) * stride,
                                 sizeof(double) * width, size_t(height) * count, cudaMemcpyHostToDevice));
    int W = width, H = height;
    prepared_dims(width, height, max_side, W, H);
    // Pass 1 (pipeline.cpp:115-121): every corpus image's selected points and
    // oriented descriptors; the prepared (resized) rasters are kept for the
    // partner images.
    auto lists = run_lists(ctx.get(), d_corpus.as<double>(), width, height, count, max_side, d_out, d_len, true);
    d_prep.ensure(sizeof(double) * size_t(count) * W * H);
    {
      const Lane& L = ctx->lanes[ctx->last_lane];
      const double* src = (W != width || H != height) ? L.bt.pixf : d_corpus.as<double>();
      CDVZ_CUDA_CHECK(cudaMemcpy(d_prep.p, src, sizeof(double) * size_t(count) * W * H, cudaMemcpyDeviceToDevice));
    }
    std::vector<double> raw;
    std::vector<std::pair<TrainPoint, bool>> labeled;
    for (int i = 0; i < count; ++i) {
      const FrameLists& fl = lists[size_t(i)];
      if (fl.status != 0) throw std::runtime_error("training frame " + std::to_string(i) + " failed on the device");
      raw.insert(raw.end(), fl.desc.begin(), fl.desc.end());
      // Partner (pipeline.cpp:124-140): apply_transform, detect_keypoints, map_point, labels.
      const SynthTransform t = partner_transform(size_t(i));
      const int k = ((t.quarter_turns % 4) + 4) % 4;
      const int rw = (k % 2) ? H : W, rh = (k % 2) ? W : H;
      int pw = 0, ph = 0;
      transform_size(t, W, H, pw, ph);
      const size_t big = size_t(std::max(rw * rh, pw * ph));
      d_a.ensure(sizeof(double) * big);
      d_b.ensure(sizeof(double) * big);
      d_c.ensure(sizeof(double) * big);
      CDVZ_CUDA_CHECK(launch_rotate90(d_prep.as<double>() + size_t(i) * W * H, W, H, k, d_a.as<double>(), st));
      const double* cur = d_a.as<double>();
      if (t.scale != 1.0) {
        CDVZ_CUDA_CHECK(launch_resize_f64(cur, rw, rh, d_b.as<double>(), pw, ph, 1, st));
        cur = d_b.as<double>();
      }
      double* partner = (cur == d_a.as<double>()) ? d_b.as<double>() : d_a.as<double>();
      if (t.blur_sigma > 0.0) {
        const std::vector<double> taps = gaussian_kernel_taps(t.blur_sigma);
        d_taps.ensure(sizeof(double) * taps.size());
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(d_taps.p, taps.data(), sizeof(double) * taps.size(), cudaMemcpyHostToDevice, st));
        CDVZ_CUDA_CHECK(launch_blur_clamp(cur, pw, ph, d_taps.as<double>(), int(taps.size() / 2), d_c.as<double>(),
                                          partner, st));
      } else {
        partner = const_cast<double*>(cur);
      }
      CDVZ_CUDA_CHECK(cudaStreamSynchronize(st));
      // detect_keypoints on the partner as it is (no resize_max_side).
      const auto pl = run_lists(ctx.get(), partner, pw, ph, 1, std::max(pw, ph), d_out, d_len, false);
      std::vector<std::array<double, 3>> mapped(fl.selected.size());
      for (size_t s = 0; s < fl.selected.size(); ++s) {
        double mx = fl.selected[s].x, my = fl.selected[s].y, ms = fl.selected[s].sigma;
        map_point(t, W, H, mx, my, ms);
        mapped[s] = {mx, my, ms};
      }
      label_matches(fl.selected, pl[0].keypoints, mapped, 2.0, 1.3, labeled);
    }
    Bundle b = default_training_bundle(select_n);
    b.relevance = train_relevance(labeled, relevance_bins, 10);  // pipeline.cpp:151
    const long long n = (long long)(raw.size() / 128);
    // train_pca (scfv.cpp:328-352).
    if (n < 10 * 128) throw DataError("PCA training needs at least 1280 samples");
    for (double v : raw)
      if (!std::isfinite(v)) throw DataError("PCA training data contains non-finite values");
    {
      std::vector<double> col(static_cast<size_t>(n));
      for (int j = 0; j < 128; ++j) {
        for (long long t = 0; t < n; ++t) col[size_t(t)] = raw[size_t(t) * 128 + j];
        b.pca_mean[j] = eigen_packet_sum(col.data(), col.size()) / static_cast<double>(n);
      }
      std::vector<double> centred(raw.size());
      for (long long t = 0; t < n; ++t)
        for (int j = 0; j < 128; ++j) centred[size_t(t) * 128 + j] = raw[size_t(t) * 128 + j] - b.pca_mean[j];
      d_a.ensure(sizeof(double) * centred.size());
      d_b.ensure(sizeof(double) * 128 * 128);
      CDVZ_CUDA_CHECK(cudaMemcpy(d_a.p, centred.data(), sizeof(double) * centred.size(), cudaMemcpyHostToDevice));
      CDVZ_CUDA_CHECK(launch_covariance(d_a.as<double>(), n, d_b.as<double>(), st));
      std::vector<double> cov(128 * 128), vals, vecs;
      CDVZ_CUDA_CHECK(cudaMemcpyAsync(cov.data(), d_b.p, sizeof(double) * cov.size(), cudaMemcpyDeviceToHost, st));
      CDVZ_CUDA_CHECK(cudaStreamSynchronize(st));
      sym_eigen128(cov, vals, vecs);
      for (int r = 0; r < 32; ++r) {  // strongest 32, sign: largest-magnitude coefficient positive
        double v[128];
        for (int j = 0; j < 128; ++j) v[j] = vecs[size_t(j) * 128 + (127 - r)];
        int arg = 0;
        for (int j = 1; j < 128; ++j)
          if (std::abs(v[j]) > std::abs(v[arg])) arg = j;
        const double sgn = v[arg] < 0.0 ? -1.0 : 1.0;
        for (int j = 0; j < 128; ++j) b.pca_basis[size_t(r) * 128 + j] = sgn < 0.0 ? -v[j] : v[j];
      }
    }
    // pca_reduce of the corpus, then train_gmm (scfv.cpp:354-430).
    OwnedBuffer d_raw, d_x, d_mean, d_basis;
    d_raw.ensure(sizeof(double) * raw.size());
    d_x.ensure(sizeof(double) * size_t(n) * 32);
    d_mean.ensure(sizeof(double) * 128);
    d_basis.ensure(sizeof(double) * 32 * 128);
    CDVZ_CUDA_CHECK(cudaMemcpy(d_raw.p, raw.data(), sizeof(double) * raw.size(), cudaMemcpyHostToDevice));
    CDVZ_CUDA_CHECK(cudaMemcpy(d_mean.p, b.pca_mean, sizeof(double) * 128, cudaMemcpyHostToDevice));
    CDVZ_CUDA_CHECK(cudaMemcpy(d_basis.p, b.pca_basis.data(), sizeof(double) * 32 * 128, cudaMemcpyHostToDevice));
    CDVZ_CUDA_CHECK(launch_pca_rows(d_raw.as<double>(), n, d_mean.as<double>(), d_basis.as<double>(), d_x.as<double>(), st));
    std::vector<double> x(size_t(n) * 32);
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(x.data(), d_x.p, sizeof(double) * x.size(), cudaMemcpyDeviceToHost, st));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(st));
    const int nc = gmm_components;
    if (nc < 1) throw DataError("GMM needs at least one component");
    if (n < std::max<long long>(10 * 32, 2LL * nc)) throw DataError("GMM training corpus is too small");
    {
      constexpr double kFloor = 1e-3;  // kGmmSigmaFloor (scfv.hpp:26)
      std::mt19937_64 rng(seed);
      const auto centers = kmeanspp(x, n, nc, rng);
      b.nc = nc;
      b.weights.assign(size_t(nc), 1.0 / nc);
      b.means.assign(size_t(nc) * 32, 0.0);
      b.stds.assign(size_t(nc) * 32, 0.0);
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < 32; ++j) b.means[size_t(i) * 32 + j] = x[size_t(centers[size_t(i)]) * 32 + j];
      std::vector<double> col(static_cast<size_t>(n));
      double gstd[32];
      for (int j = 0; j < 32; ++j) {
        for (long long t = 0; t < n; ++t) col[size_t(t)] = x[size_t(t) * 32 + j];
        const double gm = eigen_packet_sum(col.data(), col.size()) / static_cast<double>(n);
        for (long long t = 0; t < n; ++t) {
          const double d = col[size_t(t)] - gm;
          col[size_t(t)] = d * d;
        }
        gstd[j] = std::max(std::sqrt(eigen_packet_sum(col.data(), col.size()) / static_cast<double>(n)), kFloor);
      }
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < 32; ++j) b.stds[size_t(i) * 32 + j] = gstd[j];
      OwnedBuffer d_means, d_stds, d_logw, d_lnorm, d_gamma, d_nk, d_mu, d_ex2;
      d_means.ensure(sizeof(double) * nc * 32);
      d_stds.ensure(sizeof(double) * nc * 32);
      d_logw.ensure(sizeof(double) * nc);
      d_lnorm.ensure(sizeof(double) * nc);
      d_gamma.ensure(sizeof(double) * size_t(n) * nc);
      d_nk.ensure(sizeof(double) * nc);
      d_mu.ensure(sizeof(double) * nc * 32);
      d_ex2.ensure(sizeof(double) * nc * 32);
      const size_t unc = static_cast<size_t>(nc);
      std::vector<double> logw(unc), lnorm(unc), nk(unc), mu(unc * 32), ex2(unc * 32);
      for (int iter = 0; iter < em_iterations; ++iter) {
        for (int i = 0; i < nc; ++i) {  // log_weighted_densities' per-component constants (scfv.cpp:25-27)
          double s = 0.0;
          for (int j = 0; j < 32; ++j) s += std::log(b.stds[size_t(i) * 32 + j]);
          lnorm[size_t(i)] = s;
          logw[size_t(i)] = std::log(b.weights[size_t(i)]);
        }
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(d_means.p, b.means.data(), sizeof(double) * nc * 32, cudaMemcpyHostToDevice, st));
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(d_stds.p, b.stds.data(), sizeof(double) * nc * 32, cudaMemcpyHostToDevice, st));
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(d_logw.p, logw.data(), sizeof(double) * nc, cudaMemcpyHostToDevice, st));
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(d_lnorm.p, lnorm.data(), sizeof(double) * nc, cudaMemcpyHostToDevice, st));
        CDVZ_CUDA_CHECK(launch_em_step(d_x.as<double>(), n, nc, d_means.as<double>(), d_stds.as<double>(),
                                       d_logw.as<double>(), d_lnorm.as<double>(), d_gamma.as<double>(),
                                       d_nk.as<double>(), d_mu.as<double>(), d_ex2.as<double>(), st));
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(nk.data(), d_nk.p, sizeof(double) * nc, cudaMemcpyDeviceToHost, st));
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(mu.data(), d_mu.p, sizeof(double) * nc * 32, cudaMemcpyDeviceToHost, st));
        CDVZ_CUDA_CHECK(cudaMemcpyAsync(ex2.data(), d_ex2.p, sizeof(double) * nc * 32, cudaMemcpyDeviceToHost, st));
        CDVZ_CUDA_CHECK(cudaStreamSynchronize(st));
        for (int i = 0; i < nc; ++i) {  // M step (scfv.cpp:412-423)
          if (nk[size_t(i)] < 1e-10) continue;  // starved component keeps its parameters
          for (int j = 0; j < 32; ++j) {
            const double m = mu[size_t(i) * 32 + j];
            b.means[size_t(i) * 32 + j] = m;
            b.stds[size_t(i) * 32 + j] = std::sqrt(std::max(ex2[size_t(i) * 32 + j] - m * m, kFloor * kFloor));
          }
        }
        std::vector<double> w(unc);
        for (int i = 0; i < nc; ++i) w[size_t(i)] = std::max(nk[size_t(i)] / static_cast<double>(n), 1e-12);
        const double ws = eigen_packet_sum(w.data(), w.size());
        for (int i = 0; i < nc; ++i) b.weights[size_t(i)] = w[size_t(i)] / ws;
      }
    }
    // train_thresholds on the transformed corpus (pipeline.cpp:158-162).
    {
      OwnedBuffer d_ta, d_tb, d_tr;
      d_ta.ensure(sizeof(double) * 64);
      d_tb.ensure(sizeof(double) * 64);
      d_tr.ensure(sizeof(double) * raw.size());
      CDVZ_CUDA_CHECK(cudaMemcpy(d_ta.p, &b.tr_a[0][0], sizeof(double) * 64, cudaMemcpyHostToDevice));
      CDVZ_CUDA_CHECK(cudaMemcpy(d_tb.p, &b.tr_b[0][0], sizeof(double) * 64, cudaMemcpyHostToDevice));
      CDVZ_CUDA_CHECK(launch_transform_rows(d_raw.as<double>(), n, d_ta.as<double>(), d_tb.as<double>(), b.tr_scale,
                                            d_tr.as<double>(), st));
      std::vector<double> tr(raw.size());
      CDVZ_CUDA_CHECK(cudaMemcpyAsync(tr.data(), d_tr.p, sizeof(double) * tr.size(), cudaMemcpyDeviceToHost, st));
      CDVZ_CUDA_CHECK(cudaStreamSynchronize(st));
      train_thresholds(tr, n, 1.0 / 3.0, b);
    }
    const std::string text = serialize_bundle(b);
    parse_bundle(text);  // bundle.validate() (pipeline.cpp:164)
    *out_len = text.size();
    if (out && out_cap >= text.size()) std::memcpy(out, text.data(), text.size());
    else if (out) throw UsageError("output buffer too small for the bundle text");
  });
}

namespace cdvz_gpu {
cudaError_t launch_math_check(int fn, const double* a, const double* b, long long n, double* lib, double* ours,
                              cudaStream_t st);
}

extern "C" int cdvz_gpu_math_check(int device, int fn, const double* a, const double* b, size_t n, double* lib,
                                   double* ours) {
  return guarded(nullptr, [&] {
    if (!a || !lib || !ours || (fn == 0 && !b)) throw UsageError("null argument");
    if (fn != 0 && fn != 1) throw UsageError("fn must be 0 (atan2) or 1 (exp)");
    CDVZ_CUDA_CHECK(cudaSetDevice(device));
    if (n == 0) return;
    const size_t bytes = sizeof(double) * n;
    OwnedBuffer da, db, dl, dov;
    da.ensure(bytes);
    db.ensure(bytes);
    dl.ensure(bytes);
    dov.ensure(bytes);
    CDVZ_CUDA_CHECK(cudaMemcpy(da.p, a, bytes, cudaMemcpyHostToDevice));
    if (fn == 0) CDVZ_CUDA_CHECK(cudaMemcpy(db.p, b, bytes, cudaMemcpyHostToDevice));
    CDVZ_CUDA_CHECK(launch_math_check(fn, da.as<double>(), db.as<double>(), (long long)n, dl.as<double>(),
                                      dov.as<double>(), nullptr));
    CDVZ_CUDA_CHECK(cudaMemcpy(lib, dl.p, bytes, cudaMemcpyDeviceToHost));
    CDVZ_CUDA_CHECK(cudaMemcpy(ours, dov.p, bytes, cudaMemcpyDeviceToHost));
  });
}
