/*
 * cdvz_gpu.h — C ABI of the B200-native CDVS-style extractor.
 *
 * Drop-in boundary for the reference's extraction path. The reference exposes
 * no FFI; its boundary is the C++ API in proj/include/cdvz/, and each entry
 * point below states the reference interface it replaces. A C++ shim with the
 * reference's exact signatures sits on top of this ABI in
 * paper_1705_09776_b200/csrc/cdvz_gpu.hpp (cdvz::gpu::encode_image, ...).
 *
 * Conventions
 *   - Plain pointers and sizes only; every buffer is caller-owned.
 *   - Return codes follow the reference CLI's exit-code contract
 *     (proj/tools/cdvz.cpp:308-317): 0 ok, 1 usage error (UsageError),
 *     2 data error (DataError), 3 internal error. No exception crosses the ABI;
 *     the message of the last failure is available from cdvz_gpu_last_error().
 *   - A context owns one CUDA device, its streams and device buffers. It is
 *     not thread-safe: use one context per host thread (as the reference's
 *     StageTimings* is per call). Frames are independent, so several contexts
 *     (one per GPU, or several per GPU) run concurrently without coordination.
 *   - There is no CPU fallback: creating a context without a usable sm_100
 *     device fails with code 3.
 */
#ifndef CDVZ_GPU_H
#define CDVZ_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cdvz_gpu_ctx cdvz_gpu_ctx;

/* Per-frame status written by the batch encoders. */
enum {
  CDVZ_GPU_OK = 0,
  CDVZ_GPU_USAGE = 1,
  CDVZ_GPU_DATA = 2,
  CDVZ_GPU_INTERNAL = 3
};

/* Parses a CDVZ-MODEL 1 bundle text (proj/src/model_io.cpp:141-273,
 * parse_model/load_model, proj/include/cdvz/model_io.hpp:30-33), validates it,
 * computes model_crc = crc32(serialize_model(bundle)) (model_io.cpp:84) and
 * uploads the learned tables to `device`. max_batch bounds the frames per
 * device launch (0 = default 256); larger batches are processed in chunks. */
int cdvz_gpu_create(const char* bundle_text, size_t bundle_len, int device, int max_batch,
                    cdvz_gpu_ctx** out_ctx);

/* Multi-device form of cdvz_gpu_create (SURVEY.md §8(b) "create with a device
 * list"): one single-device context per entry of devices[0..ndev), same
 * bundle. Host batches passed to cdvz_gpu_encode_batch / _rgb / _f64 are split
 * into contiguous frame ranges, one host thread per device (the GPU analogue
 * of the reference's run_indexed fan-out, proj/src/parallel.cpp:40-78), and
 * the containers are gathered in frame order: output is byte-identical to a
 * single-device context's. There is no collective (frames are independent).
 * Device-resident entry points (encode_device, debug_get, events, device
 * allocations) need a single-device context and return CDVZ_GPU_USAGE here.
 * A device index may repeat (several contexts on one GPU). */
int cdvz_gpu_create_multi(const char* bundle_text, size_t bundle_len, const int* devices, int ndev, int max_batch,
                          cdvz_gpu_ctx** out_ctx);

/* Number of visible CUDA devices (0 when there is none). */
int cdvz_gpu_visible_devices(void);

/* Number of devices a context drives (1 for cdvz_gpu_create); their indices
 * are written to devices[0..min(n, cap)). */
int cdvz_gpu_device_count(const cdvz_gpu_ctx* ctx, int* devices, int cap);

/* Releases every device and pinned host buffer of the context. */
void cdvz_gpu_destroy(cdvz_gpu_ctx* ctx);

/* Message of the last failing call on this context (or of the last failing
 * cdvz_gpu_create on this thread when ctx is NULL). */
const char* cdvz_gpu_last_error(const cdvz_gpu_ctx* ctx);

/* Host-only bundle validation (no device needed): parse + validate + the
 * model_crc a context would stamp. Same error codes as cdvz_gpu_create. */
int cdvz_gpu_bundle_check(const char* bundle_text, size_t bundle_len, uint32_t* model_crc, int* components);

/* model_crc stamped into every container and the GMM component count. */
int cdvz_gpu_bundle_info(const cdvz_gpu_ctx* ctx, uint32_t* model_crc, int* components, int* select_n);

/* Batch form of encode_image + serialize_container
 * (proj/src/pipeline.cpp:54-97, proj/include/cdvz/pipeline.hpp:18-20;
 *  proj/src/container.cpp:32-58, proj/include/cdvz/container.hpp:27).
 *
 * pixels: `count` 8-bit grey frames of width x height, row stride `stride`
 *   bytes, frame i at pixels + i*height*stride; a byte b is the intensity
 *   b/255 exactly as load_image reads a PGM (proj/src/image.cpp:79-87).
 * mode_id: 0..5 = 512B,1K,2K,4K,8K,16K (mode_by_id, transform_coding.cpp:33-37).
 * max_side: EncodeOptions::max_side (pipeline.hpp:14-16); 640 by default.
 * out/out_cap: concatenated CDVZ1 containers in frame order; offsets[count+1]
 *   receives each container's byte range. status[count] receives each frame's
 *   result; a failing frame has an empty range and never aborts the batch.
 * Host buffers may be pageable or pinned (cdvz_gpu_host_alloc); both copies
 * (pixels in, containers out) happen inside the call. Returns 0 when the call
 * itself succeeded (check status[] per frame). A frame whose keypoint or
 * orientation lists outgrow the batch capacities is re-encoded on its own with
 * the largest counts the reference can produce, so content alone never fails
 * a frame the reference encodes. */
int cdvz_gpu_encode_batch(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride,
                          int count, int mode_id, int max_side, uint8_t* out, size_t out_cap,
                          size_t* offsets, int* status);

/* cdvz_gpu_encode_batch split in two for streams of batches (a video feed, a
 * crawler): submit enqueues the copies, every kernel and the container copies
 * back and returns a ticket at once; wait(ticket) hands the containers,
 * offsets and status to the caller's buffers (exactly what encode_batch
 * would have written) and returns the call's result code. Up to two
 * submitted batches are in flight per context, so one batch's copies and
 * kernels overlap the previous one's tail; a third submit first completes the
 * oldest (its wait then returns the held result). All buffers of a submitted
 * call must stay valid until its wait returns. On a multi-device context
 * submit hands every device its share through that device's own submit and
 * wait gathers the containers in frame order (two calls in flight there too),
 * provided out_cap leaves a full slot (cdvz_gpu_container_slot) per frame.
 * Ticket 0 means the call completed inside submit (a multi-device call
 * without that room, or a batch above 4 GB, runs synchronously). Errors
 * found while enqueuing are returned by submit. */
int cdvz_gpu_encode_batch_submit(cdvz_gpu_ctx* ctx, const uint8_t* pixels, int width, int height, size_t stride,
                                 int count, int mode_id, int max_side, uint8_t* out, size_t out_cap,
                                 size_t* offsets, int* status, uint64_t* ticket);
int cdvz_gpu_encode_batch_wait(cdvz_gpu_ctx* ctx, uint64_t ticket);

/* GrayImage form of cdvz_gpu_encode_batch — the reference's own input type
 * (proj/include/cdvz/image.hpp:11-18: row-major doubles, rows = height): the
 * raster an in-process producer hands to encode_image (synth_image,
 * apply_transform, a decoder), with no 8-bit quantisation. `stride` is in
 * doubles. Each frame is checked like validate() (proj/src/image.cpp:46-51)
 * on the device: a non-finite value or one outside [0, 1] gives that frame
 * status CDVZ_GPU_DATA and an empty range. Then resize_max_side and the rest
 * of the pipeline run unchanged. */
int cdvz_gpu_encode_batch_f64(cdvz_gpu_ctx* ctx, const double* pixels, int width, int height, size_t stride,
                              int count, int mode_id, int max_side, uint8_t* out, size_t out_cap, size_t* offsets,
                              int* status);

/* train_model (proj/src/pipeline.cpp:99-166, TrainOptions pipeline.hpp:22-28)
 * with the heavy work on device `device`: pass 1 over the corpus (detection,
 * selection, description) and the detection of each image's synthetic partner
 * (apply_transform, synthetic.cpp:78-90) run through the extractor; the PCA
 * covariance and projection, the EM iterations of the GMM and the descriptor
 * transform run as GPU kernels; relevance tables, k-means++ seeding, the
 * eigensolver and the quantiles on the host. `corpus` holds `count` >= 20
 * GrayImages of one size (row-major doubles in [0, 1], row stride `stride`
 * doubles). Writes the bundle text (serialize_model) to `out` (needs *out_len
 * bytes; pass out = NULL to query). Defaults of the reference: seed 7, 8
 * components, 25 EM iterations, select_n 300, max_side 640, 16 bins. The
 * libm (exp / log) and eigensolver differ from glibc / Eigen in the last
 * bits, so the PCA, GMM and quantizer sections are numerically, not bitwise,
 * the reference's. */
int cdvz_gpu_train_model(int device, const double* corpus, int count, int width, int height, size_t stride,
                         uint64_t seed, int gmm_components, int em_iterations, int select_n, int max_side,
                         int relevance_bins, char* out, size_t out_cap, size_t* out_len);

/* PPM form of cdvz_gpu_encode_batch: `count` interleaved 8-bit RGB frames
 * (row stride `stride` >= 3*width bytes). Each pixel becomes the grey value
 * (0.299 r + 0.587 g + 0.114 b) * (1/255) on the device, exactly as
 * load_image reads a P6 file (proj/src/image.cpp:82-87); resize_max_side then
 * runs on that grey plane and the rest of the pipeline is unchanged. Same
 * outputs and error behaviour as cdvz_gpu_encode_batch. */
int cdvz_gpu_encode_batch_rgb(cdvz_gpu_ctx* ctx, const uint8_t* rgb, int width, int height, size_t stride,
                              int count, int mode_id, int max_side, uint8_t* out, size_t out_cap,
                              size_t* offsets, int* status);

/* Header of an in-memory binary PGM (P5) or PPM (P6) file, parsed like
 * load_image (proj/src/image.cpp:53-77; read_pnm_token :17-36): whitespace
 * and '#' comments skipped between fields, maxval must be 255, both sides
 * >= 8, one whitespace byte before the raster, and the raster must be
 * complete. Sets *channels to 1 (P5) or 3 (P6) and *raster_offset to the
 * raster's byte offset in `file` (pass file + offset to cdvz_gpu_encode_batch
 * or cdvz_gpu_encode_batch_rgb with stride = width * channels). Host-only; no
 * context. Returns CDVZ_GPU_DATA for a malformed file (message in
 * cdvz_gpu_last_error(NULL)). */
int cdvz_gpu_pnm_parse(const uint8_t* file, size_t len, int* width, int* height, int* channels,
                       size_t* raster_offset);

/* Same pipeline on frames already resident in device memory (d_pixels is a
 * device pointer to count*height*stride bytes). Containers stay on the device
 * in fixed slots of cdvz_gpu_container_slot(mode) bytes; d_lengths[count]
 * (device) receives the lengths, 0 for a failed frame. Asynchronous: returns
 * once the work is enqueued (ordered after earlier calls on this context);
 * cdvz_gpu_sync waits. No capacity retry on this path (a frame that overflows
 * gets length 0). This is the HBM-resident throughput path of bench.py's
 * `value`. */
int cdvz_gpu_encode_device(cdvz_gpu_ctx* ctx, const uint8_t* d_pixels, int width, int height, size_t stride,
                           int count, int mode_id, int max_side, uint8_t* d_out, uint32_t* d_lengths);
size_t cdvz_gpu_container_slot(int mode_id);
int cdvz_gpu_sync(cdvz_gpu_ctx* ctx);

/* Device time of the last batch per reference stage label, in order
 * detection, selection, description, compression, aggregation
 * (StageTimings, proj/include/cdvz/parallel.hpp:117-134; pipeline.cpp:19-94).
 * Measured with CUDA events around each stage's kernels; waits for the
 * context's enqueued work. On a multi-device context: the sum over devices. */
int cdvz_gpu_stage_times(cdvz_gpu_ctx* ctx, double ms[5]);

/* Launch/kernel bookkeeping for the last batch: number of kernel launches
 * (no synchronisation when pyramid_ms and pyramid_bytes are NULL) and the
 * measured time of the octave (pyramid + extrema) kernels, with the
 * algorithmic HBM bytes they moved (waits for enqueued work). */
int cdvz_gpu_kernel_stats(cdvz_gpu_ctx* ctx, int* launches, double* pyramid_ms, double* pyramid_bytes);

/* Stage-level results of frame `frame` of the last batch for parity tests,
 * as flat doubles (layouts match the oracle's orc_trace_get):
 *   "refined:<o>"  x y sigma octave p rho p_ss d per point of octave o
 *   "keypoints"    after cross-octave dedup (d filled)
 *   "selected"     top-n after selection
 *   "oriented"     keypoint layout + theta
 *   "descriptors"  128 per oriented point
 *   "x" "gamma" "gm" "gv"  SCFV matrices (row-major)
 *   "norms"        SCFVDescriptor::norms: scfv_delta of each selected
 *                  component, ascending component order (scfv.cpp:240-251)
 *   "gauss:<o>:<k>" octave o, level k raster
 * *n receives the element count; nothing is copied when cap is too small. */
int cdvz_gpu_debug_get(cdvz_gpu_ctx* ctx, const char* name, int frame, double* dst, size_t cap, size_t* n);

/* Debug flags. Bit 0 keeps per-octave survivor lists of the next batch for
 * cdvz_gpu_debug_get ("refined:<o>"; one device copy per octave). Bit 1 turns
 * off the FP32 pre-screen of the extrema kernel so every pixel takes the
 * exact FP64 test (used to prove the screen never drops a candidate). Bit 2
 * runs a batch's kernels on one stream, unoverlapped, so per-kernel event
 * times are standalone (bench.py's roofline measurement). Bit 3 disables the
 * TMA tile loads of the extrema kernel (plain loads instead; parity tests).
 * Bit 5 plans tiny list capacities so ordinary frames overflow them and take
 * the host path's capacity retry (tests of that path). */
int cdvz_gpu_set_debug(cdvz_gpu_ctx* ctx, int on);

/* CUDA events on the context's stream (slots 0..3), for callers timing the
 * device-resident path without a CUDA runtime of their own. */
int cdvz_gpu_event_record(cdvz_gpu_ctx* ctx, int slot);
int cdvz_gpu_event_elapsed(cdvz_gpu_ctx* ctx, int slot_a, int slot_b, double* ms);

/* Deterministic synthetic frames on the device (proj/src/synthetic.cpp:11-61,
 * synth_corpus seeds base + i*0x9E3779B97F4A7C15), quantised to bytes like
 * save_pgm. d_out receives count*height*width bytes. */
int cdvz_gpu_synth_frames(cdvz_gpu_ctx* ctx, uint64_t base_seed, int count, int width, int height, uint8_t* d_out);

/* Device / pinned host memory helpers for callers without a CUDA runtime. */
int cdvz_gpu_device_alloc(cdvz_gpu_ctx* ctx, size_t bytes, void** ptr);
int cdvz_gpu_device_free(cdvz_gpu_ctx* ctx, void* ptr);
int cdvz_gpu_host_alloc(cdvz_gpu_ctx* ctx, size_t bytes, void** ptr);
int cdvz_gpu_host_free(cdvz_gpu_ctx* ctx, void* ptr);
int cdvz_gpu_copy(cdvz_gpu_ctx* ctx, void* dst, const void* src, size_t bytes, int kind /* 1 H2D, 2 D2H, 3 D2D */);

/* Releases the context's per-batch device buffers (pyramid, lists, sample
 * records; they are re-planned by the next call). The model tables stay. */
int cdvz_gpu_trim(cdvz_gpu_ctx* ctx);

/* Microbenchmark of the octave kernel pair alone (k_blur + k_detect_walk over
 * every octave): `count` device-resident u8 frames
 * of width x height at native size, `iters` timed passes after one warm-up.
 * Returns the CUDA-event time per pass and the pair's algorithmic bytes per
 * pass. No reference counterpart: a measurement hook. */
int cdvz_gpu_pyramid_bench(cdvz_gpu_ctx* ctx, const uint8_t* d_pixels, int width, int height, int count, int iters,
                           double* ms_per_iter, double* bytes_per_iter);

/* Verification hook for the kernels' FP64 math (csrc/dmath.cuh): evaluates
 * the CUDA library's atan2(a, b) (fn 0) or exp(a) (fn 1; b unused) and the
 * constant-memory restatement the kernels call on `n` host inputs on
 * `device`, writing both results (host arrays). No reference counterpart. */
int cdvz_gpu_math_check(int device, int fn, const double* a, const double* b, size_t n, double* lib, double* ours);

/* ------------------------------------------------------------------------
 * Compressed-domain matching and retrieval: an index of
 * CDVZ1 containers decoded on the device, queried in batches.
 * ------------------------------------------------------------------------ */
typedef struct cdvz_gpu_index cdvz_gpu_index;

/* Decodes `count` containers (blob + offsets[count+1]) on `device`: the
 * reference's parse_container (proj/src/container.cpp:60-93) with
 * parse_scfv / unpack_local (proj/src/scfv.cpp:300-326,
 * proj/src/transform_coding.cpp:272-305) for a whole index. id_rank[i] is
 * item i's rank in ascending id order — the tie-break retrieve applies to
 * item ids (proj/src/eval.cpp:91-94); NULL means index order. Every container
 * must pass the reference's checks (DataError otherwise, naming the item) and
 * share one model bundle and mode. */
int cdvz_gpu_index_create(int device, const uint8_t* blob, const size_t* offsets, int count, const int32_t* id_rank,
                          cdvz_gpu_index** out);
void cdvz_gpu_index_destroy(cdvz_gpu_index* idx);
const char* cdvz_gpu_index_last_error(const cdvz_gpu_index* idx);
int cdvz_gpu_index_info(const cdvz_gpu_index* idx, int* count, int* mode_id, uint32_t* model_crc, int* components,
                        long long* total_codes);

/* retrieve (proj/src/eval.cpp:76-124, proj/include/cdvz/eval.hpp:49-55) for
 * `nq` query containers at once: rank the index by scfv_similarity, re-rank
 * the top `rerank_depth` by count_local_matches(ratio_test), and write each
 * query's first `max_results` (0 = all) ranked items and scores to
 * out_items / out_scores (nq x max_results, row-major) with the reference's
 * scores: local + (sim + 1) / 2 in the head, (sim + 1) / 2 - 1 beyond it. */
int cdvz_gpu_retrieve(cdvz_gpu_index* idx, const uint8_t* query_blob, const size_t* query_offsets, int nq,
                      double ratio_test, int rerank_depth, int max_results, int32_t* out_items, double* out_scores);

/* match_pair (proj/src/eval.cpp:66-74, eval.hpp:44-47) for `np` pairs
 * (query pairs[2k], index item pairs[2k+1]): global similarity
 * (scfv_similarity, scfv.cpp:255-278) and mutual ratio-test local matches
 * (count_local_matches, eval.cpp:47-64). */
int cdvz_gpu_match_pairs(cdvz_gpu_index* idx, const uint8_t* query_blob, const size_t* query_offsets, int nq,
                         const int32_t* pairs, int np, double ratio_test, double* global_sim, int32_t* local_matches);

#ifdef __cplusplus
}
#endif

#endif /* CDVZ_GPU_H */
