// Compressed-domain matching and retrieval over CDVZ1 bitstreams (SURVEY.md
// §8(f) rank 1, with the decoder of rank 3 underneath).
//
// Replaces parse_container / parse_scfv / unpack_local
// (proj/src/container.cpp:60-93, proj/src/scfv.cpp:300-326,
// proj/src/transform_coding.cpp:272-305), scfv_similarity (scfv.cpp:255-278),
// ternary_distance (transform_coding.cpp:219-226), count_local_matches /
// match_pair / retrieve (proj/src/eval.cpp:17-124).
//
// Layout. An index of N containers is decoded on the device once:
//   mask[N][kMaskWords] u64  selected components (bit i of byte i/8)
//   plane[N][nc] u32         mean sign plane of component i (0 if unselected)
//   code_off[N+1]            first code of each item in codes[]
//   codes[total][2] uint4    ternary symbols as two bit planes: P (+1), M (-1)
// so |a - b| summed over a code is popc(Pa ^ Pb) + popc(Ma ^ Mb) — the
// reference's integer ternary_distance with no per-symbol loop.
//
// Retrieval of Q queries: one thread per (query, item) forms the global
// similarity exactly as the reference (integer accumulation, one double
// division); a stable segmented radix sort (CUB) orders each query's list by
// (similarity desc, id asc); one CTA per (query, head item) counts mutual
// ratio-test matches; one warp per query re-ranks the head by (local matches,
// similarity, id) and writes the reference's scores.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/device/device_segmented_radix_sort.cuh>

#include "../../include/cdvz_gpu.h"
#include "bundle.hpp"
#include "common.cuh"

namespace cdvz_gpu {

constexpr int kMaxComponents = 1024;
constexpr int kMaskWords = kMaxComponents / 64;

// Per-item header decoded from the container (container.cpp:60-93).
struct ItemHdr {
  int status;      // 0 ok, else the first failing check (see k_parse_headers)
  int mode, nc, width, height;
  uint32_t model_crc;
  int n_codes, elements, local_mode, n_selected;
  long long codes_at;  // byte offset of the first packed code in the blob
};

__device__ __forceinline__ uint32_t rd_u32(const uint8_t* p) {
  return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}
__device__ __forceinline__ int rd_u16(const uint8_t* p) { return int(p[0]) | (int(p[1]) << 8); }

// Thread per container: magic, CRC-32, header, section lengths, parse_scfv,
// local block header. Status codes: 1 truncated, 2 magic, 3 checksum,
// 4 unknown mode, 5 section lengths, 6 global block, 7 local block,
// 8 reserved symbol pattern (set by k_parse_codes), 9 too many components.
__global__ void __launch_bounds__(128) k_parse_headers(const uint8_t* blob, const size_t* off, int n, ItemHdr* hdr,
                                                        unsigned long long* mask, uint32_t* plane, int nc_cap) {
  __shared__ uint32_t table[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = uint32_t(i);
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    table[i] = c;
  }
  __syncthreads();
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n) return;
  ItemHdr h{};
  const uint8_t* p = blob + off[it];
  const long long len = (long long)(off[it + 1] - off[it]);
  auto done = [&](int st) {
    h.status = st;
    hdr[it] = h;
  };
  if (len < 28) return done(1);
  const char magic[5] = {'C', 'D', 'V', 'Z', '1'};
  for (int i = 0; i < 5; ++i)
    if (p[i] != uint8_t(magic[i])) return done(2);
  const long long body = len - 4;
  uint32_t c = 0xFFFFFFFFu;  // crc32 (common.cpp:11-35)
  for (long long i = 0; i < body; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  if ((c ^ 0xFFFFFFFFu) != rd_u32(p + body)) return done(3);
  h.mode = p[5];
  if (h.mode > 5) return done(4);
  h.width = rd_u16(p + 6);
  h.height = rd_u16(p + 8);
  h.nc = rd_u16(p + 10);
  h.model_crc = rd_u32(p + 12);
  const long long glen = rd_u32(p + 16), llen = rd_u32(p + 20);
  if (24 + glen + llen != body) return done(5);
  if (h.nc > nc_cap) return done(9);
  // parse_scfv (scfv.cpp:300-326): mask, then one u32 (two with variance
  // planes, modes 8K/16K) per selected component in ascending order.
  const bool variance = h.mode >= 4;
  const int mask_bytes = (h.nc + 7) / 8;
  if (glen < mask_bytes) return done(6);
  const uint8_t* g = p + 24;
  int sel = 0;
  for (int b = 0; b < mask_bytes; ++b) sel += __popc(g[b]);
  if (glen != (long long)mask_bytes + (long long)sel * (variance ? 8 : 4)) return done(6);
  unsigned long long* m = mask + (long long)it * kMaskWords;
  uint32_t* pl = plane + (long long)it * nc_cap;
  for (int w = 0; w < kMaskWords; ++w) m[w] = 0ull;
  int rank = 0;
  for (int b = 0; b < mask_bytes; ++b)
    for (int k = 0; k < 8; ++k) {
      if (!((g[b] >> k) & 1)) continue;
      const int i = 8 * b + k;
      if (i < h.nc) {
        m[i >> 6] |= 1ull << (i & 63);
        pl[i] = rd_u32(g + mask_bytes + (long long)rank * (variance ? 8 : 4));
      }
      ++rank;
    }
  h.n_selected = sel;
  // unpack_local header (transform_coding.cpp:272-285).
  const uint8_t* l = g + glen;
  if (llen < 4) return done(7);
  h.local_mode = l[0];
  h.elements = l[1];
  h.n_codes = rd_u16(l + 2);
  if (h.local_mode > 5 || h.elements < 1 || h.elements > 128) return done(7);
  const long long per = 6 + (2LL * h.elements + 7) / 8;
  if (llen != 4 + (long long)h.n_codes * per) return done(7);
  h.codes_at = (long long)off[it] + 24 + glen + 4;
  done(0);
}

// Thread per code: the 2-bit symbols 00 = 0, 01 = +1, 10 = -1 become bit
// planes P and M; 11 is the reserved pattern unpack_local rejects.
__global__ void __launch_bounds__(256) k_parse_codes(const uint8_t* blob, ItemHdr* hdr, const int* code_off, int n,
                                                      uint4* codes) {
  const int total = code_off[n];
  const int gc = blockIdx.x * blockDim.x + threadIdx.x;
  if (gc >= total) return;
  int lo = 0, hi = n;  // item = last index with code_off[item] <= gc
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (code_off[mid] <= gc) lo = mid;
    else hi = mid;
  }
  const ItemHdr& h = hdr[lo];
  const int k = gc - code_off[lo];
  const long long per = 6 + (2LL * h.elements + 7) / 8;
  const uint8_t* s = blob + h.codes_at + (long long)k * per + 6;
  uint32_t P[4] = {0, 0, 0, 0}, M[4] = {0, 0, 0, 0};
  bool bad = false;
  for (int e = 0; e < h.elements; ++e) {
    const int bits = (s[e >> 2] >> (2 * (e & 3))) & 3;
    if (bits == 1) P[e >> 5] |= 1u << (e & 31);
    else if (bits == 2) M[e >> 5] |= 1u << (e & 31);
    else if (bits == 3) bad = true;
  }
  if (bad) atomicCAS(&hdr[lo].status, 0, 8);
  codes[2LL * gc] = make_uint4(P[0], P[1], P[2], P[3]);
  codes[2LL * gc + 1] = make_uint4(M[0], M[1], M[2], M[3]);
}

struct Decoded {
  int n = 0, nc_cap = 0;
  unsigned long long* mask = nullptr;
  uint32_t* plane = nullptr;
  int* code_off = nullptr;
  uint4* codes = nullptr;
};

// scfv_similarity (scfv.cpp:255-278) of query q and item it.
__device__ __forceinline__ double global_sim(const Decoded& A, int a, const Decoded& B, int b, int nc) {
  const unsigned long long* ma = A.mask + (long long)a * kMaskWords;
  const unsigned long long* mb = B.mask + (long long)b * kMaskWords;
  const uint32_t* pa = A.plane + (long long)a * A.nc_cap;
  const uint32_t* pb = B.plane + (long long)b * B.nc_cap;
  long long accum = 0;
  int common = 0;
  const int words = (nc + 63) / 64;
  for (int w = 0; w < words; ++w) {
    unsigned long long both = ma[w] & mb[w];
    while (both) {
      const int i = 64 * w + __ffsll((long long)both) - 1;
      both &= both - 1;
      accum += 32 - 2 * __popc(pa[i] ^ pb[i]);
      ++common;
    }
  }
  if (common == 0) return -1.0;
  return static_cast<double>(accum) / (32.0 * common);
}

// Order-preserving map of a double to u64 (descending radix sort keys).
__device__ __forceinline__ unsigned long long order_key(double d) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  const unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)u);
}

// Thread per (query, position p of the id order): key = similarity, value = item.
// Queries q0 + blockIdx.y of the batch; keys / vals hold this chunk's rows.
__global__ void __launch_bounds__(256) k_global_keys(Decoded Q, Decoded X, const int* perm, int n, int nc, int q0,
                                                      unsigned long long* keys, int* vals) {
  const int q = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int it = perm[p];
  keys[(long long)q * n + p] = order_key(global_sim(Q, q0 + q, X, it, nc));
  vals[(long long)q * n + p] = it;
}

// count_local_matches (eval.cpp:25-64) of query codes A and item codes B,
// one CTA per pair. Nearest and second-nearest by (distance, index), both
// directions, then mutual nearest neighbours passing the ratio test.
constexpr int kLMThreads = 128;
__device__ int count_local(const uint4* A, int na, const uint4* B, int nb, double ratio, uint4* sA, uint4* sB, int* a_best,
                           int* a_d1, int* a_d2, int* b_best, int* b_d1, int* b_d2, int* red) {
  if (na == 0 || nb == 0) return 0;
  for (int i = threadIdx.x; i < 2 * na; i += blockDim.x) sA[i] = A[i];
  for (int i = threadIdx.x; i < 2 * nb; i += blockDim.x) sB[i] = B[i];
  __syncthreads();
  auto nearest = [&](const uint4* x, int nx, const uint4* pool, int npool, int* best, int* d1, int* d2) {
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      const uint4 p = x[2 * i], m = x[2 * i + 1];
      int bi = -1, bd = 0x7fffffff, sd = 0x7fffffff;
      for (int j = 0; j < npool; ++j) {
        const uint4 q = pool[2 * j], r = pool[2 * j + 1];
        const int d = __popc(p.x ^ q.x) + __popc(p.y ^ q.y) + __popc(p.z ^ q.z) + __popc(p.w ^ q.w) +
                      __popc(m.x ^ r.x) + __popc(m.y ^ r.y) + __popc(m.z ^ r.z) + __popc(m.w ^ r.w);
        if (d < bd) {
          sd = bd;
          bd = d;
          bi = j;
        } else if (d < sd) {
          sd = d;
        }
      }
      best[i] = bi;
      d1[i] = bd;
      d2[i] = sd;
    }
  };
  nearest(sA, na, sB, nb, a_best, a_d1, a_d2);
  nearest(sB, nb, sA, na, b_best, b_d1, b_d2);
  __syncthreads();
  auto passes = [&](int best, int d1, int d2, int pool) {  // passes_ratio, eval.cpp:39-43
    if (best < 0) return false;
    if (pool < 2) return true;
    return double(d1) < ratio * double(d2);
  };
  int cnt = 0;
  for (int i = threadIdx.x; i < na; i += blockDim.x) {
    if (!passes(a_best[i], a_d1[i], a_d2[i], nb)) continue;
    const int j = a_best[i];
    if (b_best[j] != i || !passes(b_best[j], b_d1[j], b_d2[j], na)) continue;
    ++cnt;
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  int total = 0;
  for (int w = 0; w < kLMThreads / 32; ++w) total += red[w];
  __syncthreads();
  return total;
}

// One CTA per (query, head rank r): the item is vals[q][r].
__global__ void __launch_bounds__(kLMThreads) k_local_head(Decoded Q, Decoded X, const int* vals, int n, int head,
                                                           double ratio, int max_codes, int q0, int* local) {
  extern __shared__ __align__(16) uint8_t lm_smem[];
  const int lq = blockIdx.y, r = blockIdx.x, q = q0 + lq;
  const int it = vals[(long long)lq * n + r];
  const int na = Q.code_off[q + 1] - Q.code_off[q], nb = X.code_off[it + 1] - X.code_off[it];
  uint4* sA = reinterpret_cast<uint4*>(lm_smem);
  uint4* sB = sA + 2 * max_codes;
  int* ib = reinterpret_cast<int*>(sB + 2 * max_codes);
  __shared__ int red[kLMThreads / 32];
  const int c = count_local(Q.codes + 2LL * Q.code_off[q], na, X.codes + 2LL * X.code_off[it], nb, ratio, sA, sB, ib,
                            ib + max_codes, ib + 2 * max_codes, ib + 3 * max_codes, ib + 4 * max_codes, ib + 5 * max_codes,
                            red);
  if (threadIdx.x == 0) local[(long long)lq * head + r] = c;
}

// One CTA per explicit (query, item) pair: global similarity + local matches.
__global__ void __launch_bounds__(kLMThreads) k_match_pairs(Decoded Q, Decoded X, const int* pairs, int nc, double ratio,
                                                            int max_codes, double* sim, int* local) {
  extern __shared__ __align__(16) uint8_t lm_smem[];
  const int k = blockIdx.x;
  const int q = pairs[2 * k], it = pairs[2 * k + 1];
  const int na = Q.code_off[q + 1] - Q.code_off[q], nb = X.code_off[it + 1] - X.code_off[it];
  uint4* sA = reinterpret_cast<uint4*>(lm_smem);
  uint4* sB = sA + 2 * max_codes;
  int* ib = reinterpret_cast<int*>(sB + 2 * max_codes);
  __shared__ int red[kLMThreads / 32];
  const int c = count_local(Q.codes + 2LL * Q.code_off[q], na, X.codes + 2LL * X.code_off[it], nb, ratio, sA, sB, ib,
                            ib + max_codes, ib + 2 * max_codes, ib + 3 * max_codes, ib + 4 * max_codes, ib + 5 * max_codes,
                            red);
  if (threadIdx.x == 0) {
    local[k] = c;
    sim[k] = global_sim(Q, q, X, it, nc);
  }
}

// One warp per query: re-rank the head by (local desc, similarity desc, id
// asc) and write every item's final rank and score (eval.cpp:97-123).
// CTA per query: threads r < head rank the re-ranked head, every thread
// copies the tail (the full ranked list is the output: n entries per query).
constexpr int kFinishThreads = 256;
__global__ void __launch_bounds__(kFinishThreads) k_finish(const unsigned long long* keys, const int* vals,
                                                           const int* local, const int* id_rank, int n, int head,
                                                           int max_results, int q0, int* out_items,
                                                           double* out_scores) {
  const int q = blockIdx.x, lane = threadIdx.x;
  const unsigned long long* kq = keys + (long long)q * n;
  const int* vq = vals + (long long)q * n;
  const int* lq = local + (long long)q * head;
  int* oi = out_items + (long long)(q0 + q) * max_results;
  double* os = out_scores + (long long)(q0 + q) * max_results;
  for (int r = lane; r < head; r += kFinishThreads) {
    const int lr = lq[r];
    const double sr = key_value(kq[r]);
    const int ir = id_rank[vq[r]];
    int pos = 0;
    for (int s = 0; s < head; ++s) {
      const int ls = lq[s];
      const double ss = key_value(kq[s]);
      const int is = id_rank[vq[s]];
      pos += (ls > lr || (ls == lr && (ss > sr || (ss == sr && is < ir)))) ? 1 : 0;
    }
    if (pos < max_results) {
      oi[pos] = vq[r];
      os[pos] = lr + (sr + 1.0) / 2.0;
    }
  }
  for (int r = head + lane; r < min(n, max_results); r += kFinishThreads) {
    oi[r] = vq[r];
    os[r] = (key_value(kq[r]) + 1.0) / 2.0 - 1.0;
  }
}

}  // namespace cdvz_gpu

using namespace cdvz_gpu;

namespace {

thread_local std::string g_index_error;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    CDVZ_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(n, 16)));
    bytes = n;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// A decoded set of containers on the device (the index, or a batch of queries).
struct DecodedSet {
  DevBuf blob, off, hdr, mask, plane, code_off, codes;
  std::vector<ItemHdr> h;
  Decoded view;
  int mode = -1, nc = 0, elements = 0, local_mode = -1, max_codes = 0;
  uint32_t model_crc = 0;
  long long total_codes = 0;

  void decode(const uint8_t* host_blob, const size_t* host_off, int n, cudaStream_t st, const char* what) {
    if (n <= 0) throw DataError(std::string(what) + " is empty");
    const size_t bytes = host_off[n] - host_off[0];
    blob.ensure(bytes);
    std::vector<size_t> rel(size_t(n) + 1);
    for (int i = 0; i <= n; ++i) rel[size_t(i)] = host_off[i] - host_off[0];
    // Dense plane rows are sized by the largest component count the headers
    // announce (bytes 10-11); the device parse re-validates every field.
    int nc_cap = 1;
    for (int i = 0; i < n; ++i) {
      const uint8_t* p = host_blob + host_off[i];
      if (host_off[i + 1] - host_off[i] >= 12) nc_cap = std::max(nc_cap, int(p[10]) | (int(p[11]) << 8));
    }
    nc_cap = std::min(nc_cap, kMaxComponents);
    off.ensure(sizeof(size_t) * (size_t(n) + 1));
    hdr.ensure(sizeof(ItemHdr) * size_t(n));
    mask.ensure(sizeof(unsigned long long) * kMaskWords * size_t(n));
    plane.ensure(sizeof(uint32_t) * size_t(nc_cap) * size_t(n));
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(blob.p, host_blob + host_off[0], bytes, cudaMemcpyHostToDevice, st));
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(off.p, rel.data(), sizeof(size_t) * rel.size(), cudaMemcpyHostToDevice, st));
    CDVZ_CUDA_CHECK(cudaMemsetAsync(plane.p, 0, sizeof(uint32_t) * size_t(nc_cap) * size_t(n), st));
    k_parse_headers<<<(n + 127) / 128, 128, 0, st>>>(blob.as<uint8_t>(), off.as<size_t>(), n, hdr.as<ItemHdr>(),
                                                      mask.as<unsigned long long>(), plane.as<uint32_t>(), nc_cap);
    CDVZ_CUDA_CHECK(cudaGetLastError());
    h.resize(size_t(n));
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(h.data(), hdr.p, sizeof(ItemHdr) * size_t(n), cudaMemcpyDeviceToHost, st));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(st));
    check(what);
    std::vector<int> co(size_t(n) + 1, 0);
    for (int i = 0; i < n; ++i) {
      co[size_t(i) + 1] = co[size_t(i)] + h[size_t(i)].n_codes;
      max_codes = std::max(max_codes, h[size_t(i)].n_codes);
    }
    total_codes = co[size_t(n)];
    code_off.ensure(sizeof(int) * co.size());
    codes.ensure(2 * sizeof(uint4) * size_t(std::max<long long>(1, total_codes)));
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(code_off.p, co.data(), sizeof(int) * co.size(), cudaMemcpyHostToDevice, st));
    if (total_codes > 0) {
      k_parse_codes<<<unsigned((total_codes + 255) / 256), 256, 0, st>>>(blob.as<uint8_t>(), hdr.as<ItemHdr>(),
                                                                        code_off.as<int>(), n, codes.as<uint4>());
      CDVZ_CUDA_CHECK(cudaGetLastError());
    }
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(h.data(), hdr.p, sizeof(ItemHdr) * size_t(n), cudaMemcpyDeviceToHost, st));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(st));
    check(what);
    view.n = n;
    view.nc_cap = nc_cap;
    view.mask = mask.as<unsigned long long>();
    view.plane = plane.as<uint32_t>();
    view.code_off = code_off.as<int>();
    view.codes = codes.as<uint4>();
  }

  // The reference throws DataError from parse_container on the first bad
  // container; an index (or query batch) must also share one model bundle,
  // one mode and one local code layout.
  void check(const char* what) {
    static const char* reasons[] = {"",
                                    "container truncated",
                                    "container magic mismatch",
                                    "container checksum mismatch",
                                    "unknown mode id",
                                    "container section lengths disagree with its size",
                                    "global descriptor length does not match its mask",
                                    "local block length does not match its header",
                                    "reserved symbol pattern in local block",
                                    "too many mixture components"};
    for (size_t i = 0; i < h.size(); ++i) {
      const ItemHdr& x = h[i];
      if (x.status) throw DataError(std::string(what) + " item " + std::to_string(i) + ": " + reasons[x.status]);
      if (i == 0) {
        mode = x.mode;
        nc = x.nc;
        model_crc = x.model_crc;
        elements = x.elements;
        local_mode = x.local_mode;
      } else if (x.model_crc != model_crc) {
        throw DataError(std::string(what) + " item " + std::to_string(i) + " was encoded with a different model bundle");
      } else if (x.mode != mode || x.nc != nc || x.elements != elements || x.local_mode != local_mode) {
        throw DataError(std::string(what) + " item " + std::to_string(i) + " mode mismatch");
      }
    }
  }
};

}  // namespace

struct cdvz_gpu_index {
  int device = 0;
  cudaStream_t st = nullptr;
  std::string err;
  DecodedSet items;
  DevBuf perm, id_rank, keys, vals, keys2, vals2, seg, local, temp, out_i, out_s, pairs, psim, ploc;
  std::vector<int> h_perm, h_rank;
  ~cdvz_gpu_index() {
    if (st) cudaStreamDestroy(st);
  }
};

namespace {

template <class F>
int guarded_index(cdvz_gpu_index* idx, F&& f) {
  try {
    f();
    if (idx) idx->err.clear();
    return CDVZ_GPU_OK;
  } catch (const UsageError& e) {
    (idx ? idx->err : g_index_error) = e.what();
    return CDVZ_GPU_USAGE;
  } catch (const DataError& e) {
    (idx ? idx->err : g_index_error) = e.what();
    return CDVZ_GPU_DATA;
  } catch (const std::exception& e) {
    (idx ? idx->err : g_index_error) = e.what();
    return CDVZ_GPU_INTERNAL;
  }
}

void check_queries(const cdvz_gpu_index* idx, const DecodedSet& q) {
  // retrieve / match_pair (eval.cpp:66-88): same bundle, same mode.
  if (q.model_crc != idx->items.model_crc) throw DataError("index container was encoded with a different model bundle");
  if (q.mode != idx->items.mode || q.nc != idx->items.nc) throw DataError("index container mode mismatch");
  if (q.elements != idx->items.elements || q.local_mode != idx->items.local_mode)
    throw DataError("ternary codes from different modes cannot be compared");
}

size_t lm_smem_bytes(int max_codes) { return 2 * 2 * sizeof(uint4) * size_t(max_codes) + 6 * sizeof(int) * size_t(max_codes); }

}  // namespace

extern "C" {

int cdvz_gpu_index_create(int device, const uint8_t* blob, const size_t* offsets, int count, const int32_t* id_rank,
                          cdvz_gpu_index** out) {
  return guarded_index(nullptr, [&] {
    if (!out || (!blob && count > 0) || !offsets) throw UsageError("null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw std::runtime_error("no CUDA device available (the matcher has no CPU fallback)");
    if (device < 0 || device >= ndev) throw UsageError("device index out of range");
    if (count <= 0) throw DataError("retrieval index is empty");
    CDVZ_CUDA_CHECK(cudaSetDevice(device));
    auto idx = std::make_unique<cdvz_gpu_index>();
    idx->device = device;
    CDVZ_CUDA_CHECK(cudaStreamCreateWithFlags(&idx->st, cudaStreamNonBlocking));
    idx->items.decode(blob, offsets, count, idx->st, "index");
    // Item ids: id_rank[i] is item i's rank in ascending id order (the
    // reference's tie-break, eval.cpp:91-94); NULL means index order.
    idx->h_rank.resize(size_t(count));
    for (int i = 0; i < count; ++i) idx->h_rank[size_t(i)] = id_rank ? id_rank[i] : i;
    idx->h_perm.assign(size_t(count), -1);
    for (int i = 0; i < count; ++i) {
      const int r = idx->h_rank[size_t(i)];
      if (r < 0 || r >= count || idx->h_perm[size_t(r)] != -1) throw UsageError("id_rank is not a permutation");
      idx->h_perm[size_t(r)] = i;
    }
    idx->perm.ensure(sizeof(int) * size_t(count));
    idx->id_rank.ensure(sizeof(int) * size_t(count));
    CDVZ_CUDA_CHECK(cudaMemcpy(idx->perm.p, idx->h_perm.data(), sizeof(int) * size_t(count), cudaMemcpyHostToDevice));
    CDVZ_CUDA_CHECK(cudaMemcpy(idx->id_rank.p, idx->h_rank.data(), sizeof(int) * size_t(count), cudaMemcpyHostToDevice));
    *out = idx.release();
  });
}

void cdvz_gpu_index_destroy(cdvz_gpu_index* idx) {
  if (!idx) return;
  cudaSetDevice(idx->device);
  cudaStreamSynchronize(idx->st);
  delete idx;
}

const char* cdvz_gpu_index_last_error(const cdvz_gpu_index* idx) { return idx ? idx->err.c_str() : g_index_error.c_str(); }

int cdvz_gpu_index_info(const cdvz_gpu_index* idx, int* count, int* mode_id, uint32_t* model_crc, int* components,
                        long long* total_codes) {
  if (!idx) return CDVZ_GPU_USAGE;
  if (count) *count = idx->items.view.n;
  if (mode_id) *mode_id = idx->items.mode;
  if (model_crc) *model_crc = idx->items.model_crc;
  if (components) *components = idx->items.nc;
  if (total_codes) *total_codes = idx->items.total_codes;
  return CDVZ_GPU_OK;
}

int cdvz_gpu_retrieve(cdvz_gpu_index* idx, const uint8_t* qblob, const size_t* qoff, int nq, double ratio_test,
                      int rerank_depth, int max_results, int32_t* out_items, double* out_scores) {
  return guarded_index(idx, [&] {
    if (!idx || !qblob || !qoff || !out_items || !out_scores) throw UsageError("null argument");
    if (nq <= 0) return;
    CDVZ_CUDA_CHECK(cudaSetDevice(idx->device));
    const int n = idx->items.view.n;
    const int head = std::min(n, std::max(0, rerank_depth));
    const int mr = max_results <= 0 ? n : std::min(n, max_results);
    DecodedSet qs;
    qs.decode(qblob, qoff, nq, idx->st, "query batch");
    check_queries(idx, qs);
    // Queries run in chunks: qc * n stays below 2^31 (CUB's segment offsets
    // are int) and qc within the grid's y limit; ~24 B of sort buffers per
    // (query, item) pair bound a chunk to ~6 GB.
    const long long cap_pairs = std::min<long long>(0x7fffffffLL, 1LL << 28);
    long long qmax = 65535;
    if (const char* e = std::getenv("CDVZ_GPU_RETRIEVE_QCHUNK")) qmax = std::max(1LL, std::min(qmax, std::atoll(e)));  // tests
    const int qc = int(std::max<long long>(1, std::min<long long>({(long long)nq, qmax, cap_pairs / std::max(1, n)})));
    const size_t tot = size_t(qc) * size_t(n);
    idx->keys.ensure(sizeof(unsigned long long) * tot);
    idx->vals.ensure(sizeof(int) * tot);
    idx->keys2.ensure(sizeof(unsigned long long) * tot);
    idx->vals2.ensure(sizeof(int) * tot);
    idx->seg.ensure(sizeof(int) * (size_t(qc) + 1));
    idx->local.ensure(sizeof(int) * std::max<size_t>(1, size_t(qc) * size_t(head)));
    idx->out_i.ensure(sizeof(int) * size_t(nq) * size_t(mr));
    idx->out_s.ensure(sizeof(double) * size_t(nq) * size_t(mr));
    std::vector<int> seg(size_t(qc) + 1);
    for (int q = 0; q <= qc; ++q) seg[size_t(q)] = q * n;
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(idx->seg.p, seg.data(), sizeof(int) * seg.size(), cudaMemcpyHostToDevice, idx->st));
    const int mc = std::max(1, std::max(qs.max_codes, idx->items.max_codes));
    for (int q0 = 0; q0 < nq; q0 += qc) {
      const int nqc = std::min(qc, nq - q0);
      const int ntot = nqc * n;
      k_global_keys<<<dim3((n + 255) / 256, nqc), 256, 0, idx->st>>>(qs.view, idx->items.view, idx->perm.as<int>(), n,
                                                                      idx->items.nc, q0,
                                                                      idx->keys.as<unsigned long long>(),
                                                                      idx->vals.as<int>());
      CDVZ_CUDA_CHECK(cudaGetLastError());
      // Stable descending sort by similarity within each query: items enter in
      // ascending id order, so ties keep ascending ids (eval.cpp:91-94).
      size_t temp_bytes = 0;
      CDVZ_CUDA_CHECK(cub::DeviceSegmentedRadixSort::SortPairsDescending(
          nullptr, temp_bytes, idx->keys.as<unsigned long long>(), idx->keys2.as<unsigned long long>(),
          idx->vals.as<int>(), idx->vals2.as<int>(), ntot, nqc, idx->seg.as<int>(), idx->seg.as<int>() + 1, 0, 64,
          idx->st));
      idx->temp.ensure(temp_bytes);
      CDVZ_CUDA_CHECK(cub::DeviceSegmentedRadixSort::SortPairsDescending(
          idx->temp.p, temp_bytes, idx->keys.as<unsigned long long>(), idx->keys2.as<unsigned long long>(),
          idx->vals.as<int>(), idx->vals2.as<int>(), ntot, nqc, idx->seg.as<int>(), idx->seg.as<int>() + 1, 0, 64,
          idx->st));
      if (head > 0) {
        const size_t sm = lm_smem_bytes(mc);
        CDVZ_CUDA_CHECK(cudaFuncSetAttribute(k_local_head, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k_local_head<<<dim3(head, nqc), kLMThreads, sm, idx->st>>>(qs.view, idx->items.view, idx->vals2.as<int>(), n,
                                                                    head, ratio_test, mc, q0, idx->local.as<int>());
        CDVZ_CUDA_CHECK(cudaGetLastError());
      }
      k_finish<<<nqc, kFinishThreads, 0, idx->st>>>(idx->keys2.as<unsigned long long>(), idx->vals2.as<int>(), idx->local.as<int>(),
                                        idx->id_rank.as<int>(), n, head, mr, q0, idx->out_i.as<int>(),
                                        idx->out_s.as<double>());
      CDVZ_CUDA_CHECK(cudaGetLastError());
    }
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(out_items, idx->out_i.p, sizeof(int) * size_t(nq) * size_t(mr), cudaMemcpyDeviceToHost,
                                    idx->st));
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(out_scores, idx->out_s.p, sizeof(double) * size_t(nq) * size_t(mr),
                                    cudaMemcpyDeviceToHost, idx->st));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(idx->st));
  });
}

int cdvz_gpu_match_pairs(cdvz_gpu_index* idx, const uint8_t* qblob, const size_t* qoff, int nq, const int32_t* pairs,
                         int np, double ratio_test, double* global_sim, int32_t* local_matches) {
  return guarded_index(idx, [&] {
    if (!idx || !qblob || !qoff || (!pairs && np > 0) || (np > 0 && (!global_sim || !local_matches)))
      throw UsageError("null argument");
    if (np <= 0) return;
    CDVZ_CUDA_CHECK(cudaSetDevice(idx->device));
    DecodedSet qs;
    qs.decode(qblob, qoff, nq, idx->st, "query batch");
    check_queries(idx, qs);
    for (int k = 0; k < np; ++k)
      if (pairs[2 * k] < 0 || pairs[2 * k] >= nq || pairs[2 * k + 1] < 0 || pairs[2 * k + 1] >= idx->items.view.n)
        throw UsageError("pair index out of range");
    idx->pairs.ensure(sizeof(int) * 2 * size_t(np));
    idx->psim.ensure(sizeof(double) * size_t(np));
    idx->ploc.ensure(sizeof(int) * size_t(np));
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(idx->pairs.p, pairs, sizeof(int) * 2 * size_t(np), cudaMemcpyHostToDevice, idx->st));
    const int mc = std::max(1, std::max(qs.max_codes, idx->items.max_codes));
    const size_t sm = lm_smem_bytes(mc);
    CDVZ_CUDA_CHECK(cudaFuncSetAttribute(k_match_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    k_match_pairs<<<np, kLMThreads, sm, idx->st>>>(qs.view, idx->items.view, idx->pairs.as<int>(), idx->items.nc,
                                                    ratio_test, mc, idx->psim.as<double>(), idx->ploc.as<int>());
    CDVZ_CUDA_CHECK(cudaGetLastError());
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(global_sim, idx->psim.p, sizeof(double) * size_t(np), cudaMemcpyDeviceToHost, idx->st));
    CDVZ_CUDA_CHECK(cudaMemcpyAsync(local_matches, idx->ploc.p, sizeof(int) * size_t(np), cudaMemcpyDeviceToHost, idx->st));
    CDVZ_CUDA_CHECK(cudaStreamSynchronize(idx->st));
  });
}

}  // extern "C"
