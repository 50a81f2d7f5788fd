// K2/K3 — per-frame keypoint list assembly and K4 — relevance selection.
//
// k_merge_octave (one CTA per frame) restores the reference's candidate order
// and applies cross-octave dedup:
//   * rank: a survivor's position in (y, x, sigma) order is the number of set
//     bits before its key in the octave's raster bitmap (k_octave set them),
//     which reproduces std::sort in detect_extrema (scale_space.cpp:207-213)
//     followed by the order-preserving filter of refine_candidates (:267-269);
//   * dedup (scale_space.cpp:272-302): previous points are bucketed in an
//     8 px grid (the pair test needs |dx|,|dy| < 2, so the 3x3 neighbourhood
//     of buckets holds every candidate pair), decisions are the reference's
//     per pair and order-independent; survivors are compacted previous-first.
// k_select (one CTA per frame) fills the centre distance, scores the five
// lookup tables (relevance.cpp:24-30, 54-69) and takes the top select_n by
// the reference's total order (score desc, |p| desc, y, x, index;
// relevance.cpp:71-93) with an exact MSB-first radix select on the 5-field
// key, then a bitonic sort of the winners.
#include <algorithm>
#include <cstddef>

#include "common.cuh"

namespace cdvz_gpu {

namespace {

constexpr int kMergeThreads = 1024;
constexpr size_t kMergeSmemBudget = 200 * 1024;  // dynamic shared memory of k_merge_octave

// Block-wide exclusive scan over one int per thread (1024 threads).
__device__ int block_exclusive_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += n;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int x = lane < nw ? warp_tot[lane] : 0;
    int xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += n;
    }
    if (lane < nw) warp_tot[lane] = xi - x;
    if (lane == nw - 1) warp_tot[32] = xi;
  }
  __syncthreads();
  const int res = warp_tot[wid] + incl - v;
  total = warp_tot[32];
  __syncthreads();
  return res;
}

// Order-preserving compaction of `n` flags (keep != 0) into dst positions:
// pos[i] = number of kept before i. Elements go in rounds of blockDim.x
// consecutive indices (thread t takes element round + t), so the emits of a
// warp touch consecutive records.
template <class Keep, class Emit>
__device__ int compact(int n, Keep keep, Emit emit, int* warp_tot) {
  int base = 0;
  for (int r0 = 0; r0 < n; r0 += blockDim.x) {
    const int i = r0 + threadIdx.x;
    const bool k = i < n && keep(i);
    int total = 0;
    const int pos = block_exclusive_scan(k ? 1 : 0, warp_tot, total);
    if (k) emit(i, base + pos);
    base += total;
  }
  return base;
}

}  // namespace

// Restores octave o's survivor order and merges it into the accumulated list.
__global__ void __launch_bounds__(kMergeThreads) k_merge_octave(Batch bt, int o) {
  extern __shared__ int sm[];
  __shared__ int warp_tot[33];
  const int f = blockIdx.x;
  const int w = bt.ow[o], h = bt.oh[o];
  const int nwords = (2 * w * h + 31) / 32;
  uint32_t* bm = bt.bitmap + f * bt.bitmap_words + bt.bm_off[o];
  int n = bt.raw_count[f * bt.n_oct + o];
  if (n > bt.cap_oct) n = bt.cap_oct;
  const KP* raw = bt.raw + ((long long)f * bt.n_oct + o) * bt.cap_oct;

  // Exclusive popcount prefix of the bitmap, per word: thread t owns a
  // contiguous run of 16-byte groups (plan() pads every octave's bitmap to
  // whole groups), counts it, a block scan places the runs, and a second read
  // of the run (L1) writes its prefixes — two vector loads and four popcounts
  // per group, no per-word shuffles.
  // In shared memory when it fits (merge_smem_bytes), else in global scratch.
  const int n4 = (nwords + 3) >> 2;
  int* prefix = (size_t(4 * n4) * sizeof(int) <= kMergeSmemBudget) ? sm : bt.bm_prefix + f * bt.bitmap_words + bt.bm_off[o];
  uint4* bm4 = reinterpret_cast<uint4*>(bm);
  {
    const int per = (n4 + int(blockDim.x) - 1) / int(blockDim.x);
    const int g0 = min(n4, int(threadIdx.x) * per), g1 = min(n4, g0 + per);
    int cnt = 0;
    for (int g = g0; g < g1; ++g) {
      const uint4 v = bm4[g];
      cnt += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    int total = 0;
    int run = block_exclusive_scan(cnt, warp_tot, total);
    int4* p4 = reinterpret_cast<int4*>(prefix);
    for (int g = g0; g < g1; ++g) {
      const uint4 v = bm4[g];
      int4 q;
      q.x = run;
      q.y = q.x + __popc(v.x);
      q.z = q.y + __popc(v.y);
      q.w = q.z + __popc(v.z);
      run = q.w + __popc(v.w);
      p4[g] = q;
    }
  }
  __syncthreads();

  const int src = (o + 1) & 1, dst = o & 1;  // acc ping-pong: octave o writes acc[o & 1]
  KP* out_sorted = (o == 0) ? bt.acc[dst] + (long long)f * bt.cap_acc : bt.cur + (long long)f * bt.cap_acc;
  if (n <= bt.cap_acc) {
    // Ranks from the keys alone, then the 64-byte records move in 16-byte
    // pieces by consecutive threads (coalesced stores; each record's four
    // pieces are one contiguous read).
    int* src_of = bt.scratch_idx + (long long)f * bt.cap_acc;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t key = raw[i].key;
      const uint32_t word = key >> 5, bit = key & 31u;
      src_of[prefix[word] + __popc(bm[word] & ((1u << bit) - 1u))] = i;
    }
    __syncthreads();
    // Every rank is known, so the bitmap can be cleared for the next batch on
    // the way: only the words holding a survivor's bit are non-zero, and
    // each record's last piece carries its key (one store per survivor).
    static_assert(offsetof(KP, key) == 60, "KP key in the last 4 bytes");
    const uint4* s4 = reinterpret_cast<const uint4*>(raw);
    uint4* d4 = reinterpret_cast<uint4*>(out_sorted);
    for (int c = threadIdx.x; c < 4 * n; c += blockDim.x) {
      const uint4 v = s4[4 * src_of[c >> 2] + (c & 3)];
      d4[c] = v;
      if ((c & 3) == 3) bm[v.w >> 5] = 0u;
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const KP k = raw[i];
      const uint32_t word = k.key >> 5, bit = k.key & 31u;
      const int rank = prefix[word] + __popc(bm[word] & ((1u << bit) - 1u));
      out_sorted[rank] = k;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) bm[raw[i].key >> 5] = 0u;  // ready for the next batch
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bt.raw_count[f * bt.n_oct + o] = 0;
    bt.oct_count[f * bt.n_oct + o] = n;
  }

  if (o == 0) {
    if (threadIdx.x == 0) bt.acc_count[f * 2 + dst] = n;
    return;
  }

  // ---- dedup against the accumulated list (scale_space.cpp:272-302)
  const KP* prev = bt.acc[src] + (long long)f * bt.cap_acc;
  const int np = bt.acc_count[f * 2 + src];
  const KP* cur = out_sorted;
  const int nc = n;
  const int cell_px = bt.merge_cell;
  const double inv_cell = 1.0 / cell_px;
  const int gw = bt.W / cell_px + 3, gh = bt.H / cell_px + 3;
  int* cell_start = sm;                  // gw*gh + 1 (reuses the prefix space)
  int* cell_fill = sm + gw * gh + 1;     // gw*gh
  uint8_t* drop_prev = bt.flags + (long long)f * 2 * bt.cap_acc;
  uint8_t* drop_cur = drop_prev + bt.cap_acc;
  int* sorted_idx = bt.scratch_idx + (long long)f * bt.cap_acc;
  auto cell_of = [&](double x, double y) {
    int cxi = int(floor(x * inv_cell)) + 1, cyi = int(floor(y * inv_cell)) + 1;
    cxi = max(0, min(gw - 1, cxi));
    cyi = max(0, min(gh - 1, cyi));
    return cyi * gw + cxi;
  };
  for (int i = threadIdx.x; i < gw * gh; i += blockDim.x) cell_fill[i] = 0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) drop_prev[i] = 0;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) drop_cur[i] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < np; j += blockDim.x) atomicAdd(&cell_fill[cell_of(prev[j].x, prev[j].y)], 1);
  __syncthreads();
  {
    const int ncell = gw * gh;
    const int per = (ncell + blockDim.x - 1) / blockDim.x;
    const int lo = min(ncell, int(threadIdx.x) * per), hi = min(ncell, lo + per);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += cell_fill[i];
    int total = 0;
    int run = block_exclusive_scan(cnt, warp_tot, total);
    for (int i = lo; i < hi; ++i) {
      cell_start[i] = run;
      run += cell_fill[i];
    }
    if (threadIdx.x == 0) cell_start[ncell] = total;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < gw * gh; i += blockDim.x) cell_fill[i] = cell_start[i];
  __syncthreads();
  for (int j = threadIdx.x; j < np; j += blockDim.x) {
    const int pos = atomicAdd(&cell_fill[cell_of(prev[j].x, prev[j].y)], 1);
    sorted_idx[pos] = j;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const KP c = cur[i];
    const int cc = cell_of(c.x, c.y);
    const int ccx = cc % gw, ccy = cc / gw;
    bool dc = false;
    for (int yy = max(0, ccy - 1); yy <= min(gh - 1, ccy + 1); ++yy)
      for (int xx = max(0, ccx - 1); xx <= min(gw - 1, ccx + 1); ++xx) {
        const int cell = yy * gw + xx;
        for (int q = cell_start[cell]; q < cell_start[cell + 1]; ++q) {
          const int j = sorted_idx[q];
          const KP pj = prev[j];
          const double dx = c.x - pj.x, dy = c.y - pj.y;
          if (dx * dx + dy * dy >= 4.0) continue;
          const double ratio = c.sigma / pj.sigma;
          if (!(ratio >= 1.0 / 1.3 && ratio <= 1.3)) continue;
          if (fabs(pj.p) >= fabs(c.p)) dc = true;
          else drop_prev[j] = 1;
        }
      }
    drop_cur[i] = dc ? 1 : 0;
  }
  __syncthreads();
  // Survivors: previous first, then current, each in order. The positions
  // are scanned first (source index per output slot, in the now free
  // sorted_idx scratch), then the 64-byte records move in 16-byte pieces by
  // consecutive threads with no barrier in between.
  KP* out = bt.acc[dst] + (long long)f * bt.cap_acc;
  const int cap = bt.cap_acc;
  int* src_of = sorted_idx;
  auto move = [&](const KP* from, int count, int at) {
    const uint4* s4 = reinterpret_cast<const uint4*>(from);
    uint4* d4 = reinterpret_cast<uint4*>(out + at);
    const int m = min(count, cap - at);
    for (int c = threadIdx.x; c < 4 * m; c += blockDim.x) d4[c] = s4[4 * src_of[c >> 2] + (c & 3)];
  };
  const int kept_prev = compact(
      np, [&](int i) { return drop_prev[i] == 0; }, [&](int i, int pos) { src_of[pos] = i; }, warp_tot);
  __syncthreads();
  move(prev, kept_prev, 0);
  __syncthreads();
  const int kept_cur = compact(
      nc, [&](int i) { return drop_cur[i] == 0; }, [&](int i, int pos) { src_of[pos] = i; }, warp_tot);
  __syncthreads();
  if (kept_prev < cap) move(cur, kept_cur, kept_prev);
  if (threadIdx.x == 0) {
    int total = kept_prev + kept_cur;
    if (total > bt.cap_acc) {
      total = bt.cap_acc;
      atomicOr(&bt.status[f], 4);
    }
    bt.acc_count[f * 2 + dst] = total;
  }
}

// Dedup grid cell side: 8 px, doubled until the two per-cell int arrays fit
// the shared-memory budget (any side >= 2 keeps every pair with |dx|, |dy| < 2
// inside the 3x3 neighbourhood of cells).
int merge_cell_px(int W, int H) {
  int c = 8;
  while (sizeof(int) * (2 * size_t(W / c + 3) * size_t(H / c + 3) + 1) > kMergeSmemBudget) c *= 2;
  return c;
}

// Dynamic shared memory of octave o's merge: its bitmap prefix (when it fits)
// and, above octave 0, the dedup grid that reuses the same space.
size_t merge_smem_bytes(const Batch& bt, int o) {
  const size_t words = ((size_t(2) * bt.ow[o] * bt.oh[o] + 31) / 32 + 3) & ~size_t(3);  // padded to 16-byte groups
  const size_t need = words * sizeof(int) <= kMergeSmemBudget ? words : 0;  // else global prefix
  const size_t cells = size_t(bt.W / bt.merge_cell + 3) * (bt.H / bt.merge_cell + 3);
  const size_t grid = o > 0 ? 2 * cells + 1 : 0;
  return sizeof(int) * std::max<size_t>(1, need > grid ? need : grid);
}

cudaError_t launch_merge(const Batch& bt, int o, cudaStream_t st) {
  const size_t smem = merge_smem_bytes(bt, o);
  static size_t configured[kMaxDevices] = {};
  const cudaError_t e = once_per_device(configured, smem, [&] {
    return cudaFuncSetAttribute(k_merge_octave, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  });
  if (e != cudaSuccess) return e;
  k_merge_octave<<<bt.nframes, kMergeThreads, smem, st>>>(bt, o);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- selection

namespace {

// upper_bound over edges, clamped (relevance.cpp:24-30).
__device__ __forceinline__ double lut(const double* edges, const double* vals, int nb, double x) {
  int lo = 0, hi = nb + 1;  // first index with edges[idx] > x in [0, nb+1]
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (edges[mid] > x) hi = mid;
    else lo = mid + 1;
  }
  int bin = lo - 1;
  bin = bin < 0 ? 0 : (bin > nb - 1 ? nb - 1 : bin);
  return vals[bin];
}

// The five 64-bit words of the reference's total order, ascending = better.
struct SelKey { unsigned long long k[5]; };

// k_select's dynamic shared memory: winner indices, then (16-byte aligned)
// their keys and ranks.
constexpr int kRankSortMax = 2048;  // winners rank-sorted with their keys in shared memory (104 KB at the limit)
__host__ __device__ inline size_t select_key_offset(int select_n) {
  return (size_t(select_n) * sizeof(int) + 15) & ~size_t(15);
}

__device__ __forceinline__ SelKey sel_key(double score, const KP& p, int idx) {
  SelKey s;
  // score >= 0; + 0.0 maps a -0.0 (a relevance value of -0.0 passes the
  // bundle's [0, 1] check) to +0.0, which the reference's comparisons treat alike.
  s.k[0] = ~static_cast<unsigned long long>(__double_as_longlong(score + 0.0));
  s.k[1] = ~static_cast<unsigned long long>(__double_as_longlong(fabs(p.p)));  // |p| >= 0
  // y, x >= 0 after refinement (margin >= 2), so their bit patterns order like the values.
  s.k[2] = static_cast<unsigned long long>(__double_as_longlong(p.y));
  s.k[3] = static_cast<unsigned long long>(__double_as_longlong(p.x));
  s.k[4] = static_cast<unsigned long long>(idx);
  return s;
}

__device__ __forceinline__ bool key_less(const SelKey& a, const SelKey& b) {
#pragma unroll
  for (int i = 0; i < 5; ++i)
    if (a.k[i] != b.k[i]) return a.k[i] < b.k[i];
  return false;
}

}  // namespace

__global__ void __launch_bounds__(kMergeThreads) k_select(Batch bt, Model md, EncodeConst ec) {
  extern __shared__ unsigned char ssm[];
  __shared__ int warp_tot[33];
  __shared__ int hist[256];
  __shared__ int s_remaining, s_digit, s_done;
  const int f = blockIdx.x;
  const int last = (bt.n_oct - 1) & 1;
  KP* acc = bt.acc[last] + (long long)f * bt.cap_acc;
  const int n = bt.n_oct > 0 ? bt.acc_count[f * 2 + last] : 0;
  const int want = min(n, bt.select_n);
  double* score = bt.scratch_d + (long long)f * bt.cap_acc;
  uint8_t* state = bt.flags + (long long)f * 2 * bt.cap_acc;  // 0 alive, 1 selected, 2 rejected

  // fill_center_distance + relevance product (relevance.cpp:54-69)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    KP k = acc[i];
    const double dist = hypot(k.x - ec.cx, k.y - ec.cy);
    k.d = ec.half_diag > 0.0 ? fmin(dist / ec.half_diag, 1.0) : 0.0;
    acc[i].d = k.d;
    double s = 1.0;
    s *= lut(md.rel_edges[0], md.rel_vals[0], md.rel_nb[0], k.sigma);
    s *= lut(md.rel_edges[1], md.rel_vals[1], md.rel_nb[1], k.p);
    s *= lut(md.rel_edges[2], md.rel_vals[2], md.rel_nb[2], k.d);
    s *= lut(md.rel_edges[3], md.rel_vals[3], md.rel_nb[3], k.rho);
    s *= lut(md.rel_edges[4], md.rel_vals[4], md.rel_nb[4], k.pss);
    score[i] = s;
    state[i] = 0;
  }
  if (threadIdx.x == 0) {
    s_remaining = want;
    s_done = (want == n) ? 1 : 0;
  }
  __syncthreads();
  if (n > want) {
    // MSB-first radix select over the 320-bit key (8-bit digits).
    for (int digit = 0; digit < 40 && !s_done; ++digit) {
      const int word = digit >> 3, shift = 56 - 8 * (digit & 7);
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      // Word 0 (the score) needs no keypoint record.
      auto key_word = [&](int i) {
        return word == 0 ? ~static_cast<unsigned long long>(__double_as_longlong(score[i]))
                         : sel_key(score[i], acc[i], i).k[word];
      };
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (state[i] == 0) atomicAdd(&hist[(key_word(i) >> shift) & 0xFF], 1);
      __syncthreads();
      if (threadIdx.x < 32) {
        // First digit whose inclusive count reaches the remaining quota: lane l
        // owns bins 8l .. 8l + 7; a warp scan of the lane sums finds the lane,
        // which then walks its eight bins (the sequential scan's answer).
        const int l = threadIdx.x, rem = s_remaining;
        int own = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) own += hist[8 * l + q];
        int incl = own;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, d);
          if (l >= d) incl += v;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, incl >= rem);
        const int first = __ffs(hit) - 1;  // rem <= alive count, so some lane reaches it
        if (l == first) {
          int run = incl - own, d = 8 * l;
          for (; d < 8 * l + 7; ++d) {
            if (run + hist[d] >= rem) break;
            run += hist[d];
          }
          s_digit = d;
          s_remaining = rem - run;
          if (hist[d] == rem - run) s_done = 2;  // the whole bucket fits exactly
        }
      }
      __syncthreads();
      const int dsel = s_digit;
      const bool take_bucket = s_done == 2;
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (state[i] == 0) {
          const int dv = int((key_word(i) >> shift) & 0xFF);
          if (dv < dsel || (dv == dsel && take_bucket)) state[i] = 1;
          else if (dv > dsel) state[i] = 2;
        }
      __syncthreads();
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) state[i] = 1;
    __syncthreads();
  }
  // Gather winners (any order), then order them by the full key. Up to
  // kRankSortMax winners: a rank sort (keys are unique — the index is the last
  // word), each winner's rank counted over chunks of the others by several
  // threads, three barriers in all; larger selection budgets: a bitonic
  // network on the indices (shared memory for the keys would not fit).
  int* win = reinterpret_cast<int*>(ssm);
  const int got = compact(
      n, [&](int i) { return state[i] == 1; }, [&](int i, int pos) { win[pos] = i; }, warp_tot);
  __syncthreads();
  KP* sel = bt.sel + (long long)f * bt.select_n;
  if (bt.select_n <= kRankSortMax) {
    SelKey* wkey = reinterpret_cast<SelKey*>(ssm + select_key_offset(bt.select_n));
    int* rnk = reinterpret_cast<int*>(wkey + bt.select_n);
    for (int i = threadIdx.x; i < got; i += blockDim.x) {
      wkey[i] = sel_key(score[win[i]], acc[win[i]], win[i]);
      rnk[i] = 0;
    }
    __syncthreads();
    const int chunks = got > 0 ? max(1, int(blockDim.x) / got) : 1;
    for (int t = threadIdx.x; t < got * chunks; t += blockDim.x) {
      const int i = t % got, c = t / got;
      const int j0 = c * got / chunks, j1 = (c + 1) * got / chunks;
      const SelKey ki = wkey[i];
      int r = 0;
      for (int j = j0; j < j1; ++j) r += key_less(wkey[j], ki) ? 1 : 0;
      atomicAdd(&rnk[i], r);
    }
    __syncthreads();
    // Sorted source list, then the records move as coalesced 16-byte pieces.
    int* src = rnk + bt.select_n;
    for (int i = threadIdx.x; i < got; i += blockDim.x) src[rnk[i]] = win[i];
    __syncthreads();
    const uint4* s4 = reinterpret_cast<const uint4*>(acc);
    uint4* d4 = reinterpret_cast<uint4*>(sel);
    for (int c = threadIdx.x; c < 4 * got; c += blockDim.x) d4[c] = s4[4 * src[c >> 2] + (c & 3)];
  } else {
    int P = 1;
    while (P < got) P <<= 1;
    for (int i = got + threadIdx.x; i < P; i += blockDim.x) win[i] = -1;
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int j = i ^ stride;
          if (j > i) {
            const int a = win[i], b = win[j];
            bool a_after_b;
            if (a < 0) a_after_b = b >= 0;
            else if (b < 0) a_after_b = false;
            else a_after_b = key_less(sel_key(score[b], acc[b], b), sel_key(score[a], acc[a], a));
            const bool up = (i & size) == 0;
            if (up == a_after_b) {
              win[i] = b;
              win[j] = a;
            }
          }
        }
        __syncthreads();
      }
    for (int r = threadIdx.x; r < got; r += blockDim.x) sel[r] = acc[win[r]];
  }
  if (threadIdx.x == 0) bt.sel_count[f] = got;
}

size_t select_smem_bytes(const Batch& bt) {
  if (bt.select_n <= kRankSortMax)
    return select_key_offset(bt.select_n) + size_t(bt.select_n) * (sizeof(SelKey) + 2 * sizeof(int));
  size_t p = 1;
  while (p < size_t(bt.select_n)) p <<= 1;
  return p * sizeof(int);
}


cudaError_t launch_select(const Batch& bt, const Model& md, const EncodeConst& ec, cudaStream_t st) {
  const size_t smem = select_smem_bytes(bt);
  cudaError_t e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k_select<<<bt.nframes, kMergeThreads, smem, st>>>(bt, md, ec);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
