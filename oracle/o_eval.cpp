// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Compressed-domain matching and retrieval restated from the reference:
// nearest_of / passes_ratio / count_local_matches / match_pair / retrieve
// (proj/src/eval.cpp:17-124). Integer distances, the ratio test in double and
// the (score, id) orderings follow the reference exactly.
#include <algorithm>
#include <limits>

#include "oracle.hpp"

namespace orc {

namespace {

struct Nearest {  // eval.cpp:18-23
  int best = -1;
  int best_dist = std::numeric_limits<int>::max();
  int second_dist = std::numeric_limits<int>::max();
};

Nearest nearest_of(const TernaryCode& code, const std::vector<TernaryCode>& pool) {  // eval.cpp:25-37
  Nearest n;
  for (std::size_t j = 0; j < pool.size(); ++j) {
    const int d = ternary_distance(code, pool[j]);
    if (d < n.best_dist) {
      n.second_dist = n.best_dist;
      n.best_dist = d;
      n.best = static_cast<int>(j);
    } else if (d < n.second_dist) {
      n.second_dist = d;
    }
  }
  return n;
}

bool passes_ratio(const Nearest& n, std::size_t pool_size, double ratio) {  // eval.cpp:39-43
  if (n.best < 0) return false;
  if (pool_size < 2) return true;
  return n.best_dist < ratio * n.second_dist;
}

}  // namespace

int count_local_matches(const std::vector<TernaryCode>& a, const std::vector<TernaryCode>& b, double ratio) {
  // eval.cpp:47-64
  if (a.empty() || b.empty()) return 0;
  std::vector<Nearest> a_to_b(a.size()), b_to_a(b.size());
  for (std::size_t i = 0; i < a.size(); ++i) a_to_b[i] = nearest_of(a[i], b);
  for (std::size_t j = 0; j < b.size(); ++j) b_to_a[j] = nearest_of(b[j], a);
  int count = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const Nearest& fwd = a_to_b[i];
    if (!passes_ratio(fwd, b.size(), ratio)) continue;
    const Nearest& rev = b_to_a[static_cast<std::size_t>(fwd.best)];
    if (rev.best != static_cast<int>(i) || !passes_ratio(rev, a.size(), ratio)) continue;
    ++count;
  }
  return count;
}

MatchResult match_pair(const EncodedImage& a, const EncodedImage& b, const MatchOptions& opts) {  // eval.cpp:66-74
  if (a.model_crc != b.model_crc) throw DataError("containers were encoded with different model bundles");
  if (a.mode_id != b.mode_id) throw DataError("containers use different modes");
  MatchResult r;
  r.global_similarity = scfv_similarity(a.global_desc, b.global_desc);
  r.local_match_count = count_local_matches(a.codes, b.codes, opts.ratio_test);
  return r;
}

RankedList retrieve(const EncodedImage& query, const std::vector<std::pair<std::string, const EncodedImage*>>& index,
                    const MatchOptions& opts) {  // eval.cpp:76-124 (serial; the reference's Engine only fans out)
  if (index.empty()) throw DataError("retrieval index is empty");
  std::vector<double> sims(index.size());
  for (std::size_t i = 0; i < index.size(); ++i) {
    const EncodedImage& e = *index[i].second;
    if (e.model_crc != query.model_crc) throw DataError("index container was encoded with a different model bundle");
    if (e.mode_id != query.mode_id) throw DataError("index container mode mismatch");
    sims[i] = scfv_similarity(query.global_desc, e.global_desc);
  }
  std::vector<std::size_t> order(index.size());
  for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
    if (sims[x] != sims[y]) return sims[x] > sims[y];
    return index[x].first < index[y].first;
  });
  const std::size_t head = std::min<std::size_t>(order.size(), static_cast<std::size_t>(std::max(0, opts.rerank_depth)));
  std::vector<std::size_t> head_idx(order.begin(), order.begin() + static_cast<std::ptrdiff_t>(head));
  std::vector<int> local(head);
  for (std::size_t r = 0; r < head; ++r)
    local[r] = count_local_matches(query.codes, index[head_idx[r]].second->codes, opts.ratio_test);
  std::vector<std::size_t> head_rank(head);
  for (std::size_t r = 0; r < head; ++r) head_rank[r] = r;
  std::sort(head_rank.begin(), head_rank.end(), [&](std::size_t x, std::size_t y) {
    if (local[x] != local[y]) return local[x] > local[y];
    const std::size_t ix = head_idx[x], iy = head_idx[y];
    if (sims[ix] != sims[iy]) return sims[ix] > sims[iy];
    return index[ix].first < index[iy].first;
  });
  RankedList out;
  for (std::size_t r = 0; r < head; ++r) {
    const std::size_t i = head_idx[head_rank[r]];
    out.items.push_back({index[i].first, local[head_rank[r]] + (sims[i] + 1.0) / 2.0});
  }
  for (std::size_t r = head; r < order.size(); ++r) {
    const std::size_t i = order[r];
    out.items.push_back({index[i].first, (sims[i] + 1.0) / 2.0 - 1.0});
  }
  return out;
}

}  // namespace orc
