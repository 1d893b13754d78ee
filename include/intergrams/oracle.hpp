// intergrams/oracle.hpp — drop-in for /root/reference/proj/include/intergrams/oracle.hpp
// (naive_count / naive_topk, src/oracle.cpp:7-47).  The exact counting runs
// on the GPU (sort + run-length reduction, ig_naive_topk in
// include/intergrams_b200.h); naive_topk over a map is the reference's host
// step.  Header-only; link with libintergrams_b200.so.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>

#include "intergrams/corpus.hpp"
#include "intergrams/counting.hpp"
#include "intergrams/intergrams.hpp"
#include "intergrams_b200.h"

namespace intergrams {

using GramCountMap = std::unordered_map<std::string, uint64_t>;

inline constexpr uint64_t kOracleCorpusGuard = 256ull << 20;  // 256 MB (oracle.hpp:17)

namespace detail {
inline TopKList exact_topk(const Corpus& corpus, size_t n, CountMode mode, uint64_t k,
                           uint64_t max_corpus_bytes, int device) {
  const CorpusCSR csr = corpus.materialize();
  ig_corpus c{csr.data.data(), csr.offsets.data(), csr.offsets.size() - 1, IG_HOST};
  ig_result r{};
  char err[1024] = {0};
  raise(ig_naive_topk(&c, static_cast<uint32_t>(n), k, mode == CountMode::kAll ? IG_MODE_ALL : IG_MODE_ONCE,
                      max_corpus_bytes, device, &r, err, sizeof(err)),
        err);
  IntergramsResult out = convert(r);
  ig_result_free(&r);
  return std::move(out.topk);
}
}  // namespace detail

// Exact per-gram counts (every distinct gram).  ConfigError once the corpus
// exceeds max_corpus_bytes (oracle.cpp:14-18) or for n > 8 (packed-u64 GPU keys).
inline GramCountMap naive_count(const Corpus& corpus, size_t n, CountMode mode,
                                uint64_t max_corpus_bytes = kOracleCorpusGuard, int device = -1) {
  if (n < 1) throw ConfigError("gram length must be >= 1");
  GramCountMap map;
  for (auto& gc : detail::exact_topk(corpus, n, mode, ~0ull, max_corpus_bytes, device))
    map.emplace(std::move(gc.gram), gc.count);
  return map;
}

// Canonical top-k of a count map (oracle.cpp:37-47).
inline TopKList naive_topk(const GramCountMap& map, size_t k) {
  if (k < 1) throw ConfigError("top-k requires k >= 1");
  TopKList list;
  list.reserve(map.size());
  for (const auto& [gram, count] : map) list.push_back(GramCount{gram, count});
  canonical_sort(list);
  if (list.size() > k) list.resize(k);
  return list;
}

// naive_topk(naive_count(corpus, n, mode, guard), k) in one GPU call (the
// top-k is selected on the device; only k entries come back).
inline TopKList naive_topk(const Corpus& corpus, size_t n, CountMode mode, size_t k,
                           uint64_t max_corpus_bytes = kOracleCorpusGuard, int device = -1) {
  if (n < 1) throw ConfigError("gram length must be >= 1");
  return detail::exact_topk(corpus, n, mode, k, max_corpus_bytes, device);
}

}  // namespace intergrams
