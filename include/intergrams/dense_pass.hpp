// intergrams/dense_pass.hpp — drop-in for
// /root/reference/proj/include/intergrams/dense_pass.hpp (src/dense_pass.cpp):
// the exact dense pass over all 256^n grams, n in [1, 3], counted on the GPU
// (ig_count_dense) and selected on the GPU (ig_top_k).  Header-only.
#pragma once

#include <string>

#include "intergrams/corpus.hpp"
#include "intergrams/counting.hpp"
#include "intergrams/intergrams.hpp"
#include "intergrams/pipeline.hpp"
#include "intergrams_b200.h"

namespace intergrams {

inline constexpr size_t kMaxDenseGramLen = 3;

inline size_t dense_capacity(size_t n) {  // dense_pass.cpp:5-10
  if (n < 1 || n > kMaxDenseGramLen) throw ConfigError("dense pass supports gram lengths 1..3");
  return size_t{1} << (8 * n);
}

inline std::string dense_gram(size_t id, size_t n) {  // dense_pass.cpp:12-19
  std::string gram(n, '\0');
  for (size_t i = n; i-- > 0;) {
    gram[i] = static_cast<char>(id & 0xff);
    id >>= 8;
  }
  return gram;
}

// Exact counts over the full 256^n space (dense_pass.cpp:21-39).
inline CountTable count_dense(const Corpus& corpus, size_t n, const CountingOptions& opt,
                              int device = -1) {
  CountTable table(dense_capacity(n));
  const CorpusCSR csr = corpus.materialize();
  ig_corpus c{csr.data.data(), csr.offsets.data(), csr.offsets.size() - 1, IG_HOST};
  char err[1024] = {0};
  detail::raise(ig_count_dense(&c, static_cast<uint32_t>(n),
                               opt.mode == CountMode::kAll ? IG_MODE_ALL : IG_MODE_ONCE, device,
                               table.data(), err, sizeof(err)),
                err);
  return table;
}

// Canonical top-k of a dense table (dense_pass.cpp:41-43), on the GPU.
inline TopKList topk_dense(const CountTable& table, size_t n, size_t k, int device = -1) {
  if (k < 1) throw ConfigError("top_k requires k >= 1");
  const size_t kk = std::min<size_t>(k, table.capacity());
  std::vector<uint64_t> keys(kk + 1), counts(kk + 1);
  uint64_t len = 0;
  char err[1024] = {0};
  detail::raise(ig_top_k(table.raw().data(), table.capacity(), k, nullptr, device, keys.data(),
                         counts.data(), &len, err, sizeof(err)),
                err);
  TopKList out;
  for (uint64_t i = 0; i < len; ++i) out.push_back(GramCount{dense_gram(keys[i], n), counts[i]});
  return out;
}

inline CountTable count_trigrams(const Corpus& corpus, const CountingOptions& opt) {
  return count_dense(corpus, 3, opt);
}
inline TopKList topk_trigrams(const CountTable& table, size_t k_prime) {
  return topk_dense(table, 3, k_prime);
}

}  // namespace intergrams
