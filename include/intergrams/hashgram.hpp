// intergrams/hashgram.hpp — drop-in for /root/reference/proj/include/intergrams/hashgram.hpp
// (HashgramConfig :19-31, mix64 / hash_ngram :33-39, HashgramResult :69-72,
// run_hashgram :74, src/hashgram.cpp:325-383).  Both passes run on the GPU
// (ig_hashgram_topk); merge / workers / flush_batch_size / trie_second_pass
// never change results and are accepted unused.  BucketSet (:41-58) is the
// host membership test; topk_buckets (:60-66) selects on the GPU (ig_top_k).
#pragma once

#include <algorithm>
#include <cstdint>
#include <string_view>
#include <vector>

#include "intergrams/corpus.hpp"
#include "intergrams/counting.hpp"
#include "intergrams/intergrams.hpp"
#include "intergrams_b200.h"

namespace intergrams {

struct HashgramConfig {
  uint64_t buckets = uint64_t{1} << 31;  // B
  size_t n = 6;
  size_t k = 10000;
  CountMode mode = CountMode::kOnce;
  uint64_t seed = 0;
  MergeStrategy merge = MergeStrategy::kBatchedFlush;
  size_t workers = 1;
  size_t flush_batch_size = 8;
  bool trie_second_pass = false;
  int device = -1;  // CUDA ordinal (-1: current)

  void validate() const {  // hashgram.cpp:16-20
    if (buckets < 1) throw ConfigError("bucket count B must be >= 1");
    if (n < 1) throw ConfigError("gram length n must be >= 1");
    if (k < 1) throw ConfigError("k must be >= 1");
  }
};

inline uint64_t mix64(std::string_view bytes, uint64_t seed) {
  return ig_mix64(reinterpret_cast<const uint8_t*>(bytes.data()), bytes.size(), seed);
}

inline uint64_t hash_ngram(std::string_view gram, uint64_t seed, uint64_t buckets) {
  return mix64(gram, seed) % buckets;
}

// "h(x) in H": a dense bitset when B <= 2^32 buckets, else binary search
// over the sorted kept ids (hashgram.hpp:41-58).
class BucketSet {
 public:
  BucketSet(const std::vector<uint64_t>& kept, uint64_t bucket_count) {
    if (bucket_count <= (uint64_t{1} << 32)) {
      bits_.assign((bucket_count + 63) / 64, 0);
      for (uint64_t b : kept)
        if (b < bucket_count) bits_[b >> 6] |= uint64_t{1} << (b & 63);
    } else {
      sorted_ = kept;
      std::sort(sorted_.begin(), sorted_.end());
      sorted_.erase(std::unique(sorted_.begin(), sorted_.end()), sorted_.end());
    }
  }
  bool contains(uint64_t bucket) const {
    if (!bits_.empty()) return (bits_[bucket >> 6] >> (bucket & 63)) & 1;
    return std::binary_search(sorted_.begin(), sorted_.end(), bucket);
  }

 private:
  std::vector<uint64_t> bits_;
  std::vector<uint64_t> sorted_;
};

struct BucketCount {
  uint64_t bucket = 0;
  uint64_t count = 0;
};

// Top-k buckets, count descending then bucket id ascending (hashgram.hpp:60-66):
// the canonical selection with key = id, on the GPU.
inline std::vector<BucketCount> topk_buckets(const CountTable& table, size_t k, int device = -1) {
  if (k < 1) throw ConfigError("top_k requires k >= 1");
  std::vector<BucketCount> out;
  if (table.capacity() == 0) return out;
  const size_t kk = std::min<size_t>(k, table.capacity());
  std::vector<uint64_t> keys(kk + 1), counts(kk + 1);
  uint64_t len = 0;
  char err[1024] = {0};
  detail::raise(ig_top_k(table.raw().data(), table.capacity(), k, nullptr, device, keys.data(),
                         counts.data(), &len, err, sizeof(err)),
                err);
  out.reserve(len);
  for (uint64_t i = 0; i < len; ++i) out.push_back(BucketCount{keys[i], counts[i]});
  return out;
}

struct HashgramResult {
  TopKList topk;
  std::vector<PassResult> passes;
};

inline HashgramResult run_hashgram(const Corpus& corpus, const HashgramConfig& cfg) {
  cfg.validate();
  const CorpusCSR csr = corpus.materialize();
  ig_corpus c{csr.data.data(), csr.offsets.data(), csr.offsets.size() - 1, IG_HOST};
  ig_hashgram_params p{};
  p.buckets = cfg.buckets;
  p.n = static_cast<uint32_t>(cfg.n);
  p.k = cfg.k;
  p.mode = cfg.mode == CountMode::kAll ? IG_MODE_ALL : IG_MODE_ONCE;
  p.seed = cfg.seed;
  p.flush_batch_size = cfg.flush_batch_size;
  p.trie_second_pass = cfg.trie_second_pass ? 1 : 0;
  p.device = cfg.device;
  ig_result r{};
  char err[1024] = {0};
  detail::raise(ig_hashgram_topk(&c, &p, &r, err, sizeof(err)), err);
  IntergramsResult out = detail::convert(r);
  ig_result_free(&r);
  return HashgramResult{std::move(out.topk), std::move(out.passes)};
}

}  // namespace intergrams
