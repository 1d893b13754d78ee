// intergrams/intergrams.hpp — drop-in for
// /root/reference/proj/include/intergrams/intergrams.hpp: the same
// IntergramConfig (:19-33), PassResult (:35-47), IntergramsResult (:49-53),
// candidate_id (:56-59) and run_intergrams (:74-75), executed by the sm_100a
// library through the C-ABI in include/intergrams_b200.h.  Header-only; link
// with paper_2511_14955_b200/_lib/libintergrams_b200.so.
#pragma once

#include <cassert>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "intergrams/common.hpp"
#include "intergrams/corpus.hpp"
#include "intergrams/counting.hpp"
#include "intergrams/pipeline.hpp"
#include "intergrams/trie.hpp"
#include "intergrams_b200.h"

namespace intergrams {

struct IntergramConfig {
  size_t n = 6;
  size_t k = 10000;
  double z = 1.5;  // k' = ceil(z*k)
  CountMode mode = CountMode::kOnce;
  MergeStrategy merge = MergeStrategy::kBatchedFlush;  // no effect on the GPU
  size_t workers = 1;                                   // no effect on the GPU
  size_t flush_batch_size = 8;                          // validated only
  bool frequency_ordered_trie = true;                   // no effect on results
  int device = -1;                                      // CUDA ordinal (-1: current)
  // Several GPUs of this process (the reference's data parallelism,
  // pipeline.hpp:101-199, on GPUs): whole-sequence shards balanced by bytes,
  // one NCCL all-reduce per pass (ig_topk_ngrams_multi).  Empty: `device`
  // alone, unless IG_DEVICES="0,1,..." names them (for unmodified callers).
  std::vector<int> devices;

  std::vector<int> device_list() const {
    if (!devices.empty()) return devices;
    std::vector<int> v;
    if (const char* e = std::getenv("IG_DEVICES")) {
      for (const char* p = e; *p;) {
        char* end = nullptr;
        const long d = std::strtol(p, &end, 10);
        if (end == p) break;
        v.push_back(static_cast<int>(d));
        p = *end ? end + 1 : end;
      }
    }
    return v;
  }

  size_t k_prime() const { return static_cast<size_t>(std::ceil(z * static_cast<double>(k))); }
  void validate() const {
    if (n < 1) throw ConfigError("gram length n must be >= 1");
    if (k < 1) throw ConfigError("k must be >= 1");
    if (!(z >= 1.0)) throw ConfigError("oversample factor z must be >= 1");
    if (flush_batch_size < 1) throw ConfigError("flush batch size must be >= 1");
  }
};

struct PassResult {
  std::string label;
  size_t gram_len = 0;
  double seconds = 0.0;
  uint64_t bytes_processed = 0;
  size_t candidate_space = 0;
  size_t retained = 0;
  bool retained_short = false;

  double throughput_bps() const {
    return seconds > 0.0 ? static_cast<double>(bytes_processed) / seconds : 0.0;
  }
};

struct IntergramsResult {
  TopKList topk;
  std::vector<PassResult> passes;
  std::vector<std::string> diagnostics;
};

inline size_t candidate_id(size_t prefix_ordinal, unsigned last_byte) {
  assert(last_byte <= 255);
  return prefix_ordinal * 256 + last_byte;
}

// Gram bytes of an extension-pass candidate id (intergrams.hpp:61-66).
inline std::string candidate_gram(const TopKList& prefixes, size_t id) {
  std::string gram = prefixes[id >> 8].gram;
  gram.push_back(static_cast<char>(id & 0xff));
  return gram;
}

namespace detail {

inline void raise(int rc, const char* err) {
  switch (rc) {
    case IG_OK: return;
    case IG_ECONFIG: throw ConfigError(err);
    case IG_EIO: throw IoError(err);
    case IG_EINVALID: throw std::invalid_argument(err);
    default: throw DeviceError(err);
  }
}

inline IntergramsResult convert(const ig_result& r) {
  IntergramsResult out;
  out.topk.reserve(r.len);
  for (uint64_t i = 0; i < r.len; ++i) {
    std::string g(r.gram_len, '\0');
    if (r.grams) {  // every n (the only form for n > 8)
      for (uint32_t b = 0; b < r.gram_len; ++b)
        g[b] = static_cast<char>(r.grams[i * r.gram_len + b]);
    } else {
      for (uint32_t b = 0; b < r.gram_len; ++b)
        g[b] = static_cast<char>((r.keys[i] >> (8 * (r.gram_len - 1 - b))) & 0xff);
    }
    out.topk.push_back(GramCount{std::move(g), r.counts[i]});
  }
  for (uint32_t i = 0; i < r.num_passes; ++i) {
    const ig_pass_stat& p = r.passes[i];
    out.passes.push_back(PassResult{p.label, p.gram_len, p.seconds, p.bytes_processed,
                                    p.candidate_space, p.retained, p.retained_short != 0});
  }
  std::string d = r.diagnostics ? r.diagnostics : "";
  size_t s = 0;
  while (s < d.size()) {
    size_t e = d.find('\n', s);
    if (e == std::string::npos) e = d.size();
    if (e > s) out.diagnostics.push_back(d.substr(s, e - s));
    s = e + 1;
  }
  return out;
}

inline ig_params params_of(const IntergramConfig& cfg) {
  ig_params p{};
  p.n = static_cast<uint32_t>(cfg.n);
  p.k = cfg.k;
  p.z = cfg.z;
  p.mode = cfg.mode == CountMode::kAll ? IG_MODE_ALL : IG_MODE_ONCE;
  p.flush_batch_size = cfg.flush_batch_size;
  p.device = cfg.device;
  return p;
}

}  // namespace detail

// run_intergrams (intergrams.hpp:74-75) on the GPU.  A file corpus is read by
// the library itself (host threads -> pinned slabs -> HBM, line splitting on
// the GPU); an in-memory corpus is gathered sequence by sequence the same way.
inline IntergramsResult run_intergrams(const Corpus& corpus, const IntergramConfig& cfg) {
  cfg.validate();
  ig_params p = detail::params_of(cfg);
  ig_result r{};
  char err[1024] = {0};
  const std::vector<int> devs = cfg.device_list();
  if (devs.size() == 1) p.device = devs[0];
  if (devs.size() > 1) {  // sharded over several GPUs: one contiguous host corpus
    const CorpusCSR csr = corpus.materialize();
    ig_corpus c{csr.data.data(), csr.offsets.data(), csr.offsets.size() - 1, IG_HOST};
    std::vector<int32_t> d(devs.begin(), devs.end());
    detail::raise(ig_topk_ngrams_multi(&c, d.data(), static_cast<int32_t>(d.size()), &p, &r, err,
                                       sizeof(err)),
                  err);
    IntergramsResult out = detail::convert(r);
    ig_result_free(&r);
    return out;
  }
  if (!corpus.spec().in_memory.has_value()) {
    std::vector<std::string> roots;
    for (const auto& root : corpus.spec().roots) roots.push_back(root.string());
    std::vector<const char*> ptrs;
    for (const auto& root : roots) ptrs.push_back(root.c_str());
    ig_file_corpus spec{ptrs.data(), ptrs.size(), corpus.spec().recurse ? 1 : 0,
                        corpus.spec().line_mode ? 1 : 0, corpus.spec().chunk_size};
    detail::raise(ig_topk_ngrams_files(&spec, &p, &r, err, sizeof(err)), err);
    IntergramsResult out = detail::convert(r);
    ig_result_free(&r);
    return out;
  }
  // in-memory: the sequences are gathered in place (no packed copy) by the
  // library's host threads into pinned slabs that stream under the dense pass
  const std::vector<std::string>& seqs = *corpus.spec().in_memory;
  std::vector<const uint8_t*> ptrs(seqs.size());
  std::vector<uint64_t> lens(seqs.size());
  for (size_t q = 0; q < seqs.size(); ++q) {
    ptrs[q] = reinterpret_cast<const uint8_t*>(seqs[q].data());
    lens[q] = seqs[q].size();
  }
  detail::raise(ig_topk_ngrams_seqs(ptrs.data(), lens.data(), seqs.size(), &p, &r, err,
                                    sizeof(err)),
                err);
  IntergramsResult out = detail::convert(r);
  ig_result_free(&r);
  return out;
}

// extend_pass (intergrams.hpp:68-72, src/intergrams.cpp:44-66) on the GPU:
// counts the j-grams whose (j-1)-prefix is in the trie into 256 * trie.size()
// candidate ids; trie.depth() must equal j-1 (ConfigError otherwise).
inline CountTable extend_pass(const Corpus& corpus, const PrefixTrie& trie, size_t j,
                              const CountingOptions& opt, uint64_t* bytes_processed = nullptr,
                              int device = -1) {
  std::vector<uint64_t> keys;
  keys.reserve(trie.size());
  for (const auto& g : trie.grams()) {
    if (g.size() > IG_MAX_N) throw ConfigError("gram length above 8 is not supported");
    uint64_t k = 0;
    for (unsigned char b : g) k = (k << 8) | b;
    keys.push_back(k);
  }
  CountTable table(256 * trie.size());
  const CorpusCSR csr = corpus.materialize();
  ig_corpus c{csr.data.data(), csr.offsets.data(), csr.offsets.size() - 1, IG_HOST};
  uint64_t bytes = 0;
  char err[1024] = {0};
  detail::raise(ig_extend_pass(&c, keys.empty() ? nullptr : keys.data(), keys.size(),
                               static_cast<uint32_t>(trie.depth()), static_cast<uint32_t>(j),
                               opt.mode == CountMode::kAll ? IG_MODE_ALL : IG_MODE_ONCE, device,
                               table.data(), &bytes, err, sizeof(err)),
                err);
  if (bytes_processed) *bytes_processed = bytes;
  return table;
}

}  // namespace intergrams
