// intergrams/metrics.hpp — drop-in for /root/reference/proj/include/intergrams/metrics.hpp
// (src/metrics.cpp): the bit-exact result TSV (:202-232), jaccard (:16-31),
// prefix_recall (:33-81), featurize (:83-132, on the GPU via ig_featurize) and
// the Table-4-style RunReport (:134-200; to_json renders the reference's
// nlohmann dump(2) layout without the dependency).  Header-only.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <optional>
#include <string>
#include <string_view>
#include <unordered_set>
#include <utility>
#include <vector>

#include "intergrams/common.hpp"
#include "intergrams/corpus.hpp"
#include "intergrams/counting.hpp"
#include "intergrams/intergrams.hpp"
#include "intergrams/oracle.hpp"
#include "intergrams_b200.h"

namespace intergrams {

inline std::string topk_to_tsv(const TopKList& list) {
  std::string out;
  for (const auto& gc : list) {
    out += to_hex(gc.gram);
    out += '\t';
    out += std::to_string(gc.count);
    out += '\n';
  }
  return out;
}

inline TopKList topk_from_tsv(const std::string& text) {
  TopKList list;
  size_t start = 0;
  while (start < text.size()) {
    size_t end = text.find('\n', start);
    if (end == std::string::npos) end = text.size();
    const std::string line = text.substr(start, end - start);
    start = end + 1;
    if (line.empty()) continue;
    const size_t tab = line.find('\t');
    if (tab == std::string::npos) throw ConfigError("malformed result line (no tab): " + line);
    list.push_back(GramCount{from_hex(line.substr(0, tab)), std::stoull(line.substr(tab + 1))});
  }
  return list;
}

// |A ∩ B| / |A ∪ B| over the gram sets; 1.0 when both are empty.
inline double jaccard(const TopKList& a, const TopKList& b) {
  std::unordered_set<std::string_view> sa, sb;
  for (const auto& gc : a) sa.insert(gc.gram);
  for (const auto& gc : b) sb.insert(gc.gram);
  size_t inter = 0;
  for (const auto& g : sa) inter += sb.count(g);
  const size_t uni = sa.size() + sb.size() - inter;
  return uni == 0 ? 1.0 : static_cast<double>(inter) / static_cast<double>(uni);
}

// Fraction of the exact top-k (n_small+1)-grams whose n_small-byte prefix is
// among the exact top-ceil(z*k) n_small-grams, per z (metrics.cpp:33-70).
inline std::vector<double> prefix_recall_curve(const Corpus& corpus, size_t k,
                                               const std::vector<double>& zs, size_t n_small,
                                               CountMode mode,
                                               uint64_t oracle_guard = kOracleCorpusGuard) {
  if (k < 1) throw ConfigError("prefix_recall requires k >= 1");
  for (double z : zs)
    if (!(z >= 1.0)) throw ConfigError("prefix_recall requires z >= 1");
  const GramCountMap small_counts = naive_count(corpus, n_small, mode, oracle_guard);
  const TopKList top_big = naive_topk(corpus, n_small + 1, mode, k, oracle_guard);
  std::vector<double> out;
  for (double z : zs) {
    const size_t keep = static_cast<size_t>(std::ceil(z * static_cast<double>(k)));
    const TopKList top_small = naive_topk(small_counts, keep);
    std::unordered_set<std::string_view> prefixes;
    for (const auto& gc : top_small) prefixes.insert(gc.gram);
    if (top_big.empty()) {
      out.push_back(1.0);
      continue;
    }
    size_t hit = 0;
    for (const auto& gc : top_big) hit += prefixes.count(std::string_view(gc.gram.data(), n_small));
    out.push_back(static_cast<double>(hit) / static_cast<double>(top_big.size()));
  }
  return out;
}

inline double prefix_recall(const Corpus& corpus, size_t k, double z, size_t n_small,
                            CountMode mode, uint64_t oracle_guard = kOracleCorpusGuard) {
  return prefix_recall_curve(corpus, k, {z}, n_small, mode, oracle_guard)[0];
}

struct FeatureMatrix {
  uint64_t rows = 0;
  uint64_t cols = 0;
  // (row, col) coordinates of set entries, sorted by row then col.
  std::vector<std::pair<uint64_t, uint32_t>> entries;

  std::vector<uint64_t> column_popcounts() const {
    std::vector<uint64_t> pops(cols, 0);
    for (const auto& [row, col] : entries) pops[col] += 1;
    return pops;
  }
};

// Boolean occurrence matrix of `vocab` over the corpus sequences, on the GPU.
// `workers` has no GPU meaning.  Vocabulary grams must share one length
// (std::invalid_argument otherwise, metrics.cpp:88-93); lengths above 8 are
// a ConfigError of the packed-u64 GPU path.
inline FeatureMatrix featurize(const Corpus& corpus, const TopKList& vocab, size_t workers = 1,
                               int device = -1) {
  (void)workers;
  const size_t n = vocab.empty() ? 0 : vocab[0].gram.size();
  for (const auto& gc : vocab)
    if (gc.gram.size() != n)
      throw std::invalid_argument("featurize: vocab grams must share one length");
  if (!vocab.empty() && n > IG_MAX_N)
    throw ConfigError("featurize: gram length above 8 is not supported by the GPU path");
  std::vector<uint64_t> keys;
  keys.reserve(vocab.size());
  for (const auto& gc : vocab) {
    uint64_t key = 0;
    for (unsigned char b : gc.gram) key = (key << 8) | b;
    keys.push_back(key);
  }
  const CorpusCSR csr = corpus.materialize();
  ig_corpus c{csr.data.data(), csr.offsets.data(), csr.offsets.size() - 1, IG_HOST};
  ig_matrix m{};
  char err[1024] = {0};
  detail::raise(ig_featurize(&c, keys.empty() ? nullptr : keys.data(), keys.size(),
                             static_cast<uint32_t>(n), device, &m, err, sizeof(err)),
                err);
  FeatureMatrix out;
  out.rows = m.rows;
  out.cols = m.cols;
  out.entries.reserve(m.nnz);
  for (uint64_t i = 0; i < m.nnz; ++i) out.entries.emplace_back(m.row[i], m.col[i]);
  ig_matrix_free(&m);
  return out;
}

namespace detail {

// Shortest round-trip decimal digits of a finite positive double:
// value = 0.d1d2...dk * 10^exp10 style is returned as (digits, n) where the
// decimal point sits after n digits (v = digits * 10^(n - k)).
inline void shortest_digits(double v, std::string& digits, int& n) {
  char buf[40];
  for (int prec = 0; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*e", prec, v);
    if (std::strtod(buf, nullptr) == v || prec == 17) break;
  }
  // buf = d[.ddd]e±XX
  digits.clear();
  const char* p = buf;
  for (; *p && *p != 'e'; ++p)
    if (*p != '.') digits.push_back(*p);
  const int e = std::atoi(p + 1);
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  n = e + 1;
}

// nlohmann::json number_float rendering (dump_float -> to_chars ->
// format_buffer with kMinExp = -4, kMaxExp = 15).
inline std::string json_double(double x) {
  if (!std::isfinite(x)) return "null";
  std::string out;
  if (std::signbit(x)) {
    out.push_back('-');
    x = -x;
  }
  if (x == 0) return out + "0.0";
  std::string d;
  int n = 0;
  shortest_digits(x, d, n);
  const int k = static_cast<int>(d.size());
  if (k <= n && n <= 15) return out + d + std::string(n - k, '0') + ".0";
  if (0 < n && n <= 15) return out + d.substr(0, n) + "." + d.substr(n);
  if (-4 < n && n <= 0) return out + "0." + std::string(-n, '0') + d;
  out += d.substr(0, 1);
  if (k > 1) out += "." + d.substr(1);
  const int e = n - 1;
  char eb[16];
  std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
  return out + eb;
}

inline std::string json_string(const std::string& s) {
  std::string out = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          out += b;
        } else {
          out.push_back(static_cast<char>(c));
        }
    }
  }
  return out + "\"";
}

}  // namespace detail

// Table-4-style report: one row per pass plus totals.
struct RunReport {
  std::string algorithm;
  std::string config_echo;
  std::vector<PassResult> passes;
  double total_seconds = 0.0;
  std::optional<double> jaccard_vs_reference;

  std::string to_tsv() const {
    std::string out = "step\truntime_s\tthroughput\n";
    char b[64];
    for (const auto& p : passes) {
      std::snprintf(b, sizeof(b), "%.4f", p.seconds);
      out += p.label + "\t" + b + "\t";
      const double bps = p.throughput_bps();
      if (bps <= 0.0) {
        out += "-";
      } else {
        std::snprintf(b, sizeof(b), "%.3f MB/s", bps / 1e6);
        out += b;
      }
      out += "\n";
    }
    std::snprintf(b, sizeof(b), "%.4f", total_seconds);
    out += std::string("total\t") + b + "\t-\n";
    if (jaccard_vs_reference.has_value()) {
      std::snprintf(b, sizeof(b), "%.6f", *jaccard_vs_reference);
      out += std::string("jaccard\t") + b + "\t-\n";
    }
    return out;
  }

  // The reference's JSON (schema_version 1): keys in sorted order, 2-space
  // indentation, nlohmann number formatting.
  std::string to_json() const {
    using detail::json_double;
    using detail::json_string;
    std::string o = "{\n";
    o += "  \"algorithm\": " + json_string(algorithm) + ",\n";
    o += "  \"config\": " + json_string(config_echo) + ",\n";
    if (jaccard_vs_reference.has_value())
      o += "  \"jaccard_vs_reference\": " + json_double(*jaccard_vs_reference) + ",\n";
    o += "  \"schema_version\": 1,\n";
    if (passes.empty()) {
      o += "  \"steps\": [],\n";
    } else {
      o += "  \"steps\": [\n";
      for (size_t i = 0; i < passes.size(); ++i) {
        const PassResult& p = passes[i];
        o += "    {\n";
        o += "      \"bytes_processed\": " + std::to_string(p.bytes_processed) + ",\n";
        o += "      \"candidate_space\": " + std::to_string(p.candidate_space) + ",\n";
        o += "      \"gram_len\": " + std::to_string(p.gram_len) + ",\n";
        o += "      \"label\": " + json_string(p.label) + ",\n";
        o += "      \"retained\": " + std::to_string(p.retained) + ",\n";
        o += std::string("      \"retained_short\": ") + (p.retained_short ? "true" : "false") +
             ",\n";
        o += "      \"seconds\": " + json_double(p.seconds) + ",\n";
        o += "      \"throughput_bps\": " + json_double(p.throughput_bps()) + "\n";
        o += i + 1 < passes.size() ? "    },\n" : "    }\n";
      }
      o += "  ],\n";
    }
    o += "  \"total_seconds\": " + json_double(total_seconds) + "\n}";
    return o;
  }
};

inline RunReport make_report(std::string algorithm, std::string config_echo,
                             std::vector<PassResult> passes) {
  RunReport r;
  r.algorithm = std::move(algorithm);
  r.config_echo = std::move(config_echo);
  r.passes = std::move(passes);
  for (const auto& p : r.passes) r.total_seconds += p.seconds;
  return r;
}

}  // namespace intergrams
