// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference sources, compiled straight from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libigref.so with
// -Dintergrams=ig_ref (the reference namespace renamed so it can never be
// confused with, or linked into, the product library).  It exposes exactly
// the reference calls the parity tests and the CPU baseline need:
//   run_intergrams   proj/src/intergrams.cpp:68-166
//   count_dense      proj/src/dense_pass.cpp:21-39
//   extend_pass      proj/src/intergrams.cpp:44-66
//   naive_count/topk proj/src/oracle.cpp:7-47
//   run_hashgram     proj/src/hashgram.cpp:325-383 (and mix64 :22-59)
//   featurize        proj/src/metrics.cpp:83-132
//   jaccard          proj/src/metrics.cpp:16-31
//   RunReport        proj/src/metrics.cpp:134-200 (to_tsv / to_json)
//   Corpus(spec)     proj/src/corpus.cpp:13-152 (file enumeration + records)
// No reference source is copied into this repository.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "intergrams/dense_pass.hpp"
#include "intergrams/hashgram.hpp"
#include "intergrams/metrics.hpp"
#include "intergrams/intergrams.hpp"
#include "intergrams/oracle.hpp"

namespace {

using namespace ig_ref;

Corpus make_corpus(const uint8_t* data, const uint64_t* off, uint64_t m) {
  std::vector<std::string> seqs;
  seqs.reserve(m);
  for (uint64_t i = 0; i < m; ++i) {
    seqs.emplace_back(reinterpret_cast<const char*>(data + off[i]),
                      off[i + 1] - off[i]);
  }
  return make_memory_corpus(std::move(seqs));
}

void put_err(char* err, size_t len, const char* msg) {
  if (err && len) {
    std::strncpy(err, msg, len - 1);
    err[len - 1] = 0;
  }
}

// 0 ok, 2 ConfigError, 3 IoError, 5 invalid_argument/logic_error, 4 other.
template <typename F>
int guarded(char* err, size_t len, F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    put_err(err, len, e.what());
    return 2;
  } catch (const IoError& e) {
    put_err(err, len, e.what());
    return 3;
  } catch (const std::logic_error& e) {
    put_err(err, len, e.what());
    return 5;
  } catch (const std::exception& e) {
    put_err(err, len, e.what());
    return 4;
  }
}

CountMode to_mode(int mode) { return mode == 1 ? CountMode::kAll : CountMode::kOnce; }

}  // namespace

extern "C" {

typedef struct {
  char label[48];
  uint32_t gram_len;
  double seconds;
  uint64_t bytes_processed;
  uint64_t candidate_space;
  uint64_t retained;
  int32_t retained_short;
} igref_pass;

unsigned igref_hardware_concurrency() {
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : hw;
}

// ig_ref::run_intergrams over an already-built corpus: grams k*n bytes (gram
// i at i*n); seconds = wall time of run_intergrams alone.
static void run_on(const Corpus& corpus, uint32_t n, uint64_t k, double z, int mode,
                   uint32_t workers, uint8_t* grams, uint64_t* counts, uint64_t* out_len,
                   igref_pass* passes, uint32_t max_passes, uint32_t* num_passes, char* diag,
                   size_t diag_len, double* seconds) {
  IntergramConfig cfg;
  cfg.n = n;
  cfg.k = k;
  cfg.z = z;
  cfg.mode = to_mode(mode);
  cfg.workers = workers ? workers : igref_hardware_concurrency();
  const auto t0 = std::chrono::steady_clock::now();
  const IntergramsResult r = run_intergrams(corpus, cfg);
  const auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  *out_len = r.topk.size();
  for (size_t i = 0; i < r.topk.size(); ++i) {
    std::memcpy(grams + i * n, r.topk[i].gram.data(), n);
    counts[i] = r.topk[i].count;
  }
  uint32_t np = 0;
  for (const auto& p : r.passes) {
    if (np >= max_passes) break;
    igref_pass& o = passes[np++];
    std::memset(&o, 0, sizeof(o));
    std::strncpy(o.label, p.label.c_str(), sizeof(o.label) - 1);
    o.gram_len = static_cast<uint32_t>(p.gram_len);
    o.seconds = p.seconds;
    o.bytes_processed = p.bytes_processed;
    o.candidate_space = p.candidate_space;
    o.retained = p.retained;
    o.retained_short = p.retained_short;
  }
  *num_passes = np;
  std::string d;
  for (const auto& s : r.diagnostics) d += s + "\n";
  if (diag && diag_len) put_err(diag, diag_len, d.c_str());
}

// Runs ig_ref::run_intergrams on an in-memory corpus (CSR data/off; the
// corpus materialisation is excluded from *seconds).
int igref_run_intergrams(const uint8_t* data, const uint64_t* off, uint64_t m,
                         uint32_t n, uint64_t k, double z, int mode,
                         uint32_t workers, uint8_t* grams, uint64_t* counts,
                         uint64_t* out_len, igref_pass* passes,
                         uint32_t max_passes, uint32_t* num_passes, char* diag,
                         size_t diag_len, double* seconds, char* err,
                         size_t err_len) {
  return guarded(err, err_len, [&] {
    const Corpus corpus = make_corpus(data, off, m);
    run_on(corpus, n, k, z, mode, workers, grams, counts, out_len, passes, max_passes,
           num_passes, diag, diag_len, seconds);
  });
}

// The same over a file corpus (CorpusSpec: one root, whole-file records or
// fixed chunk_size records, corpus.cpp:55-119): equal-length configs read as
// one flat file with chunk_size = the sequence length reproduce the
// sequence boundaries exactly without a second in-memory copy.
int igref_run_intergrams_file(const char* root, uint64_t chunk_size, uint32_t n, uint64_t k,
                              double z, int mode, uint32_t workers, uint8_t* grams,
                              uint64_t* counts, uint64_t* out_len, igref_pass* passes,
                              uint32_t max_passes, uint32_t* num_passes, char* diag,
                              size_t diag_len, double* seconds, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    CorpusSpec spec;
    spec.roots.emplace_back(root);
    spec.chunk_size = chunk_size;
    const Corpus corpus(std::move(spec));
    run_on(corpus, n, k, z, mode, workers, grams, counts, out_len, passes, max_passes,
           num_passes, diag, diag_len, seconds);
  });
}

int igref_count_dense(const uint8_t* data, const uint64_t* off, uint64_t m,
                      uint32_t n, int mode, uint32_t workers, uint64_t* table,
                      char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const Corpus corpus = make_corpus(data, off, m);
    CountingOptions opt;
    opt.mode = to_mode(mode);
    opt.workers = workers ? workers : 1;
    const CountTable t = count_dense(corpus, n, opt);
    std::memcpy(table, t.raw().data(), t.capacity() * sizeof(uint64_t));
  });
}

// ig_ref::extend_pass over a trie built from prefixes (nprefix grams of plen
// bytes, rank order).  table: 256*nprefix u64.
int igref_extend_pass(const uint8_t* data, const uint64_t* off, uint64_t m,
                      const uint8_t* prefixes, uint64_t nprefix, uint32_t plen,
                      uint32_t j, int mode, uint64_t* table,
                      uint64_t* bytes_processed, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const Corpus corpus = make_corpus(data, off, m);
    TopKList list;
    for (uint64_t i = 0; i < nprefix; ++i) {
      list.push_back(GramCount{
          std::string(reinterpret_cast<const char*>(prefixes + i * plen), plen),
          nprefix - i});
    }
    const PrefixTrie trie = PrefixTrie::build(list);
    CountingOptions opt;
    opt.mode = to_mode(mode);
    uint64_t bytes = 0;
    const CountTable t = extend_pass(corpus, trie, j, opt, &bytes);
    std::memcpy(table, t.raw().data(), t.capacity() * sizeof(uint64_t));
    if (bytes_processed) *bytes_processed = bytes;
  });
}

// ig_ref::naive_topk(naive_count(...)).  grams: k*n bytes.
int igref_naive_topk(const uint8_t* data, const uint64_t* off, uint64_t m,
                     uint32_t n, int mode, uint64_t k, uint8_t* grams,
                     uint64_t* counts, uint64_t* out_len, char* err,
                     size_t err_len) {
  return guarded(err, err_len, [&] {
    const Corpus corpus = make_corpus(data, off, m);
    const TopKList top = naive_topk(naive_count(corpus, n, to_mode(mode), ~0ull), k);
    *out_len = top.size();
    for (size_t i = 0; i < top.size(); ++i) {
      std::memcpy(grams + i * n, top[i].gram.data(), n);
      counts[i] = top[i].count;
    }
  });
}

uint64_t igref_mix64(const uint8_t* bytes, uint64_t len, uint64_t seed) {
  return mix64(std::string_view(reinterpret_cast<const char*>(bytes), len), seed);
}

// ig_ref::run_hashgram.  grams: k*n bytes.
int igref_hashgram(const uint8_t* data, const uint64_t* off, uint64_t m,
                   uint32_t n, uint64_t k, int mode, uint64_t buckets,
                   uint64_t seed, uint32_t workers, int trie, uint8_t* grams,
                   uint64_t* counts, uint64_t* out_len, igref_pass* passes,
                   uint32_t max_passes, uint32_t* num_passes, char* err,
                   size_t err_len) {
  return guarded(err, err_len, [&] {
    const Corpus corpus = make_corpus(data, off, m);
    HashgramConfig cfg;
    cfg.buckets = buckets;
    cfg.n = n;
    cfg.k = k;
    cfg.mode = to_mode(mode);
    cfg.seed = seed;
    cfg.workers = workers ? workers : 1;
    cfg.trie_second_pass = trie != 0;
    const HashgramResult r = run_hashgram(corpus, cfg);
    *out_len = r.topk.size();
    for (size_t i = 0; i < r.topk.size(); ++i) {
      std::memcpy(grams + i * n, r.topk[i].gram.data(), n);
      counts[i] = r.topk[i].count;
    }
    uint32_t np = 0;
    for (const auto& p : r.passes) {
      if (np >= max_passes) break;
      igref_pass& o = passes[np++];
      std::memset(&o, 0, sizeof(o));
      std::strncpy(o.label, p.label.c_str(), sizeof(o.label) - 1);
      o.gram_len = static_cast<uint32_t>(p.gram_len);
      o.seconds = p.seconds;
      o.bytes_processed = p.bytes_processed;
      o.candidate_space = p.candidate_space;
      o.retained = p.retained;
      o.retained_short = p.retained_short;
    }
    *num_passes = np;
  });
}

// ig_ref::featurize.  vocab: ncols grams of n bytes.  entries: (row << 32) |
// col, capacity cap; *nnz the number written; *rows the matrix rows.
int igref_featurize(const uint8_t* data, const uint64_t* off, uint64_t m,
                    const uint8_t* vocab, uint64_t ncols, uint32_t n,
                    uint32_t workers, uint64_t* entries, uint64_t cap,
                    uint64_t* nnz, uint64_t* rows, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const Corpus corpus = make_corpus(data, off, m);
    TopKList v;
    for (uint64_t j = 0; j < ncols; ++j)
      v.push_back(GramCount{std::string(reinterpret_cast<const char*>(vocab + j * n), n), 1});
    const FeatureMatrix mat = featurize(corpus, v, workers ? workers : 1);
    if (mat.entries.size() > cap) throw std::runtime_error("entries capacity too small");
    for (size_t i = 0; i < mat.entries.size(); ++i)
      entries[i] = (mat.entries[i].first << 32) | mat.entries[i].second;
    *nnz = mat.entries.size();
    *rows = mat.rows;
  });
}

// ig_ref::Corpus over files: enumerates roots (recurse / line / chunk) and
// materialises the records.  data may be NULL (sizes only).  Returns the file
// count in *num_files.
int igref_corpus_files(const char* const* roots, uint64_t nroots, int recurse, int line_mode,
                       uint64_t chunk_size, uint8_t* data, uint64_t cap, uint64_t* offsets,
                       uint64_t offcap, uint64_t* num_seqs, uint64_t* total, uint64_t* num_files,
                       char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    CorpusSpec spec;
    for (uint64_t i = 0; i < nroots; ++i) spec.roots.emplace_back(roots[i]);
    spec.recurse = recurse != 0;
    spec.line_mode = line_mode != 0;
    spec.chunk_size = chunk_size;
    const Corpus corpus(std::move(spec));
    uint64_t m = 0, t = 0;
    if (offsets && offcap) offsets[0] = 0;
    corpus.for_each([&](const Sequence& s) {
      if (data && t + s.bytes.size() <= cap) std::memcpy(data + t, s.bytes.data(), s.bytes.size());
      t += s.bytes.size();
      ++m;
      if (offsets && m < offcap) offsets[m] = t;
    });
    *num_seqs = m;
    *total = t;
    *num_files = corpus.files().size();
  });
}

// ig_ref::jaccard of two result TSV texts.
double igref_jaccard_tsv(const char* a, const char* b) {
  return jaccard(topk_from_tsv(a), topk_from_tsv(b));
}

// RunReport::to_tsv / to_json (json != 0) of the given rows into out.
int igref_report(const char* algorithm, const char* echo, const igref_pass* passes,
                 uint32_t np, int has_jaccard, double jacc, int json, char* out,
                 size_t out_len) {
  return guarded(out, out_len, [&] {
    std::vector<PassResult> rows;
    for (uint32_t i = 0; i < np; ++i) {
      PassResult r;
      r.label = passes[i].label;
      r.gram_len = passes[i].gram_len;
      r.seconds = passes[i].seconds;
      r.bytes_processed = passes[i].bytes_processed;
      r.candidate_space = passes[i].candidate_space;
      r.retained = passes[i].retained;
      r.retained_short = passes[i].retained_short != 0;
      rows.push_back(r);
    }
    RunReport rep = make_report(algorithm, echo, rows);
    if (has_jaccard) rep.jaccard_vs_reference = jacc;
    const std::string s = json ? rep.to_json() : rep.to_tsv();
    if (s.size() + 1 > out_len) throw std::runtime_error("report buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

}  // extern "C"
