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
// No reference source is copied into this repository.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "intergrams/dense_pass.hpp"
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

// Runs ig_ref::run_intergrams. grams: k*n bytes (gram i at i*n). seconds:
// wall time of run_intergrams alone (corpus materialisation excluded).
int igref_run_intergrams(const uint8_t* data, const uint64_t* off, uint64_t m,
                         uint32_t n, uint64_t k, double z, int mode,
                         uint32_t workers, uint8_t* grams, uint64_t* counts,
                         uint64_t* out_len, igref_pass* passes,
                         uint32_t max_passes, uint32_t* num_passes, char* diag,
                         size_t diag_len, double* seconds, char* err,
                         size_t err_len) {
  return guarded(err, err_len, [&] {
    const Corpus corpus = make_corpus(data, off, m);
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
  });
}

// ig_ref::count_dense into table (256^n u64).
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

}  // extern "C"
