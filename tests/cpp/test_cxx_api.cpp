// C++ drop-in API test: the reference's own call shapes (run_intergrams on a
// Corpus with an IntergramConfig) compiled against include/intergrams/ and the
// B200 library.  Mirrors proj/tests/test_intergrams.cpp and test_corpus.cpp
// cases.  Usage: test_cxx_api [--no-gpu]
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>

#include <unistd.h>

#include "intergrams/intergrams.hpp"
#include "intergrams/metrics.hpp"

using namespace intergrams;

static int failures = 0;
#define CHECK(x)                                                        \
  do {                                                                  \
    if (!(x)) {                                                         \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static IntergramConfig config(size_t n, size_t k, double z, CountMode mode) {
  IntergramConfig cfg;
  cfg.n = n;
  cfg.k = k;
  cfg.z = z;
  cfg.mode = mode;
  return cfg;
}

int main(int argc, char** argv) {
  const bool gpu = !(argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0);
  // invalid configs (test_intergrams.cpp:239-243) fail before any device work
  CHECK(throws<ConfigError>([] { config(0, 1, 1.0, CountMode::kOnce).validate(); }));
  CHECK(throws<ConfigError>([] { config(4, 0, 1.0, CountMode::kOnce).validate(); }));
  CHECK(throws<ConfigError>([] { config(4, 1, 0.5, CountMode::kOnce).validate(); }));
  CHECK(throws<ConfigError>([] {
    run_intergrams(make_memory_corpus({"abcd"}), config(9, 1, 1.5, CountMode::kAll));
  }));
  CHECK(topk_from_tsv("616161\t2\n616162\t1\n") ==
        (TopKList{GramCount{"aaa", 2}, GramCount{"aab", 1}}));
  CHECK(throws<ConfigError>([] { from_hex("6"); }));

  // file enumeration: sorted paths, chunk and line records (corpus.cpp:40-135)
  namespace fs = std::filesystem;
  const fs::path dir = fs::temp_directory_path() / ("ig_cxx_" + std::to_string(::getpid()));
  fs::create_directories(dir);
  { std::ofstream(dir / "b.txt", std::ios::binary) << "abab\nabba\n\nxyz"; }
  { std::ofstream(dir / "a.bin", std::ios::binary) << "0123456789"; }
  CorpusSpec spec;
  spec.roots = {dir};
  spec.chunk_size = 4;
  std::vector<std::string> chunks;
  Corpus(spec).for_each([&](const Sequence& s) { chunks.push_back(s.bytes); });
  CHECK((chunks == std::vector<std::string>{"0123", "4567", "89", "abab", "\nabb", "a\n\nx", "yz"}));
  spec.chunk_size = 0;
  spec.line_mode = true;
  std::vector<std::string> lines;
  Corpus(spec).for_each([&](const Sequence& s) { lines.push_back(s.bytes); });
  CHECK((lines == std::vector<std::string>{"0123456789", "abab", "abba", "", "xyz"}));
  CHECK(throws<ConfigError>([] {
    CorpusSpec bad;
    bad.roots = {"/nonexistent/path/for/test"};
    Corpus c(bad);
  }));

  if (gpu) {
    // four-way tie resolves canonically (test_intergrams.cpp:119-125)
    auto r = run_intergrams(make_memory_corpus({"abab", "abba"}), config(4, 1, 100.0, CountMode::kOnce));
    CHECK(r.topk.size() == 1 && r.topk[0] == (GramCount{"abab", 1}));
    // SPEC.md:693 golden TSV
    r = run_intergrams(make_memory_corpus({"aaaa", "aaab"}), config(3, 2, 1.0, CountMode::kOnce));
    CHECK(topk_to_tsv(r.topk) == "616161\t2\n616162\t1\n");
    // diagnostics on degenerate corpora (test_intergrams.cpp:210-217)
    r = run_intergrams(make_memory_corpus({"aaaa", "aaab"}), config(4, 5, 10.0, CountMode::kOnce));
    CHECK(!r.diagnostics.empty() && r.topk.size() == 2);
    // empty survivor list before an extension pass -> ConfigError (probe P5)
    CHECK(throws<ConfigError>([] {
      run_intergrams(make_memory_corpus({"ab"}), config(4, 3, 1.5, CountMode::kAll));
    }));
    // a file corpus in line mode equals the same lines in memory
    auto rf = run_intergrams(Corpus(spec), config(4, 5, 2.0, CountMode::kAll));
    auto rm = run_intergrams(make_memory_corpus(lines), config(4, 5, 2.0, CountMode::kAll));
    CHECK(rf.topk == rm.topk && !rf.topk.empty());
    // per-pass rows (test_intergrams.cpp:219-237)
    r = run_intergrams(make_memory_corpus({"the cat sat on the mat", "the cat ate"}),
                       config(6, 4, 2.0, CountMode::kOnce));
    size_t counting = 0;
    for (const auto& p : r.passes) counting += p.bytes_processed > 0;
    CHECK(counting == 4 && r.passes.size() == 8);
  }
  fs::remove_all(dir);
  std::printf("%s: %d failures\n", gpu ? "gpu" : "no-gpu", failures);
  return failures ? 1 : 0;
}
