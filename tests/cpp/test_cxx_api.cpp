// C++ drop-in API test: the reference's own call shapes (run_intergrams on a
// Corpus with an IntergramConfig) compiled against include/intergrams/ and the
// B200 library.  Mirrors proj/tests/test_intergrams.cpp and test_corpus.cpp
// cases.  Usage: test_cxx_api [--no-gpu]
#include <cstdio>
#include <optional>
#include <span>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>

#include <unistd.h>

#include "intergrams/dense_pass.hpp"
#include "intergrams/intergrams.hpp"
#include "intergrams/metrics.hpp"
#include "intergrams/trie.hpp"

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
  // any n passes validation (the reference has no upper bound)
  CHECK(!throws<ConfigError>([] { config(40, 1, 1.5, CountMode::kAll).validate(); }));
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

  {  // host containers and the prefix set (test_counting.cpp, test_trie.cpp)
    SeenBitset b(130);
    b.mark(0);
    b.mark(129);
    b.mark(129);
    CHECK(b.popcount() == 2 && b.test(129) && !b.test(64));
    CountTable table(130);
    SeenBitset* batch[] = {&b};
    flush_batch(std::span<SeenBitset* const>(batch, 1), table);
    CHECK(table[0] == 1 && table[129] == 1 && table.total() == 2 && b.popcount() == 0);
    CountTable tt(3);
    tt.increment_all(0, 3);
    tt.increment_all(1, 3);
    tt.increment_all(2, 1);
    const auto top = top_k(tt, 2, [](size_t id) { return std::string(1, char('a' + id)); });
    CHECK(top.size() == 2 && top[0] == (GramCount{"a", 3}) && top[1] == (GramCount{"b", 3}));
    const TopKList pre{{std::string("\x00\x00\x00", 3), 9}, {std::string("\x00\x00\x01", 3), 8},
                       {std::string("\x00\x0f\x11", 3), 7}, {std::string("\xff\x00\xfe", 3), 6}};
    const PrefixTrie trie = PrefixTrie::build(pre);
    CHECK(trie.depth() == 3 && trie.size() == 4);
    for (size_t r = 0; r < pre.size(); ++r) CHECK(trie.lookup(pre[r].gram) == std::optional<uint32_t>(r));
    CHECK(!trie.contains(std::string("\x00\x0a\xaf", 3)));
    CHECK(throws<std::invalid_argument>([] { PrefixTrie::build({{"ab", 1}, {"abc", 1}}); }));
    CHECK(throws<std::invalid_argument>([] { PrefixTrie::build({{"ab", 2}, {"ab", 1}}); }));
    CHECK(throws<std::invalid_argument>([&] { (void)trie.lookup("ab"); }));
    CHECK(!PrefixTrie().contains("abc") && PrefixTrie().depth() == 0);
    CHECK(dense_capacity(2) == 65536 && dense_gram(0x616263, 3) == "abc");
    CHECK(throws<ConfigError>([] { dense_capacity(4); }));
  }

  if (gpu) {
    // pass-level API on the GPU (test_dense_pass.cpp:50-62, 88-118; test_intergrams.cpp:48-67)
    CountingOptions once;
    CountingOptions all;
    all.mode = CountMode::kAll;
    CountTable t1 = count_trigrams(make_memory_corpus({"aaaa"}), once);
    CHECK(t1[0x616161] == 1 && t1.total() == 1);
    t1 = count_trigrams(make_memory_corpus({"aaaa"}), all);
    CHECK(t1[0x616161] == 2 && t1.total() == 2);
    const CountTable t2 = count_trigrams(make_memory_corpus({"aaaa", "aaab"}), once);
    const TopKList tk = topk_trigrams(t2, 2);
    CHECK(tk.size() == 2 && tk[0] == (GramCount{"aaa", 2}) && tk[1] == (GramCount{"aab", 1}));
    CHECK(topk_trigrams(t2, 10).size() == 2);
    const TopKList five = topk_trigrams(count_trigrams(make_memory_corpus({"abcxbcd"}), once), 5);
    CHECK(five.size() == 5);
    for (size_t i = 1; i < five.size(); ++i) CHECK(five[i - 1].gram < five[i].gram);
    uint64_t bp = 0;
    const CountTable ext =
        extend_pass(make_memory_corpus({"abab"}), PrefixTrie::build({{"aba", 1}}), 4, once, &bp);
    CHECK(ext.capacity() == 256 && ext[candidate_id(0, 'b')] == 1 && ext.total() == 1 && bp == 4);
    CHECK(throws<ConfigError>([&] {
      extend_pass(make_memory_corpus({"abcd"}), PrefixTrie::build({{"ab", 1}}), 4, once);
    }));
    CHECK(candidate_gram({{"aba", 1}}, candidate_id(0, 'b')) == "abab");
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
