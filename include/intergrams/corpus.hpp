// intergrams/corpus.hpp — drop-in for /root/reference/proj/include/intergrams/corpus.hpp
// (corpus.hpp:23-67; enumeration semantics of src/corpus.cpp:40-152): regular
// files gathered from all roots and sorted lexicographically by path, then
// records in file order — whole file, '\n'-separated lines, or fixed-size
// chunks — or an in-memory list.  File enumeration and record walking are the
// library's (ingest.cu, over the C ABI); this header only adapts them to the
// reference's class.
//
// GPU extension: materialize() packs the enumeration into one CSR buffer
// (bytes + offsets) — the layout the C-ABI uploads to HBM.
#pragma once

#include <cstdint>
#include <exception>
#include <filesystem>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "intergrams/common.hpp"
#include "intergrams_b200.h"

namespace intergrams {

struct Sequence {
  uint64_t id = 0;
  std::string bytes;
};

struct CorpusSpec {
  std::vector<std::filesystem::path> roots;
  bool recurse = false;
  bool line_mode = false;
  uint64_t chunk_size = 0;
  std::optional<std::vector<std::string>> in_memory;
};

struct CorpusStats {
  uint64_t sequences = 0;
  uint64_t ngrams = 0;
  uint64_t bytes_total = 0;
};

// CSR view of a whole corpus: sequence i is data[offsets[i] .. offsets[i+1]).
struct CorpusCSR {
  std::vector<uint8_t> data;
  std::vector<uint64_t> offsets{0};
};

class Corpus {
 public:
  // File corpora: the library enumerates the roots (ig_file_corpus_list —
  // the reference's rules, ingest.cu) once here; records are read by the
  // library on each walk (ig_file_corpus_records).
  explicit Corpus(CorpusSpec spec) : spec_(std::move(spec)) {
    if (spec_.in_memory.has_value()) return;
    with_spec([&](const ig_file_corpus& fc) {
      struct Ctx {
        std::vector<std::filesystem::path>* out;
      } ctx{&files_};
      const ig_file_fn fn = [](const char* path, uint64_t, void* user) -> int {
        static_cast<Ctx*>(user)->out->emplace_back(path);
        return 0;
      };
      char err[512] = {0};
      rethrow(ig_file_corpus_list(&fc, fn, &ctx, err, sizeof(err)), err, nullptr);
    });
  }

  // Visits every sequence in enumeration order.
  void for_each(const std::function<void(const Sequence&)>& fn) const {
    if (spec_.in_memory.has_value()) {
      Sequence seq;
      uint64_t id = 0;
      for (const auto& bytes : *spec_.in_memory) {
        seq.id = id++;
        seq.bytes = bytes;
        fn(seq);
      }
      return;
    }
    with_spec([&](const ig_file_corpus& fc) {
      struct Ctx {
        const std::function<void(const Sequence&)>* fn;
        Sequence seq;
        std::exception_ptr ex;
      } ctx{&fn, {}, nullptr};
      const ig_record_fn rec = [](uint64_t id, const uint8_t* p, uint64_t n, void* user) -> int {
        Ctx& c = *static_cast<Ctx*>(user);
        try {
          c.seq.id = id;
          c.seq.bytes.assign(reinterpret_cast<const char*>(p), n);
          (*c.fn)(c.seq);
          return 0;
        } catch (...) {
          c.ex = std::current_exception();  // rethrown on the caller's side
          return 1;
        }
      };
      char err[512] = {0};
      const int rc = ig_file_corpus_records(&fc, rec, &ctx, err, sizeof(err));
      rethrow(rc, err, ctx.ex);
    });
  }

  CorpusStats stats(size_t n) const {
    if (n < 1) throw ConfigError("gram length must be >= 1");
    CorpusStats st;
    for_each([&](const Sequence& s) {
      ++st.sequences;
      st.bytes_total += s.bytes.size();
      if (s.bytes.size() + 1 > n) st.ngrams += s.bytes.size() - n + 1;
    });
    return st;
  }

  // One pass over the enumeration into a CSR buffer (what the GPU consumes).
  CorpusCSR materialize() const {
    CorpusCSR c;
    for_each([&](const Sequence& s) {
      c.data.insert(c.data.end(), s.bytes.begin(), s.bytes.end());
      c.offsets.push_back(c.data.size());
    });
    return c;
  }

  const std::vector<std::filesystem::path>& files() const { return files_; }
  const CorpusSpec& spec() const { return spec_; }

 private:
  // The spec as the C ABI's ig_file_corpus (roots as C strings).
  template <typename F>
  void with_spec(F&& f) const {
    std::vector<std::string> roots;
    for (const auto& r : spec_.roots) roots.push_back(r.string());
    std::vector<const char*> ptrs;
    for (const auto& r : roots) ptrs.push_back(r.c_str());
    ig_file_corpus fc{};
    fc.roots = ptrs.data();
    fc.num_roots = ptrs.size();
    fc.recurse = spec_.recurse ? 1 : 0;
    fc.line_mode = spec_.line_mode ? 1 : 0;
    fc.chunk_size = spec_.chunk_size;
    f(fc);
  }

  static void rethrow(int rc, const char* err, std::exception_ptr ex) {
    if (ex) std::rethrow_exception(ex);
    if (rc == IG_OK) return;
    if (rc == IG_ECONFIG) throw ConfigError(err);
    if (rc == IG_EIO) throw IoError(err);
    throw DeviceError(err);
  }

  CorpusSpec spec_;
  std::vector<std::filesystem::path> files_;
};

inline Corpus make_memory_corpus(std::vector<std::string> sequences) {
  CorpusSpec spec;
  spec.in_memory = std::move(sequences);
  return Corpus(std::move(spec));
}

}  // namespace intergrams
