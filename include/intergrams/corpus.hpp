// intergrams/corpus.hpp — drop-in for /root/reference/proj/include/intergrams/corpus.hpp
// (corpus.hpp:23-67; enumeration semantics of src/corpus.cpp:40-152): regular
// files gathered from all roots and sorted lexicographically by path, then
// records in file order — whole file, '\n'-separated lines, or fixed-size
// chunks — or an in-memory list.  Header-only.
//
// GPU extension: materialize() packs the enumeration into one CSR buffer
// (bytes + offsets) — the layout the C-ABI uploads to HBM.
#pragma once

#include <algorithm>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "intergrams/common.hpp"

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
  explicit Corpus(CorpusSpec spec) : spec_(std::move(spec)) {
    namespace fs = std::filesystem;
    if (spec_.in_memory.has_value()) return;
    if (spec_.roots.empty()) throw ConfigError("corpus spec has no roots and no in-memory data");
    for (const auto& root : spec_.roots) {
      std::error_code ec;
      if (fs::is_regular_file(root, ec)) {
        files_.push_back(root);
      } else if (fs::is_directory(root, ec)) {
        if (spec_.recurse) {
          for (fs::recursive_directory_iterator it(root, ec), end; it != end; it.increment(ec)) {
            if (ec) throw IoError("cannot traverse directory: " + root.string());
            if (it->is_regular_file()) files_.push_back(it->path());
          }
        } else {
          for (fs::directory_iterator it(root, ec), end; it != end; it.increment(ec)) {
            if (ec) throw IoError("cannot traverse directory: " + root.string());
            if (it->is_regular_file()) files_.push_back(it->path());
          }
        }
      } else {
        throw ConfigError("corpus root does not exist: " + root.string());
      }
    }
    std::sort(files_.begin(), files_.end(),
              [](const fs::path& a, const fs::path& b) { return a.native() < b.native(); });
    files_.erase(std::unique(files_.begin(), files_.end()), files_.end());
  }

  // Visits every sequence in enumeration order.
  void for_each(const std::function<void(const Sequence&)>& fn) const {
    uint64_t next_id = 0;
    if (spec_.in_memory.has_value()) {
      Sequence seq;
      for (const auto& bytes : *spec_.in_memory) {
        seq.id = next_id++;
        seq.bytes = bytes;
        fn(seq);
      }
      return;
    }
    for (const auto& path : files_) walk_file(path, next_id, fn);
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
  void walk_file(const std::filesystem::path& path, uint64_t& next_id,
                 const std::function<void(const Sequence&)>& fn) const {
    constexpr size_t kBlock = 1 << 20;
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open file: " + path.string());
    Sequence seq;
    std::string block(kBlock, '\0');
    if (spec_.line_mode) {
      std::string carry;
      for (;;) {
        in.read(block.data(), static_cast<std::streamsize>(block.size()));
        const size_t got = static_cast<size_t>(in.gcount());
        if (in.bad()) throw IoError("read error: " + path.string());
        size_t start = 0;
        for (size_t i = 0; i < got; ++i) {
          if (block[i] == '\n') {
            seq.id = next_id++;
            seq.bytes = std::move(carry);
            seq.bytes.append(block, start, i - start);
            carry.clear();
            fn(seq);
            start = i + 1;
          }
        }
        carry.append(block, start, got - start);
        if (got < block.size()) break;
      }
      if (!carry.empty()) {
        seq.id = next_id++;
        seq.bytes = std::move(carry);
        fn(seq);
      }
    } else if (spec_.chunk_size > 0) {
      for (;;) {
        std::string chunk(spec_.chunk_size, '\0');
        in.read(chunk.data(), static_cast<std::streamsize>(spec_.chunk_size));
        const size_t got = static_cast<size_t>(in.gcount());
        if (in.bad()) throw IoError("read error: " + path.string());
        if (got == 0) break;
        chunk.resize(got);
        seq.id = next_id++;
        seq.bytes = std::move(chunk);
        fn(seq);
        if (got < spec_.chunk_size) break;
      }
    } else {
      std::string data;
      for (;;) {
        in.read(block.data(), static_cast<std::streamsize>(block.size()));
        const size_t got = static_cast<size_t>(in.gcount());
        if (in.bad()) throw IoError("read error: " + path.string());
        data.append(block, 0, got);
        if (got < block.size()) break;
      }
      seq.id = next_id++;
      seq.bytes = std::move(data);
      fn(seq);
    }
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
