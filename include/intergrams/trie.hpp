// intergrams/trie.hpp — drop-in for /root/reference/proj/include/intergrams/trie.hpp
// (src/trie.cpp): the immutable prefix set of an extension pass, ordinal =
// rank in the survivor list.  On the GPU the set is a perfect hash built by
// the library (route_kernels.cu); this host object keeps the reference's
// build validation, lookup semantics and the ordinal order the GPU pass is
// given.  Header-only.
#pragma once

#include <algorithm>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "intergrams/counting.hpp"

namespace intergrams {

class PrefixTrie {
 public:
  PrefixTrie() = default;  // empty trie: depth 0, contains nothing

  // trie.cpp:20-60: equal-length, non-empty, distinct grams; ordinal = index.
  // The layout flag never changes lookups (accepted for API parity).
  static PrefixTrie build(const TopKList& prefixes, bool frequency_ordered_layout = true) {
    (void)frequency_ordered_layout;
    PrefixTrie t;
    if (prefixes.empty()) return t;
    const size_t depth = prefixes[0].gram.size();
    if (depth == 0) throw std::invalid_argument("trie prefixes must be non-empty");
    if (prefixes.size() > (size_t{1} << 31))
      throw std::invalid_argument("too many prefixes for 32-bit ordinals");
    std::vector<std::unordered_set<std::string>> levels(depth);
    for (size_t r = 0; r < prefixes.size(); ++r) {
      const std::string& g = prefixes[r].gram;
      if (g.size() != depth) throw std::invalid_argument("trie prefixes must share one length");
      if (!t.ordinal_.emplace(g, static_cast<uint32_t>(r)).second)
        throw std::invalid_argument("duplicate prefix in trie input");
      for (size_t l = 1; l < depth; ++l) levels[l].insert(g.substr(0, l));
      t.grams_.push_back(g);
    }
    t.depth_ = depth;
    t.size_ = prefixes.size();
    t.nodes_ = 1;
    for (size_t l = 1; l < depth; ++l) t.nodes_ += levels[l].size();
    return t;
  }

  size_t depth() const { return depth_; }
  size_t size() const { return size_; }
  size_t node_count() const { return nodes_; }  // root + distinct proper prefixes

  std::optional<uint32_t> lookup(std::string_view window) const {
    if (size_ == 0) return std::nullopt;  // trie.cpp:140
    if (window.size() != depth_) throw std::invalid_argument("trie lookup window length != depth");
    const auto it = ordinal_.find(std::string(window));
    if (it == ordinal_.end()) return std::nullopt;
    return it->second;
  }
  bool contains(std::string_view window) const { return lookup(window).has_value(); }

  // The grams in ordinal order (what the GPU extension pass is given).
  const std::vector<std::string>& grams() const { return grams_; }

 private:
  size_t depth_ = 0, size_ = 0, nodes_ = 0;
  std::unordered_map<std::string, uint32_t> ordinal_;
  std::vector<std::string> grams_;
};

}  // namespace intergrams
