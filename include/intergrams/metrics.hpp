// intergrams/metrics.hpp — the result TSV of /root/reference/proj/src/metrics.cpp:202-232
// (lowercase hex gram, TAB, decimal count, LF), the bit-exact golden format.
#pragma once

#include <string>

#include "intergrams/common.hpp"
#include "intergrams/counting.hpp"

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

}  // namespace intergrams
