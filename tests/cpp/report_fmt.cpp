// Prints RunReport::to_tsv() / to_json() of the drop-in header
// (include/intergrams/metrics.hpp) for rows read from stdin, one per line:
//   label<TAB>gram_len<TAB>seconds(%a)<TAB>bytes<TAB>cand<TAB>retained<TAB>short
// argv: algorithm echo json(0/1) [jaccard(%a)]
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>

#include "intergrams/metrics.hpp"

using namespace intergrams;

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  std::vector<PassResult> rows;
  std::string line;
  while (std::getline(std::cin, line)) {
    if (line.empty()) continue;
    std::stringstream ss(line);
    std::string f[7];
    for (auto& x : f) std::getline(ss, x, '\t');
    PassResult p;
    p.label = f[0];
    p.gram_len = std::stoull(f[1]);
    p.seconds = std::strtod(f[2].c_str(), nullptr);
    p.bytes_processed = std::stoull(f[3]);
    p.candidate_space = std::stoull(f[4]);
    p.retained = std::stoull(f[5]);
    p.retained_short = f[6] == "1";
    rows.push_back(p);
  }
  RunReport r = make_report(argv[1], argv[2], rows);
  if (argc > 4) r.jaccard_vs_reference = std::strtod(argv[4], nullptr);
  std::cout << (std::atoi(argv[3]) ? r.to_json() : r.to_tsv());
  return 0;
}
