// cli.cpp — the `intergrams` command-line front end on the B200 library.
//
// Mirrors /root/reference/proj/src/cli.cpp: the subcommands `count`
// (:173-177), `bench` (:179-192), `compare` (:234-239) and `featurize`
// (:241-256) with the same flags, defaults, INTERGRAMS_WORKERS override
// (:22-29), config echo (:79-86), outputs (result TSV, RunReport TSV/JSON,
// COO matrix + vocab sidecar) and exit codes 0/2/3/4 (:423-440).  CLI11 is
// not vendored by the reference, so a small parser with the same surface is
// written here.  `theory` and `synth` (analysis / corpus generation) are out
// of scope and exit 2 with a message.
#include "intergrams/cli.hpp"

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <thread>
#include <type_traits>

#include "intergrams/corpus.hpp"
#include "intergrams/hashgram.hpp"
#include "intergrams/intergrams.hpp"
#include "intergrams/metrics.hpp"
#include "intergrams/oracle.hpp"

namespace intergrams {

namespace {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct HelpRequested {
  std::string text;
};

size_t default_workers() {  // cli.cpp:22-29
  if (const char* env = std::getenv("INTERGRAMS_WORKERS")) {
    const long v = std::atol(env);
    if (v >= 1) return static_cast<size_t>(v);
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : hw;
}

uint64_t parse_u64(const std::string& name, const std::string& v) {
  if (v.empty() || v.find_first_not_of("0123456789") != std::string::npos)
    throw ParseError("Invalid value '" + v + "' for option " + name);
  errno = 0;
  const unsigned long long x = std::strtoull(v.c_str(), nullptr, 10);
  if (errno == ERANGE) throw ParseError("Value '" + v + "' out of range for option " + name);
  return x;
}

double parse_double(const std::string& name, const std::string& v) {
  char* end = nullptr;
  errno = 0;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end != '\0' || errno == ERANGE)
    throw ParseError("Invalid value '" + v + "' for option " + name);
  return x;
}

// A subcommand's options: flags, valued options (optionally restricted to a
// set of choices) and one positional list.
class Command {
 public:
  explicit Command(std::string name, std::string help) : name_(std::move(name)), help_(std::move(help)) {}

  void flag(const std::string& names, bool& dst, const std::string& help) {
    add(names, false, help, {}, [&dst](const std::string&) { dst = true; });
  }
  void option(const std::string& names, std::string& dst, const std::string& help,
              std::vector<std::string> choices = {}, bool required = false) {
    add(names, true, help, choices, [&dst](const std::string& v) { dst = v; }, required);
  }
  template <typename T>
  void number(const std::string& names, T& dst, const std::string& help) {
    const std::string nm = long_name(names);
    add(names, true, help, {}, [&dst, nm](const std::string& v) {
      if constexpr (std::is_floating_point_v<T>) dst = static_cast<T>(parse_double(nm, v));
      else dst = static_cast<T>(parse_u64(nm, v));
    });
  }
  void positional(const std::string& name, std::vector<std::string>& dst, bool required,
                  int expected = -1) {
    pos_name_ = name;
    pos_ = &dst;
    pos_required_ = required;
    pos_expected_ = expected;
  }

  void parse(const std::vector<std::string>& args, size_t from) {
    bool only_pos = false;
    for (size_t i = from; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (!only_pos && a == "--") {
        only_pos = true;
        continue;
      }
      if (!only_pos && (a == "-h" || a == "--help")) throw HelpRequested{help_text()};
      if (!only_pos && a.size() > 1 && a[0] == '-' && !is_number(a)) {
        std::string key = a, val;
        bool has_val = false;
        if (a.rfind("--", 0) == 0) {
          const size_t eq = a.find('=');
          if (eq != std::string::npos) {
            key = a.substr(0, eq);
            val = a.substr(eq + 1);
            has_val = true;
          }
        } else if (a.size() > 2) {  // -n3
          key = a.substr(0, 2);
          val = a.substr(2);
          has_val = true;
        }
        Opt* o = find(key);
        if (!o) throw ParseError("The following argument was not expected: " + a);
        if (o->takes_value) {
          if (!has_val) {
            if (i + 1 >= args.size()) throw ParseError(o->display + " requires an argument");
            val = args[++i];
          }
          if (!o->choices.empty()) {
            bool ok = false;
            for (const auto& c : o->choices) ok |= c == val;
            if (!ok) throw ParseError(o->display + ": " + val + " not in {" + join(o->choices) + "}");
          }
          o->set(val);
        } else {
          if (has_val) throw ParseError(o->display + " does not take a value");
          o->set("");
        }
        o->seen = true;
        continue;
      }
      if (!pos_) throw ParseError("The following argument was not expected: " + a);
      pos_->push_back(a);
    }
    for (const auto& o : opts_)
      if (o.required && !o.seen) throw ParseError(o.display + " is required");
    if (pos_ && pos_required_ && pos_->empty()) throw ParseError(pos_name_ + " is required");
    if (pos_ && pos_expected_ >= 0 && static_cast<int>(pos_->size()) != pos_expected_)
      throw ParseError(pos_name_ + ": " + std::to_string(pos_expected_) + " required but received " +
                       std::to_string(pos_->size()));
  }

  std::string help_text() const {
    std::string s = "Usage: intergrams " + name_ + " [OPTIONS]";
    if (pos_) s += " " + pos_name_ + "...";
    s += "\n\n" + help_ + "\n\nOptions:\n";
    for (const auto& o : opts_) s += "  " + o.names + (o.takes_value ? " VALUE" : "") + "  " + o.help + "\n";
    return s;
  }

 private:
  struct Opt {
    std::string names, display, help;
    std::vector<std::string> keys;
    bool takes_value = false, required = false, seen = false;
    std::vector<std::string> choices;
    std::function<void(const std::string&)> set;
  };

  static bool is_number(const std::string& a) {
    return a.size() > 1 && a[0] == '-' && (std::isdigit(static_cast<unsigned char>(a[1])) || a[1] == '.');
  }
  static std::string long_name(const std::string& names) {
    std::string best;
    std::stringstream ss(names);
    for (std::string k; std::getline(ss, k, ',');) best = k;
    return best;
  }
  static std::string join(const std::vector<std::string>& v) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + v[i];
    return s;
  }
  void add(const std::string& names, bool takes_value, const std::string& help,
           std::vector<std::string> choices, std::function<void(const std::string&)> set,
           bool required = false) {
    Opt o;
    o.names = names;
    o.help = help;
    o.takes_value = takes_value;
    o.required = required;
    o.choices = std::move(choices);
    o.set = std::move(set);
    std::stringstream ss(names);
    for (std::string k; std::getline(ss, k, ',');) o.keys.push_back(k);
    o.display = o.keys.back();
    opts_.push_back(std::move(o));
  }
  Opt* find(const std::string& key) {
    for (auto& o : opts_)
      for (const auto& k : o.keys)
        if (k == key) return &o;
    return nullptr;
  }

  std::string name_, help_;
  std::vector<Opt> opts_;
  std::vector<std::string>* pos_ = nullptr;
  std::string pos_name_;
  bool pos_required_ = false;
  int pos_expected_ = -1;
};

struct CorpusFlags {  // cli.cpp:31-45
  std::vector<std::string> inputs;
  bool recurse = false;
  bool line_mode = false;
  uint64_t chunk_size = 0;

  CorpusSpec to_spec() const {
    CorpusSpec spec;
    for (const auto& p : inputs) spec.roots.emplace_back(p);
    spec.recurse = recurse;
    spec.line_mode = line_mode;
    spec.chunk_size = chunk_size;
    return spec;
  }
};

void add_corpus_flags(Command& cmd, CorpusFlags& f) {  // cli.cpp:47-55
  cmd.positional("inputs", f.inputs, true);
  cmd.flag("-r,--recurse", f.recurse, "descend into subdirectories");
  cmd.flag("--line-mode", f.line_mode, "each newline-delimited line is one sequence");
  cmd.number("--chunk-size", f.chunk_size, "split files into fixed-size records of this many bytes");
}

struct CountFlags {  // cli.cpp:57-88
  CorpusFlags corpus;
  std::string algorithm = "intergrams";
  size_t n = 6;
  size_t k = 10000;
  double z = 1.5;
  std::string mode = "once";
  uint64_t buckets = uint64_t{1} << 31;
  uint64_t seed = 0;
  size_t workers = default_workers();
  size_t flush_batch = 8;
  std::string merge = "flush";
  bool hashgram_trie = false;
  bool plain_trie_layout = false;
  std::string output;

  CountMode count_mode() const { return mode == "all" ? CountMode::kAll : CountMode::kOnce; }
  MergeStrategy merge_strategy() const {
    return merge == "atomic" ? MergeStrategy::kAtomic : MergeStrategy::kBatchedFlush;
  }
  std::string echo() const {
    std::ostringstream os;
    os << "algorithm=" << algorithm << " n=" << n << " k=" << k;
    if (algorithm == "intergrams") os << " z=" << z;
    if (algorithm == "hashgram") os << " B=" << buckets << " seed=" << seed;
    os << " mode=" << mode << " workers=" << workers << " flush-batch=" << flush_batch
       << " merge=" << merge;
    return os.str();
  }
};

void add_count_flags(Command& cmd, CountFlags& f) {  // cli.cpp:90-112
  add_corpus_flags(cmd, f.corpus);
  cmd.option("-a,--algorithm", f.algorithm, "intergrams | hashgram | naive",
             {"intergrams", "hashgram", "naive"});
  cmd.number("-n,--n", f.n, "gram length");
  cmd.number("-k,--k", f.k, "number of grams to return");
  cmd.number("-z,--oversample", f.z, "oversample factor; k' = ceil(z*k) candidates kept");
  cmd.option("--mode", f.mode, "once | all", {"once", "all"});
  cmd.number("-B,--buckets", f.buckets, "hashgram bucket count");
  cmd.number("--seed", f.seed, "hashgram hash seed");
  cmd.number("-w,--workers", f.workers, "counting worker threads (no effect on the GPU)");
  cmd.number("--flush-batch", f.flush_batch, "bitsets flushed together (validated only)");
  cmd.option("--merge", f.merge, "flush | atomic (no effect on the GPU)", {"flush", "atomic"});
  cmd.flag("--hashgram-trie", f.hashgram_trie, "counting-trie dictionary in the hashgram exact pass");
  cmd.flag("--plain-trie-layout", f.plain_trie_layout, "disable the frequency-ordered trie layout");
  cmd.option("-o,--output", f.output, "result file (default stdout)");
}

struct CountOutcome {
  TopKList topk;
  std::vector<PassResult> passes;
};

CountOutcome run_count_algorithm(const CountFlags& f) {  // cli.cpp:119-154
  const Corpus corpus(f.corpus.to_spec());
  CountOutcome out;
  if (f.algorithm == "naive") {
    out.topk = naive_topk(corpus, f.n, f.count_mode(), f.k, kOracleCorpusGuard);
  } else if (f.algorithm == "hashgram") {
    HashgramConfig cfg;
    cfg.buckets = f.buckets;
    cfg.n = f.n;
    cfg.k = f.k;
    cfg.mode = f.count_mode();
    cfg.seed = f.seed;
    cfg.merge = f.merge_strategy();
    cfg.workers = f.workers;
    cfg.flush_batch_size = f.flush_batch;
    cfg.trie_second_pass = f.hashgram_trie;
    HashgramResult r = run_hashgram(corpus, cfg);
    out.topk = std::move(r.topk);
    out.passes = std::move(r.passes);
  } else {
    IntergramConfig cfg;
    cfg.n = f.n;
    cfg.k = f.k;
    cfg.z = f.z;
    cfg.mode = f.count_mode();
    cfg.merge = f.merge_strategy();
    cfg.workers = f.workers;
    cfg.flush_batch_size = f.flush_batch;
    cfg.frequency_ordered_trie = !f.plain_trie_layout;
    IntergramsResult r = run_intergrams(corpus, cfg);
    out.topk = std::move(r.topk);
    out.passes = std::move(r.passes);
  }
  return out;
}

void write_text(const std::string& path, const std::string& text, std::ostream& fallback) {
  if (path.empty()) {  // cli.cpp:156-166
    fallback << text;
    return;
  }
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open output file: " + path);
  out << text;
  if (!out) throw IoError("write failed: " + path);
}

std::string read_file(const std::string& path, const std::string& what) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + what + ": " + path);
  std::stringstream buf;
  buf << in.rdbuf();
  return buf.str();
}

const char* kTopHelp =
    "top-k n-gram counting toolkit (B200)\n\n"
    "Usage: intergrams SUBCOMMAND [OPTIONS]\n\n"
    "Subcommands:\n"
    "  count      compute the top-k n-grams of a corpus\n"
    "  bench      run one algorithm and report per-pass timings\n"
    "  compare    Jaccard similarity of two result files\n"
    "  featurize  Boolean occurrence matrix for a gram vocabulary\n";

int dispatch(const std::vector<std::string>& args, std::ostream& out, std::ostream& err) {
  if (args.empty()) {
    err << "error: A subcommand is required\n";
    return 2;
  }
  const std::string& sub = args[0];
  if (sub == "-h" || sub == "--help") {
    out << kTopHelp;
    return 0;
  }
  try {
    if (sub == "count" || sub == "bench") {
      CountFlags f;
      std::string report_format = "tsv", report_file, reference_file;
      Command cmd(sub, sub == "count" ? "compute the top-k n-grams of a corpus"
                                      : "run one algorithm and report per-pass timings");
      add_count_flags(cmd, f);
      if (sub == "bench") {
        cmd.option("--report", report_format, "tsv | json", {"tsv", "json"});
        cmd.option("--report-file", report_file, "write the report here instead of stdout");
        cmd.option("--reference", reference_file, "result TSV to compute Jaccard against");
      }
      cmd.parse(args, 1);
      const CountOutcome outcome = run_count_algorithm(f);
      if (sub == "count") {  // cli.cpp:277-281
        write_text(f.output, topk_to_tsv(outcome.topk), out);
        return 0;
      }
      RunReport report = make_report(f.algorithm, f.echo(), outcome.passes);  // :283-303
      if (!reference_file.empty())
        report.jaccard_vs_reference =
            jaccard(outcome.topk, topk_from_tsv(read_file(reference_file, "reference")));
      if (!f.output.empty()) write_text(f.output, topk_to_tsv(outcome.topk), out);
      write_text(report_file, report_format == "json" ? report.to_json() + "\n" : report.to_tsv(),
                 out);
      return 0;
    }
    if (sub == "compare") {  // cli.cpp:382-396
      std::vector<std::string> files;
      Command cmd(sub, "Jaccard similarity of two result files");
      cmd.positional("files", files, true, 2);
      cmd.parse(args, 1);
      TopKList lists[2];
      for (int i = 0; i < 2; ++i) lists[i] = topk_from_tsv(read_file(files[i], "result file"));
      char line[64];
      std::snprintf(line, sizeof(line), "%.6f\n", jaccard(lists[0], lists[1]));
      out << line;
      return 0;
    }
    if (sub == "featurize") {  // cli.cpp:398-419
      CorpusFlags cf;
      std::string vocab_file, matrix_out, vocab_out;
      size_t workers = default_workers();
      Command cmd(sub, "Boolean occurrence matrix for a gram vocabulary");
      add_corpus_flags(cmd, cf);
      cmd.option("--vocab", vocab_file, "vocabulary TSV (from count)", {}, true);
      cmd.option("--matrix-out", matrix_out, "coordinate-list output file", {}, true);
      cmd.option("--vocab-out", vocab_out, "sidecar vocab file (default <matrix-out>.vocab)");
      cmd.number("-w,--workers", workers, "worker threads (no effect on the GPU)");
      cmd.parse(args, 1);
      const TopKList vocab = topk_from_tsv(read_file(vocab_file, "vocab file"));
      const Corpus corpus(cf.to_spec());
      const FeatureMatrix mat = featurize(corpus, vocab, workers);
      std::string coo;
      for (const auto& [row, col] : mat.entries) {
        coo += std::to_string(row);
        coo += '\t';
        coo += std::to_string(col);
        coo += '\n';
      }
      write_text(matrix_out, coo, out);
      std::string sidecar;
      for (const auto& gc : vocab) {
        sidecar += to_hex(gc.gram);
        sidecar += '\n';
      }
      write_text(vocab_out.empty() ? matrix_out + ".vocab" : vocab_out, sidecar, out);
      err << "rows=" << mat.rows << " cols=" << mat.cols << " nnz=" << mat.entries.size() << "\n";
      return 0;
    }
    if (sub == "theory" || sub == "synth") {
      throw ConfigError("subcommand '" + sub +
                        "' is not part of the B200 build (analysis / corpus generation are out "
                        "of scope; see DESIGN.md)");
    }
    err << "error: The following argument was not expected: " << sub << "\n";
    return 2;
  } catch (const HelpRequested& h) {
    out << h.text;
    return 0;
  } catch (const ParseError& e) {
    err << "error: " << e.what() << "\n";
    return 2;
  }
}

}  // namespace

int run_cli(const std::vector<std::string>& args, std::ostream& out, std::ostream& err) {
  try {  // cli.cpp:423-440
    return dispatch(args, out, err);
  } catch (const ConfigError& e) {
    err << "configuration error: " << e.what() << "\n";
    return 2;
  } catch (const std::domain_error& e) {
    err << "configuration error: " << e.what() << "\n";
    return 2;
  } catch (const IoError& e) {
    err << "io error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    err << "internal error: " << e.what() << "\n";
    return 4;
  }
}

}  // namespace intergrams
