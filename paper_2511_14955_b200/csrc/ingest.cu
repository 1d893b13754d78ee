// ingest.cu — corpus ingestion from files straight into HBM (SURVEY §8(f)
// row 1), with the reference's enumeration semantics (proj/src/corpus.cpp):
//   roots: regular files, or directories (recursive or not) of regular files
//          (:13-37); ConfigError "corpus root does not exist" otherwise;
//   order: all files sorted by path, duplicates removed (:40-53);
//   records per file (:55-135): the whole file; or '\n'-separated lines (a
//          final unterminated line counts when non-empty); or fixed-size
//          chunks (the last one short; an empty file has none).
//
// Data path.  The concatenation of all files is read by a pool of host
// threads (pread) into pinned slabs and copied to HBM on a copy stream, slab
// by slab, so reads and PCIe transfers overlap.  Whole-file and chunk records
// land directly in the session's corpus buffer (offsets follow from the file
// sizes).  Line records land in a raw buffer; the GPU then drops every '\n'
// byte (stream compaction into the corpus buffer) and lists the newline
// positions, from which the host derives the sequence offsets.
#include <cub/cub.cuh>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <filesystem>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "session.h"

namespace igb {

namespace fs = std::filesystem;

namespace {

constexpr size_t kSlabBytes = 32ull << 20;
constexpr int kSlabs = 16;

struct FileList {
  std::vector<std::string> paths;
  std::vector<uint64_t> start;  // byte offset of each file in the concatenation (+ total)
};

// corpus.cpp:13-53
FileList enumerate(const ig_file_corpus& spec) {
  if (!spec.roots || spec.num_roots == 0)
    throw Error(IG_ECONFIG, "corpus spec has no roots and no in-memory data");
  std::vector<fs::path> files;
  for (uint64_t r = 0; r < spec.num_roots; ++r) {
    const fs::path root(spec.roots[r] ? spec.roots[r] : "");
    std::error_code ec;
    if (fs::is_regular_file(root, ec)) {
      files.push_back(root);
      continue;
    }
    if (fs::is_directory(root, ec)) {
      auto take = [&](const fs::directory_entry& e) {
        std::error_code ec2;
        if (e.is_regular_file(ec2)) files.push_back(e.path());
      };
      if (spec.recurse) {
        for (fs::recursive_directory_iterator it(root, ec), end; it != end; it.increment(ec)) {
          if (ec) throw Error(IG_EIO, "cannot traverse directory: " + root.string());
          take(*it);
        }
      } else {
        for (fs::directory_iterator it(root, ec), end; it != end; it.increment(ec)) {
          if (ec) throw Error(IG_EIO, "cannot traverse directory: " + root.string());
          take(*it);
        }
      }
      if (ec) throw Error(IG_EIO, "cannot traverse directory: " + root.string());
      continue;
    }
    throw Error(IG_ECONFIG, "corpus root does not exist: " + root.string());
  }
  std::sort(files.begin(), files.end(),
            [](const fs::path& a, const fs::path& b) { return a.native() < b.native(); });
  files.erase(std::unique(files.begin(), files.end()), files.end());
  FileList fl;
  fl.start.push_back(0);
  for (const auto& f : files) {
    struct stat st;
    if (::stat(f.c_str(), &st) != 0) throw Error(IG_EIO, "cannot open file: " + f.string());
    fl.paths.push_back(f.string());
    fl.start.push_back(fl.start.back() + (uint64_t)st.st_size);
  }
  return fl;
}

// Offsets of whole-file (chunk == 0) or chunk records (corpus.cpp:100-135).
std::vector<uint64_t> record_offsets(const FileList& fl, uint64_t chunk) {
  std::vector<uint64_t> off{0};
  for (size_t f = 0; f < fl.paths.size(); ++f) {
    const uint64_t a = fl.start[f], b = fl.start[f + 1];
    if (chunk == 0) {
      off.push_back(b);
    } else {
      for (uint64_t x = a; x < b; x += chunk) off.push_back(std::min(x + chunk, b));
    }
  }
  return off;
}

// Pinned staging slabs of a session (allocated once, reused).
struct Slabs {
  void* host[kSlabs] = {};
  cudaEvent_t done[kSlabs] = {};
  int64_t item[kSlabs];  // last item staged in the slab (-1: none)
  int device = 0;
  std::mutex mu;
  std::condition_variable cv;
  ~Slabs() {
    for (int i = 0; i < kSlabs; ++i) {
      if (host[i]) cudaFreeHost(host[i]);
      if (done[i]) cudaEventDestroy(done[i]);
    }
  }
};

// Pinned slab sets are pooled per process: allocating 16 x 32 MiB of pinned
// memory costs ~0.3 s, which would dominate a one-shot call on a small
// corpus.  A session borrows a set on first use and returns it when it is
// destroyed; concurrent sessions get sets of their own.
struct SlabPool {
  std::mutex mu;
  std::map<int, std::vector<Slabs*>> free;  // by device (the events belong to one)
  static SlabPool& get() {
    static SlabPool* p = new SlabPool();  // never destroyed: sets live for the process
    return *p;
  }
};

void return_slabs(void* p) {
  auto* sl = static_cast<Slabs*>(p);
  SlabPool& pool = SlabPool::get();
  std::lock_guard<std::mutex> lk(pool.mu);
  pool.free[sl->device].push_back(sl);
}

Slabs& slabs_of(Session& s) {
  if (!s.slabs) {
    Slabs* sl = nullptr;
    {
      SlabPool& pool = SlabPool::get();
      std::lock_guard<std::mutex> lk(pool.mu);
      auto& v = pool.free[s.device];
      if (!v.empty()) {
        sl = v.back();
        v.pop_back();
      }
    }
    if (!sl) {
      sl = new Slabs();
      sl->device = s.device;
      try {
        for (int i = 0; i < kSlabs; ++i) {
          IGB_CUDA(cudaHostAlloc(&sl->host[i], kSlabBytes, cudaHostAllocPortable));
          IGB_CUDA(cudaEventCreateWithFlags(&sl->done[i], cudaEventDisableTiming));
        }
      } catch (...) {
        delete sl;
        throw;
      }
    }
    s.slabs = sl;
    s.slabs_free = return_slabs;
  }
  return *static_cast<Slabs*>(s.slabs);
}

// Where the streamed bytes come from: the concatenation of files, or host
// memory that is not page-locked (one contiguous buffer, or one pointer per
// sequence — the reference's in-memory Corpus without a packed copy).
struct HostSource {
  const FileList* files = nullptr;
  const uint8_t* mem = nullptr;
  const uint8_t* const* seqs = nullptr;
  const uint64_t* seq_start = nullptr;  // [m + 1] byte offset of each sequence
  uint64_t m = 0;
  uint64_t total = 0;
};

// Copies the source's bytes to dev[0 .. total) through the pinned slabs:
// reader threads take slab-sized items in order; item j reuses slab
// j % kSlabs once item j - kSlabs's copy has completed.  start() returns at
// once; wait_bytes(e) blocks until every copy of bytes [0, e) has been
// enqueued on the copy stream; finish() joins the readers, waits for the
// copies and rethrows the first reader error.
class FileStreamer {
 public:
  FileStreamer(Session& s, const HostSource& src, uint8_t* dev) : s_(s), src_(src), dev_(dev) {}
  ~FileStreamer() {
    failed_.store(true);
    sl_cv_notify();
    join();
  }

  void start() {
    total_ = src_.total;
    if (total_ == 0) return;
    sl_ = &slabs_of(s_);
    if (!s_.copy_stream)
      IGB_CUDA(cudaStreamCreateWithFlags(&s_.copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < kSlabs; ++i) sl_->item[i] = -1;
    nitems_ = (int64_t)((total_ + kSlabBytes - 1) / kSlabBytes);
    enqueued_.assign((size_t)nitems_, 0);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nthreads = (int)std::min<int64_t>(std::min<unsigned>(hw, 16u), nitems_);
    for (int i = 0; i < nthreads; ++i) pool_.emplace_back([this] { worker(); });
  }

  void wait_bytes(uint64_t end) {
    if (total_ == 0 || end == 0) return;
    const int64_t need = (int64_t)((std::min(end, total_) + kSlabBytes - 1) / kSlabBytes);
    std::unique_lock<std::mutex> lk(sl_->mu);
    sl_->cv.wait(lk, [&] { return failed_.load() || prefix_ >= need; });
    if (failed_.load()) {
      lk.unlock();
      finish();
    }
  }

  void finish() {
    join();
    if (total_) IGB_CUDA(cudaStreamSynchronize(s_.copy_stream));
    if (first_error_) std::rethrow_exception(first_error_);
  }

 private:
  void sl_cv_notify() {
    if (sl_) sl_->cv.notify_all();
  }
  void join() {
    for (auto& th : pool_)
      if (th.joinable()) th.join();
    pool_.clear();
  }

  void worker() {
    Slabs& sl = *sl_;
    int fd = -1;
    size_t fd_file = (size_t)-1;
    try {
      IGB_CUDA(cudaSetDevice(s_.device));
      for (;;) {
        const int64_t j = next_.fetch_add(1);
        if (j >= nitems_ || failed_.load()) break;
        const int b = (int)(j % kSlabs);
        {  // wait until the slab's previous item has been copied out
          std::unique_lock<std::mutex> lk(sl.mu);
          sl.cv.wait(lk, [&] { return failed_.load() || j < kSlabs || sl.item[b] == j - kSlabs; });
          if (failed_.load()) break;
        }
        if (j >= kSlabs) IGB_CUDA(cudaEventSynchronize(sl.done[b]));
        const uint64_t a0 = (uint64_t)j * kSlabBytes;
        const uint64_t a1 = std::min<uint64_t>(total_, a0 + kSlabBytes);
        uint8_t* buf = static_cast<uint8_t*>(sl.host[b]);
        if (src_.mem) {
          memcpy(buf, src_.mem + a0, a1 - a0);
        } else if (src_.seqs) {
          const uint64_t* st = src_.seq_start;
          size_t q = (size_t)(std::upper_bound(st, st + src_.m + 1, a0) - st) - 1;
          for (uint64_t x = a0; x < a1;) {
            while (st[q + 1] <= x) ++q;  // skip empty sequences
            const uint64_t e = std::min<uint64_t>(a1, st[q + 1]);
            memcpy(buf + (x - a0), src_.seqs[q] + (x - st[q]), e - x);
            x = e;
          }
        } else {
          const FileList& fl = *src_.files;
          size_t f = (size_t)(std::upper_bound(fl.start.begin(), fl.start.end(), a0) -
                              fl.start.begin()) - 1;
          uint64_t x = a0;
          while (x < a1) {
            while (fl.start[f + 1] <= x) ++f;  // skip empty files
            if (fd_file != f) {
              if (fd >= 0) ::close(fd);
              fd = ::open(fl.paths[f].c_str(), O_RDONLY);
              if (fd < 0) throw Error(IG_EIO, "cannot open file: " + fl.paths[f]);
              fd_file = f;
            }
            const uint64_t want = std::min<uint64_t>(a1, fl.start[f + 1]) - x;
            uint64_t got = 0;
            while (got < want) {
              const ssize_t r = ::pread(fd, buf + (x - a0) + got, want - got,
                                        (off_t)(x - fl.start[f] + got));
              if (r < 0) throw Error(IG_EIO, "read error: " + fl.paths[f]);
              if (r == 0) throw Error(IG_EIO, "file changed while reading: " + fl.paths[f]);
              got += (uint64_t)r;
            }
            x += want;
          }
        }
        IGB_CUDA(cudaMemcpyAsync(dev_ + a0, buf, a1 - a0, cudaMemcpyHostToDevice, s_.copy_stream));
        IGB_CUDA(cudaEventRecord(sl.done[b], s_.copy_stream));
        {
          std::lock_guard<std::mutex> lk(sl.mu);
          sl.item[b] = j;
          enqueued_[(size_t)j] = 1;
          while (prefix_ < nitems_ && enqueued_[(size_t)prefix_]) ++prefix_;
        }
        sl.cv.notify_all();
      }
    } catch (...) {
      {
        std::lock_guard<std::mutex> lk(err_mu_);
        if (!first_error_) first_error_ = std::current_exception();
      }
      failed_.store(true);
      sl.cv.notify_all();
    }
    if (fd >= 0) ::close(fd);
  }

  Session& s_;
  const HostSource& src_;
  uint8_t* dev_;
  Slabs* sl_ = nullptr;
  uint64_t total_ = 0;
  int64_t nitems_ = 0;
  std::atomic<int64_t> next_{0};
  std::atomic<bool> failed_{false};
  std::vector<uint8_t> enqueued_;
  int64_t prefix_ = 0;  // items [0, prefix_) enqueued (under sl_->mu)
  std::exception_ptr first_error_;
  std::mutex err_mu_;
  std::vector<std::thread> pool_;
};

HostSource file_source(const FileList& fl) {
  HostSource src;
  src.files = &fl;
  src.total = fl.start.back();
  return src;
}

void stream_files(Session& s, const FileList& fl, uint8_t* dev) {
  const HostSource src = file_source(fl);
  FileStreamer fs(s, src, dev);
  fs.start();
  fs.finish();
}

struct IsNewline {
  __host__ __device__ bool operator()(uint8_t b) const { return b == '\n'; }
};
struct NotNewline {
  __host__ __device__ bool operator()(uint8_t b) const { return b != '\n'; }
};
struct NewlineAt {
  const uint8_t* raw;
  __host__ __device__ bool operator()(uint64_t i) const { return raw[i] == '\n'; }
};

template <typename F>
void cub_run(Session& s, F&& f) {
  size_t need = 0;
  IGB_CUDA(f((void*)nullptr, need));
  void* tmp = s.ex.cub_tmp.get(need + 16);
  IGB_CUDA(f(tmp, need));
}

// Line records (corpus.cpp:62-95): raw bytes -> the corpus without its '\n'
// bytes (device compaction) + the sequence offsets (host, from the newline
// positions).
void load_lines(Session& s, const FileList& fl) {
  const uint64_t total = fl.start.back();
  DevBuf raw;
  uint8_t* r = raw.as<uint8_t>(total + 16);
  stream_files(s, fl, r);
  // newline positions (ascending)
  uint64_t* nl = s.ex.keys.as<uint64_t>(total + 1);
  uint64_t* nnl = s.ex.nruns.as<uint64_t>(1);
  cub::CountingInputIterator<uint64_t> idx(0);
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceSelect::If(t, b, idx, nl, nnl, (int64_t)total, NewlineAt{r}, s.stream);
  });
  uint64_t n_nl = 0;
  IGB_CUDA(cudaMemcpyAsync(&n_nl, nnl, 8, cudaMemcpyDeviceToHost, s.stream));
  IGB_CUDA(cudaStreamSynchronize(s.stream));
  std::vector<uint64_t> pos(n_nl);
  if (n_nl)
    IGB_CUDA(cudaMemcpyAsync(pos.data(), nl, n_nl * 8, cudaMemcpyDeviceToHost, s.stream));
  IGB_CUDA(cudaStreamSynchronize(s.stream));
  std::vector<uint64_t> hoff{0};
  {  // per file: a sequence per newline, then the tail when non-empty
    size_t k = 0;
    for (size_t f = 0; f < fl.paths.size(); ++f) {
      const uint64_t a = fl.start[f], b = fl.start[f + 1];
      uint64_t line_start = a;
      for (; k < n_nl && pos[k] < b; ++k) {
        // raw [line_start, pos[k]) -> compacted: subtract the newlines before
        hoff.push_back(pos[k] - k);
        line_start = pos[k] + 1;
      }
      if (line_start < b) hoff.push_back(b - k);  // unterminated last line
    }
  }
  check_offsets(hoff);
  const uint64_t out_bytes = total - n_nl;
  uint8_t* data = alloc_corpus(s, out_bytes);
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceSelect::If(t, b, r, data, nnl, (int64_t)total, NotNewline{}, s.stream);
  });
  s.launches += 2;
  finish_corpus(s, hoff);  // synchronises the stream; `raw` can go
}

// Whole-file / chunk records: offsets are known from the sizes, so the dense
// pass consumes sequence-aligned batches while the readers are still
// streaming later files (the batch gate waits for a batch's copies to be
// enqueued, then records its event).  Line records load first, then run.
void run_streamed(Session& s, const HostSource& src, std::vector<uint64_t>& hoff,
                  const ig_params& p, ig_result* out);

void run_files(Session& s, const ig_file_corpus& spec, const ig_params& p, ig_result* out) {
  use_device(s);
  const FileList fl = enumerate(spec);
  if (spec.line_mode) {
    load_lines(s, fl);
    run(s, p, out);
    return;
  }
  std::vector<uint64_t> hoff = record_offsets(fl, spec.chunk_size);
  const HostSource src = file_source(fl);
  run_streamed(s, src, hoff, p, out);
}

// A run whose corpus bytes stream from `src` through the pinned slabs while
// the dense pass consumes sequence-aligned batches as they land (the batch
// gate waits for a batch's copies to be enqueued, then records its event).
void run_streamed(Session& s, const HostSource& src, std::vector<uint64_t>& hoff,
                  const ig_params& p, ig_result* out) {
  check_offsets(hoff);
  uint8_t* data = alloc_corpus(s, src.total);
  finish_corpus(s, hoff);  // synchronises the stream (pads zeroed)
  const std::vector<uint64_t> ends = plan_batches(s);
  FileStreamer fs(s, src, data);
  fs.start();
  s.batch_gate = [&](size_t i) {
    fs.wait_bytes(ends[i]);
    IGB_CUDA(cudaEventRecord(s.batches[i].ready, s.copy_stream ? s.copy_stream : s.stream));
  };
  try {
    run(s, p, out);
  } catch (...) {
    s.batch_gate = nullptr;
    s.batches.clear();
    throw;
  }
  s.batch_gate = nullptr;
  s.batches.clear();
  fs.finish();
}

void load_files(Session& s, const ig_file_corpus& spec) {
  use_device(s);
  const FileList fl = enumerate(spec);
  if (spec.line_mode) {
    load_lines(s, fl);
    return;
  }
  std::vector<uint64_t> hoff = record_offsets(fl, spec.chunk_size);
  check_offsets(hoff);
  uint8_t* data = alloc_corpus(s, fl.start.back());
  IGB_CUDA(cudaStreamSynchronize(s.stream));  // pads zeroed before the copy stream writes
  stream_files(s, fl, data);
  finish_corpus(s, hoff);
}

}  // namespace

// Host corpus that is not page-locked (a contiguous buffer `mem`, or one
// pointer per sequence `seqs`): streamed through the pinned slabs by host
// threads, under the dense pass.
void run_host_streamed(Session& s, const uint8_t* mem, const uint8_t* const* seqs,
                       std::vector<uint64_t>& hoff, const ig_params& p, ig_result* out) {
  use_device(s);
  const std::vector<uint64_t> starts = hoff;  // finish_corpus takes hoff
  HostSource src;
  src.mem = mem;
  src.seqs = seqs;
  src.seq_start = starts.data();
  src.m = starts.size() - 1;
  src.total = starts.back();
  run_streamed(s, src, hoff, p, out);
}

}  // namespace igb

using namespace igb;

extern "C" {

int ig_file_corpus_files(const ig_file_corpus* spec, uint64_t* num_files, uint64_t* total_bytes,
                         char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!spec) throw Error(IG_ECONFIG, "null corpus spec");
    const FileList fl = enumerate(*spec);
    if (num_files) *num_files = fl.paths.size();
    if (total_bytes) *total_bytes = fl.start.back();
  });
}

int ig_file_corpus_list(const ig_file_corpus* spec, ig_file_fn fn, void* user, char* err,
                        size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!spec || !fn) throw Error(IG_ECONFIG, "null corpus spec or callback");
    const FileList fl = enumerate(*spec);
    for (size_t f = 0; f < fl.paths.size(); ++f)
      if (fn(fl.paths[f].c_str(), fl.start[f + 1] - fl.start[f], user) != 0)
        throw Error(IG_ECALLBACK, "file callback stopped the enumeration");
  });
}

int ig_file_corpus_records(const ig_file_corpus* spec, ig_record_fn fn, void* user, char* err,
                           size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!spec || !fn) throw Error(IG_ECONFIG, "null corpus spec or callback");
    const FileList fl = enumerate(*spec);
    uint64_t id = 0;
    auto emit = [&](const uint8_t* p, uint64_t n) {
      if (fn(id++, p, n, user) != 0) throw Error(IG_ECALLBACK, "record callback stopped the walk");
    };
    for (size_t f = 0; f < fl.paths.size(); ++f) {
      const uint64_t size = fl.start[f + 1] - fl.start[f];
      // the file mapped read-only; records are views into the mapping
      const uint8_t* base = nullptr;
      void* map = nullptr;
      int fd = ::open(fl.paths[f].c_str(), O_RDONLY);
      if (fd < 0) throw Error(IG_EIO, "cannot open file: " + fl.paths[f]);
      if (size) {
        map = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
        if (map == MAP_FAILED) {
          ::close(fd);
          throw Error(IG_EIO, "read error: " + fl.paths[f]);
        }
        ::madvise(map, size, MADV_SEQUENTIAL);
        base = static_cast<const uint8_t*>(map);
      }
      ::close(fd);
      struct Unmap {
        void* p;
        uint64_t n;
        ~Unmap() {
          if (p) ::munmap(p, n);
        }
      } um{map, size};
      if (spec->line_mode) {
        uint64_t a = 0;
        while (a < size) {
          const void* nl = memchr(base + a, '\n', size - a);
          const uint64_t e = nl ? (uint64_t)(static_cast<const uint8_t*>(nl) - base) : size;
          if (nl || e > a) emit(base + a, e - a);
          a = e + 1;
        }
      } else if (spec->chunk_size) {
        for (uint64_t a = 0; a < size; a += spec->chunk_size)
          emit(base + a, std::min<uint64_t>(spec->chunk_size, size - a));
      } else {
        emit(base, size);
      }
    }
  });
}

int ig_session_load_files(ig_session* s, const ig_file_corpus* spec, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!s || !spec) throw Error(IG_ECONFIG, "null session or corpus spec");
    load_files(*s, *spec);
  });
}

int ig_session_run_files(ig_session* s, const ig_file_corpus* spec, const ig_params* params,
                         ig_result* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!s || !spec || !params || !out) throw Error(IG_ECONFIG, "null argument");
    validate(*params);
    run_files(*s, *spec, *params, out);
  });
}

int ig_topk_ngrams_files(const ig_file_corpus* spec, const ig_params* params, ig_result* out,
                         char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!spec || !params || !out) throw Error(IG_ECONFIG, "null argument");
    validate(*params);
    ig_session* s = acquire_oneshot(params->device);
    try {
      run_files(*s, *spec, *params, out);
    } catch (...) {
      delete s;
      throw;
    }
    release_oneshot(s);
  });
}

int ig_session_corpus(ig_session* s, uint8_t* data, uint64_t data_cap, uint64_t* offsets,
                      uint64_t offsets_cap, uint64_t* num_seqs, uint64_t* total_bytes, char* err,
                      size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!s || !s->loaded) throw Error(IG_ECONFIG, "no corpus loaded");
    use_device(*s);
    const uint64_t m = s->dc.m, total = s->dc.total;
    if (num_seqs) *num_seqs = m;
    if (total_bytes) *total_bytes = total;
    if (offsets && offsets_cap >= m + 1) memcpy(offsets, s->hoff.data(), (m + 1) * 8);
    if (data && data_cap >= total && total) {
      IGB_CUDA(cudaMemcpyAsync(data, s->dc.data, total, cudaMemcpyDeviceToHost, s->stream));
      IGB_CUDA(cudaStreamSynchronize(s->stream));
    }
  });
}

}  // extern "C"
