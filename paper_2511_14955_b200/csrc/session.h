// session.h — the session object behind the C handle, shared by the
// Intergrams driver (session.cu) and the exact/hashgram/featurize paths
// (exact.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <cstdio>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "ig_internal.cuh"
#include "kernels.h"

namespace igb {

// Buffers of the sort-based exact counter (exact.cu).
struct ExactBufs {
  DevBuf keys, keys2, vals, vals2, chunk_cnt, chunk_base, uniq, runs, nruns, flags;
  DevBuf acc_keys, acc_counts, mrg_keys, mrg_counts, mrg_keys2, mrg_counts2;
  DevBuf kept, vocab_keys, vocab_cols, cub_tmp;
};

struct Session {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool has_coll = false;
  ig_collective coll{};
  int num_sms = 148;
  uint64_t launches = 0;

  // corpus
  DevBuf data, off, tile, order;
  // count-once short sequences (route_kernels.cu: k_once_short), by class
  DevBuf short_w, short_c;
  std::vector<uint32_t> h_short_w, h_short_c;
  uint32_t n_long = 0;  // sequences of > kShortCtaLen bytes: order[0 .. n_long)
  DevBuf direct_items, direct_gbm;  // small-alphabet work items (DirectItem), split bitmaps
  uint32_t n_direct_items = 0, n_direct_split = 0;
  // byte alphabet of the current run (count-once small-alphabet passes)
  DevBuf alpha_dev;      // u32 mask[8] | u8 arank[256] | u8 alpha[256]
  DevBuf compact;        // u32 [K' * A] direct-pass counts
  uint32_t alpha_n = 256;
  std::vector<uint8_t> h_arank;  // byte -> rank in the alphabet (host)
  int32_t corpus_alpha = -1;      // bytes present in the resident corpus (-1: not measured)
  DevBuf calpha_dev;              // u32 mask[9] | pad | u8 arank[256] | u8 alpha[256] (offset 48)
  DevBuf lut;            // u16 [2^(bits*(j-1))] rank-packed prefix -> p
  DevCorpus dc;
  bool loaded = false;

  // pass buffers
  DevBuf table, work, scratch32;
  DevBuf rankbits;    // count-all 3-byte prefix rank bitmap
  DevBuf hot_keys, hot_ids, hot_work, hot_bounds;  // count-all hot-gram tables (§3.2e)
  DevBuf sort_keys, sort_vals, sort_tmp;           // count-all survivors in key order
  DevBuf hitmask[2];  // count-all hit chaining (ping-pong by pass parity)
  // grams longer than 8 bytes (passes j >= 9): per level L >= 9 the survivor
  // ids in id order and the id -> rank table; the device array of tables
  std::vector<std::unique_ptr<DevBuf>> chain_ids, chain_remap;
  DevBuf chain_ptrs, chain_ranks, chain_sort_tmp;
  DevBuf surv_keys, surv_counts, next_keys, next_counts;
  DevBuf pkeys, hkeys, hidx, hpacked, owner, owner_cnt, owner_start, cursor, rank_of_p;
  DevBuf sel_state, sel_hist, sel_scalar, units, unit_first;
  SelectCtx sel;
  ExactBufs ex;
  RouteCtx rc;
  KernelTimer kt;
  PinnedArena pin;  // staging of the run's small transfers (reset per run / load)
  // pipelined host load: the dense pass runs batch by batch as the H2D copies land
  struct Batch {
    uint64_t t0, t1;           // count-all tiles whose bytes are all in the batch
    uint32_t u0, u1, q0, q1;   // count-once units / sequences
    cudaEvent_t ready;         // copy of the batch's bytes done (null: resident)
  };
  std::vector<Batch> batches;
  // host gate before batch i is consumed (file loads: waits until the batch's
  // copies are enqueued, then records its event); empty otherwise
  std::function<void(size_t)> batch_gate;
  std::vector<cudaEvent_t> batch_events;
  std::vector<uint64_t> hoff;  // host offsets of the loaded corpus
  std::vector<uint32_t> hufirst;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> events;

  // pinned staging slabs of the file loader (ingest.cu), created on first use
  void* slabs = nullptr;
  void (*slabs_free)(void*) = nullptr;
  // the library's own NCCL communicator (nccl.cu), when it made one
  void* nccl = nullptr;
  void (*nccl_free)(void*) = nullptr;

  ~Session() {
    if (nccl && nccl_free) nccl_free(nccl);
    if (slabs && slabs_free) slabs_free(slabs);
    for (auto e : events) cudaEventDestroy(e);
    for (auto e : batch_events) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

inline void set_err(char* err, size_t len, const char* msg) {
  if (err && len) {
    strncpy(err, msg, len - 1);
    err[len - 1] = 0;
  }
}

template <typename F>
inline int guarded(char* err, size_t len, F&& f) {
  try {
    f();
    if (guard_mode()) {  // IG_GUARD: no kernel of this call wrote out of bounds
      bool any;
      {
        std::lock_guard<std::mutex> lk(GuardRegistry::get().mu);
        any = !GuardRegistry::get().live.empty();
      }
      if (any) check_guards("C-ABI call");
    }
    if (err && len) err[0] = 0;
    return IG_OK;
  } catch (const Error& e) {
    set_err(err, len, e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_err(err, len, "host allocation failed");
    return IG_EINTERNAL;
  } catch (const std::exception& e) {
    set_err(err, len, e.what());
    return IG_EINTERNAL;
  }
}


// Event pair per step; elapsed read at the end of the run.
struct StepTimer {
  Session& s;
  size_t next = 0;
  explicit StepTimer(Session& ss) : s(ss) {}
  size_t begin() {
    if (next + 2 > s.events.size()) {
      for (int i = 0; i < 16; ++i) {
        cudaEvent_t e;
        IGB_CUDA(cudaEventCreate(&e));
        s.events.push_back(e);
      }
    }
    IGB_CUDA(cudaEventRecord(s.events[next], s.stream));
    next += 2;
    return next - 2;
  }
  void end(size_t i) { IGB_CUDA(cudaEventRecord(s.events[i + 1], s.stream)); }
  double seconds(size_t i) {
    float ms = 0;
    IGB_CUDA(cudaEventSynchronize(s.events[i + 1]));
    IGB_CUDA(cudaEventElapsedTime(&ms, s.events[i], s.events[i + 1]));
    return ms * 1e-3;
  }
};

struct Row {
  ig_pass_stat st;
  size_t ev;
};

inline Row make_row(const std::string& label, uint32_t gl, uint64_t bytes, uint64_t cap,
                    uint64_t retained, bool shrt, size_t ev) {
  Row r;
  memset(&r.st, 0, sizeof(r.st));
  snprintf(r.st.label, sizeof(r.st.label), "%s", label.c_str());
  r.st.gram_len = gl;
  r.st.bytes_processed = bytes;
  r.st.candidate_space = cap;
  r.st.retained = retained;
  r.st.retained_short = shrt ? 1 : 0;
  r.ev = ev;
  return r;
}

// Host->device through the pinned arena (src may be pageable; reusable after
// the call).  Device->host: staged, synchronised, then copied to dst.
inline void h2d(Session& s, void* dst, const void* src, size_t n) {
  if (!n) return;
  void* p = s.pin.get(n);
  memcpy(p, src, n);
  launch_copy(dst, p, n, s.stream);
  s.launches++;
}
inline void d2h(Session& s, void* dst, const void* src, size_t n) {
  if (!n) return;
  void* p = s.pin.get(n);
  launch_copy(p, src, n, s.stream);
  s.launches++;
  IGB_CUDA(cudaStreamSynchronize(s.stream));
  memcpy(dst, p, n);
}

void use_device(Session& s);
void validate(const ig_params& p);
void load_corpus(Session& s, const ig_corpus& c, bool copy_data = true);
uint8_t* alloc_corpus(Session& s, uint64_t total);
void finish_corpus(Session& s, std::vector<uint64_t>& hoff);
void check_offsets(const std::vector<uint64_t>& hoff);
void run(Session& s, const ig_params& p, ig_result* out);
std::vector<uint64_t> plan_batches(Session& s);
// A run over a host corpus that is not page-locked: `mem` (contiguous) or
// `seqs` (one pointer per sequence), offsets `hoff`; bytes stream through
// pinned slabs on host threads while the dense pass counts (ingest.cu).
void run_host_streamed(Session& s, const uint8_t* mem, const uint8_t* const* seqs,
                       std::vector<uint64_t>& hoff, const ig_params& p, ig_result* out);
template <typename CT>
void count_once_exact(Session& s, uint32_t L, const DevPrefixSet& ps, uint64_t cap, CT* table);
// Extension pass j >= 9 (exact.cu): ranks walked from the 8-byte survivors
// (ps8) through the per-level id -> rank tables (remap, device array).
template <typename CT>
void count_chain_exact(Session& s, uint32_t j, const DevPrefixSet& ps8,
                       const uint32_t* const* remap, int mode, uint64_t cap, CT* table);
void launch_scatter_rank(const uint64_t* sorted_ids, uint64_t n, uint32_t* remap,
                         cudaStream_t st);
void init_select(Session& s);

}  // namespace igb

// The opaque C handle.
struct ig_session : igb::Session {};

namespace igb {
ig_session* create(int32_t device, void* stream, const ig_collective* coll);
// An idle session of `device` for a one-shot call (or a new one), and its
// return (kept for the next call unless it held a corpus above 1 GiB).
ig_session* acquire_oneshot(int32_t device);
void release_oneshot(ig_session* s);
}  // namespace igb
