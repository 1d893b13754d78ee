// nccl.cu — the library's own NCCL communicators.
//
// The reference's only parallel strategy is data parallelism over whole
// sequences, merged into one table per pass (proj/include/intergrams/
// pipeline.hpp:101-199, merger :154-178).  On GPUs that is: each device
// counts a byte-balanced shard of whole sequences (ig_shard_range), and every
// pass's table is summed in place with one NCCL all-reduce over NVLink /
// NVSwitch; selection then runs identically on every device, so no other
// exchange exists.  Two ways to get there:
//
//   * one process per GPU (torchrun, MPI, ...): the caller moves a 128-byte
//     id from ig_nccl_unique_id to every rank; ig_session_create_nccl builds
//     the rank's communicator (ncclCommInitRank);
//   * one process, several GPUs: ig_topk_ngrams_multi builds every
//     communicator at once (ncclCommInitAll) and drives one session per
//     device from its own host thread.
//
// NCCL is loaded at first use (dlopen "libnccl.so.2"), so the library itself
// loads without it; when a framework already loaded one (torch's), the same
// copy is used.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "session.h"

namespace igb {

namespace {

struct NcclApi {
  void* h = nullptr;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*abort)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
  NcclApi a;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (a.h) break;
  }
  if (!a.h) {
    const char* e = dlerror();
    a.why = std::string("cannot load NCCL (libnccl.so.2): ") + (e ? e : "not found");
    return a;
  }
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.h, name));
    if (!fn && a.why.empty()) a.why = std::string("NCCL symbol missing: ") + name;
  };
  sym(a.get_unique_id, "ncclGetUniqueId");
  sym(a.init_rank, "ncclCommInitRank");
  sym(a.init_all, "ncclCommInitAll");
  sym(a.all_reduce, "ncclAllReduce");
  sym(a.destroy, "ncclCommDestroy");
  sym(a.abort, "ncclCommAbort");
  sym(a.error_string, "ncclGetErrorString");
  return a;
}

const NcclApi& nccl() {
  static const NcclApi a = load_nccl();
  if (!a.why.empty()) throw Error(IG_EINTERNAL, a.why);
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(IG_EINTERNAL, std::string(what) + ": " + nccl().error_string(r));
}

// A session's communicator: the ig_collective hook the driver already calls
// for every pass table (session.cu: allreduce / allreduce_table).
struct NcclColl {
  ncclComm_t comm = nullptr;
  std::atomic<bool> aborted{false};  // ncclCommAbort'ed (a rank failed)
  void abort() {
    if (!aborted.exchange(true)) nccl().abort(comm);
  }
};

int nccl_allreduce_cb(void* buf, uint64_t count, int32_t dtype, void* stream, void* user) {
  auto* c = static_cast<NcclColl*>(user);
  if (c->aborted) return 1;
  const ncclResult_t r = nccl().all_reduce(buf, buf, count, dtype == 0 ? ncclUint32 : ncclUint64,
                                           ncclSum, c->comm, static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : 1;
}

void free_coll(void* p) {
  auto* c = static_cast<NcclColl*>(p);
  if (c->comm && !c->aborted.load()) nccl().destroy(c->comm);
  delete c;
}

void attach(Session& s, ncclComm_t comm, int32_t rank, int32_t world, uint64_t bytes_total,
            uint64_t seqs_total) {
  auto* c = new NcclColl();
  c->comm = comm;
  s.nccl = c;
  s.nccl_free = free_coll;
  s.coll.rank = rank;
  s.coll.world = world;
  s.coll.bytes_total = bytes_total;
  s.coll.seqs_total = seqs_total;
  s.coll.allreduce = nccl_allreduce_cb;
  s.coll.user = c;
  s.has_coll = true;
}

}  // namespace

}  // namespace igb

using namespace igb;

extern "C" {

int ig_nccl_unique_id(uint8_t id_out[128], char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    memcpy(id_out, &id, sizeof(id));
  });
}

int ig_session_create_nccl(int32_t device, void* cuda_stream, int32_t rank, int32_t world,
                           const uint8_t id[128], uint64_t bytes_total, uint64_t seqs_total,
                           ig_session** out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!out || !id) throw Error(IG_ECONFIG, "null argument");
    if (world < 1 || rank < 0 || rank >= world) throw Error(IG_ECONFIG, "bad rank / world");
    ig_session* s = create(device, cuda_stream, nullptr);
    try {
      ncclUniqueId uid;
      memcpy(&uid, id, sizeof(uid));
      ncclComm_t comm = nullptr;
      IGB_CUDA(cudaSetDevice(s->device));
      nccl_check(nccl().init_rank(&comm, world, uid, rank), "ncclCommInitRank");
      attach(*s, comm, rank, world, bytes_total, seqs_total);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int ig_topk_ngrams_multi(const ig_corpus* corpus, const int32_t* devices, int32_t ndev,
                         const ig_params* params, ig_result* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!corpus || !devices || !params || !out) throw Error(IG_ECONFIG, "null argument");
    if (ndev < 1) throw Error(IG_ECONFIG, "device list is empty");
    if (corpus->location != IG_HOST)
      throw Error(IG_ECONFIG, "a multi-GPU run takes a host corpus (each device loads its shard)");
    validate(*params);
    const uint64_t m = corpus->num_seqs;
    const uint64_t* off = corpus->offsets;
    const uint64_t total = m ? off[m] : 0;
    std::vector<ncclComm_t> comms((size_t)ndev, nullptr);
    nccl_check(nccl().init_all(comms.data(), ndev, devices), "ncclCommInitAll");
    std::vector<ig_session*> ss((size_t)ndev, nullptr);
    std::vector<ig_result> rs((size_t)ndev);
    std::vector<std::exception_ptr> errs((size_t)ndev);
    std::atomic<bool> failed{false};
    std::mutex abort_mu;
    auto abort_all = [&] {  // unblocks the ranks waiting in a collective
      std::lock_guard<std::mutex> lk(abort_mu);
      if (failed.exchange(true)) return;
      for (auto* x : ss)
        if (x && x->nccl) static_cast<NcclColl*>(x->nccl)->abort();
    };
    try {
      for (int i = 0; i < ndev; ++i) {
        memset(&rs[(size_t)i], 0, sizeof(ig_result));
        ss[(size_t)i] = create(devices[i], nullptr, nullptr);
        attach(*ss[(size_t)i], comms[(size_t)i], i, ndev, total, m);
        comms[(size_t)i] = nullptr;  // owned by the session now
      }
    } catch (...) {
      for (auto c : comms)
        if (c) nccl().destroy(c);
      for (auto* x : ss) ig_session_destroy(x);
      throw;
    }
    std::vector<std::thread> th;
    for (int i = 0; i < ndev; ++i) {
      th.emplace_back([&, i] {
        try {
          uint64_t a = 0, b = m;
          ig_shard_range(off, m, i, ndev, &a, &b);
          std::vector<uint64_t> so(b - a + 1);
          for (uint64_t q = a; q <= b; ++q) so[q - a] = off[q] - off[a];
          ig_corpus shard{corpus->data + (m ? off[a] : 0), so.data(), b - a, IG_HOST};
          char e2[1024] = {0};
          const int rc = ig_session_run_host(ss[(size_t)i], &shard, params, &rs[(size_t)i], e2,
                                             sizeof(e2));
          if (rc != IG_OK) throw Error(rc, e2);
        } catch (...) {
          errs[(size_t)i] = std::current_exception();
          abort_all();
        }
      });
    }
    for (auto& t : th) t.join();
    std::exception_ptr first;
    for (auto& e : errs)
      if (e && !first) first = e;
    // every device selected from the same summed tables: the lists must agree
    if (!first)
      for (int i = 1; i < ndev; ++i) {
        const ig_result& a = rs[0];
        const ig_result& b = rs[(size_t)i];
        if (a.len != b.len || memcmp(a.grams, b.grams, a.len * a.gram_len) ||
            memcmp(a.counts, b.counts, a.len * 8)) {
          first = std::make_exception_ptr(
              Error(IG_EINTERNAL, "devices disagree on the top-k list"));
          break;
        }
      }
    for (int i = 0; i < ndev; ++i) {
      if (i > 0 || first) ig_result_free(&rs[(size_t)i]);
      ig_session_destroy(ss[(size_t)i]);
    }
    if (first) std::rethrow_exception(first);
    *out = rs[0];
  });
}

}  // extern "C"
