// exact.cu — sort-based exact n-gram counting on the GPU, and the three
// reference entry points built on it:
//
//   ig_naive_topk     naive_count + naive_topk    proj/src/oracle.cpp:7-47
//   ig_hashgram_topk  run_hashgram (Algorithm 1)  proj/src/hashgram.cpp:325-383
//   ig_featurize      featurize (Boolean matrix)  proj/src/metrics.cpp:83-132
//
// The Intergrams passes count into dense tables; these paths have no bounded
// id space (every distinct n-gram, or B hash buckets), so they count by
// SORTING instead:
//
//   emit     one thread per 16 byte positions of a 4096-byte chunk evaluates
//            its grams (bytes held in registers, big-endian key by funnel
//            shifts), keeps the hits of this path (every gram / its bucket /
//            grams of kept buckets / vocabulary hits), and writes them in
//            POSITION ORDER (count kernel + scan + emit kernel);
//   sort     cub radix sort of the u64 ids (count-once: pairs (id, sequence),
//            stable, so equal ids keep ascending sequence order);
//   reduce   run-length (count-all) or reduce-by-key over "first (id, seq)
//            occurrence" flags (count-once) -> unique ids + counts;
//   merge    batches of whole sequences (<= kBatchBytes) are merged by a
//            second sort + reduce-by-key;
//   top-k    stable radix sort of counts descending over the id-ascending
//            list == canonical order (count desc, gram bytes asc,
//            counting.hpp:38-41) for one gram length.
//
// Memory: ~24 B per position of a batch (keys + values, double-buffered).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "session.h"

namespace igb {

namespace {

constexpr int kXT = 256;            // threads per CTA
constexpr int kXP = 16;             // byte positions per thread
constexpr int kXChunk = kXT * kXP;  // bytes per CTA
constexpr uint64_t kBatchBytes = 512ull << 20;

enum EmitKind {
  kEmitGram = 0,       // every gram (naive)
  kEmitBucket = 1,     // its hash bucket (hash-gramming pass 1)
  kEmitKeptGram = 2,   // grams of kept buckets (hash-gramming pass 2)
  kEmitVocab = 3,      // vocabulary hits (featurize)
  kEmitCandidate = 4,  // extension-pass candidate index rank * 256 + last byte
  kEmitChain = 5       // the same for j >= 9 byte grams (rank chain, below)
};

struct EmitSpec {
  const uint8_t* data = nullptr;  // corpus byte g at data[g] (16-aligned, zero padded)
  const uint64_t* off = nullptr;  // [m+1]
  uint32_t q0 = 0, q1 = 0;        // sequences of this batch
  uint64_t g0 = 0, g1 = 0;        // their bytes: off[q0] .. off[q1]
  uint64_t c0 = 0;                // first 4096-byte chunk, g0 / kXChunk
  uint32_t n = 0;
  uint64_t seed = 0, buckets = 1;
  const uint64_t* kept_bits = nullptr;    // kept-bucket bitset, or
  const uint64_t* kept_sorted = nullptr;  // sorted kept buckets
  uint64_t nkept = 0;
  const uint64_t* vkeys = nullptr;  // vocabulary open-addressing table
  const uint32_t* vcols = nullptr;  // column per slot, ~0u = empty
  uint32_t vlg = 0;
  DevPrefixSet ps;  // kEmitCandidate: open-addressing survivor set (p = rank)
  // kEmitChain: ps holds the 8-byte survivors (p = rank in key order) and
  // remap[L - 9][p * 256 + byte] is the rank of an L-byte survivor in id
  // (= byte) order, ~0u when the L-gram did not survive
  const uint32_t* const* remap = nullptr;
};

__host__ __device__ inline uint64_t bswap64(uint64_t x) {
#ifdef __CUDA_ARCH__
  const uint32_t lo = __byte_perm((uint32_t)x, 0, 0x0123);
  const uint32_t hi = __byte_perm((uint32_t)(x >> 32), 0, 0x0123);
  return ((uint64_t)lo << 32) | hi;
#else
  return __builtin_bswap64(x);
#endif
}

// MurmurHash64A (mix64, hashgram.cpp:22-59) of a gram of n <= 8 bytes given
// as its little-endian value `le` (byte 0 lowest).
__host__ __device__ inline uint64_t mix64_le(uint64_t le, uint32_t n, uint64_t seed) {
  const uint64_t m = 0xc6a4a7935bd1e995ull;
  const int r = 47;
  uint64_t h = seed ^ ((uint64_t)n * m);
  if (n == 8) {
    uint64_t k = le;
    k *= m;
    k ^= k >> r;
    k *= m;
    h ^= k;
    h *= m;
  } else if (n > 0) {
    h ^= le;
    h *= m;
  }
  h ^= h >> r;
  h *= m;
  h ^= h >> r;
  return h;
}

__device__ __forceinline__ bool kept_bucket(const EmitSpec& sp, uint64_t b) {
  if (sp.kept_bits) return (sp.kept_bits[b >> 6] >> (b & 63)) & 1;
  uint64_t lo = 0, hi = sp.nkept;  // lower_bound
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (sp.kept_sorted[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  return lo < sp.nkept && sp.kept_sorted[lo] == b;
}

__device__ __forceinline__ uint32_t vocab_col(const EmitSpec& sp, uint64_t key) {
  uint32_t slot = (uint32_t)((key * kCuckooMul1) >> (64 - sp.vlg));
  const uint32_t mask = (1u << sp.vlg) - 1;
  for (;;) {
    const uint32_t c = sp.vcols[slot];
    if (c == 0xffffffffu) return c;
    if (sp.vkeys[slot] == key) return c;
    slot = (slot + 1) & mask;
  }
}

__device__ __forceinline__ uint32_t survivor_rank(const DevPrefixSet& ps, uint64_t key) {
  uint32_t h = hash_slot(key, ps.lgS, ps.hmask);
  for (;;) {
    const uint64_t k = ps.hkeys[h];
    if (k == key) return ps.hidx[h];
    if (k == kEmptyKey) return 0xffffffffu;
    h = (h + 1) & (ps.S - 1);
  }
}

// Evaluates this thread's 16 positions of chunk `chunk`: bit i of the result
// is set when position chunk*4096 + tid*16 + i emits val[i] (sequence seq[i]).
template <int KIND>
__device__ __forceinline__ uint32_t eval_thread(const EmitSpec& sp, uint64_t chunk,
                                                uint64_t (&val)[kXP], uint32_t (&seq)[kXP]) {
  const uint64_t p0 = chunk * kXChunk + (uint64_t)threadIdx.x * kXP;
  if (p0 + kXP <= sp.g0 || p0 >= sp.g1) return 0;
  const uint4 a = *reinterpret_cast<const uint4*>(sp.data + p0);
  const uint4 b = *reinterpret_cast<const uint4*>(sp.data + p0 + 16);
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  // sequence of the first position: last s in [q0, q1) with off[s] <= p
  const uint64_t p = p0 > sp.g0 ? p0 : sp.g0;
  uint32_t lo = sp.q0, hi = sp.q1;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sp.off[mid] <= p) lo = mid;
    else hi = mid;
  }
  uint32_t s = lo;
  uint64_t send = sp.off[s + 1];
  const uint32_t n = sp.n;
  const uint64_t nmask = n >= 8 ? ~0ull : ((1ull << (8 * n)) - 1);
  uint32_t mask = 0;
#pragma unroll
  for (int i = 0; i < kXP; ++i) {
    const uint64_t g = p0 + i;
    if (g >= sp.g0 && g < sp.g1) {
      while (g >= send) {
        ++s;
        send = sp.off[s + 1];
      }
      if (g + n <= send) {
        // bytes i .. i+7 little-endian
        const int wi = i >> 2, sh = 8 * (i & 3);
        const uint32_t l32 = __funnelshift_r(w[wi], w[wi + 1], sh);
        const uint32_t h32 = __funnelshift_r(w[wi + 1], w[wi + 2], sh);
        const uint64_t le = (((uint64_t)h32 << 32) | l32) & nmask;
        // big-endian packed gram (its first 8 bytes when n > 8)
        const uint64_t key = n >= 8 ? bswap64(le) : bswap64(le) >> (64 - 8 * n);
        bool hit = true;
        uint64_t v = key;
        if (KIND == kEmitBucket) {
          v = mix64_le(le, n, sp.seed) % sp.buckets;
        } else if (KIND == kEmitKeptGram) {
          hit = kept_bucket(sp, mix64_le(le, n, sp.seed) % sp.buckets);
        } else if (KIND == kEmitVocab) {
          const uint32_t c = vocab_col(sp, key);
          hit = c != 0xffffffffu;
          v = ((uint64_t)s << 32) | c;
        } else if (KIND == kEmitCandidate) {
          const uint32_t r = survivor_rank(sp.ps, key >> 8);
          hit = r != 0xffffffffu;
          v = (uint64_t)r * 256 + (key & 0xff);
        } else if (KIND == kEmitChain) {
          // the (n-1)-byte prefix's rank, walked up from its first 8 bytes
          // (a trie below depth 8, as PrefixTrie::lookup walks it byte by
          // byte, trie.cpp:139-160)
          uint32_t r = survivor_rank(sp.ps, key);
          for (uint32_t L = 9; L < n && r != 0xffffffffu; ++L)
            r = __ldg(sp.remap[L - 9] + ((uint64_t)r * 256 + sp.data[g + L - 1]));
          hit = r != 0xffffffffu;
          v = (uint64_t)r * 256 + sp.data[g + n - 1];
        }
        if (hit) {
          mask |= 1u << i;
          val[i] = v;
          seq[i] = s;
        }
      }
    }
  }
  return mask;
}

template <int KIND>
__global__ void __launch_bounds__(kXT) k_exact_count(EmitSpec sp, unsigned long long* cnt) {
  uint64_t v[kXP];
  uint32_t q[kXP];
  const uint32_t mask = eval_thread<KIND>(sp, sp.c0 + blockIdx.x, v, q);
  using Reduce = cub::BlockReduce<uint32_t, kXT>;
  __shared__ typename Reduce::TempStorage ts;
  const uint32_t tot = Reduce(ts).Sum((uint32_t)__popc(mask));
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

template <int KIND, bool VALS>
__global__ void __launch_bounds__(kXT) k_exact_emit(EmitSpec sp, const unsigned long long* base,
                                                    uint64_t* keys, uint32_t* vals) {
  uint64_t v[kXP];
  uint32_t q[kXP];
  const uint32_t mask = eval_thread<KIND>(sp, sp.c0 + blockIdx.x, v, q);
  using Scan = cub::BlockScan<uint32_t, kXT>;
  __shared__ typename Scan::TempStorage ts;
  uint32_t rank;
  Scan(ts).ExclusiveSum((uint32_t)__popc(mask), rank);
  uint64_t o = base[blockIdx.x] + rank;
#pragma unroll
  for (int i = 0; i < kXP; ++i) {
    if ((mask >> i) & 1) {
      keys[o] = v[i];
      if (VALS) vals[o] = q[i];
      ++o;
    }
  }
}

// flag[i] = 1 on the first element of each (id, sequence) run.
__global__ void k_first_flags(const uint64_t* keys, const uint32_t* seqs, uint64_t n,
                              uint32_t* flags) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flags[i] = (i == 0 || keys[i] != keys[i - 1] || seqs[i] != seqs[i - 1]) ? 1u : 0u;
}

__global__ void k_widen(const uint32_t* src, uint64_t n, uint64_t* dst) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

__global__ void k_set_bits(const uint64_t* ids, uint64_t n, unsigned long long* bits) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicOr(&bits[ids[i] >> 6], 1ull << (ids[i] & 63));
}

struct AddU32 {
  __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a + b; }
};
struct AddU64 {
  __device__ uint64_t operator()(uint64_t a, uint64_t b) const { return a + b; }
};

inline unsigned grid_of(uint64_t n, unsigned t = 256) { return (unsigned)((n + t - 1) / t); }

int bits_for(uint64_t maxv) {
  int b = 1;
  while (b < 64 && (maxv >> b) != 0) ++b;
  return b;
}

// cub temp storage helper: query, grow, run.
template <typename F>
void cub_call(Session& s, F&& f) {
  size_t need = 0;
  IGB_CUDA(f((void*)nullptr, need));
  void* tmp = s.ex.cub_tmp.get(need + 16);
  IGB_CUDA(f(tmp, need));
}

// Batches of whole sequences with <= kBatchBytes each (a longer sequence is
// its own batch).
std::vector<std::pair<uint32_t, uint32_t>> make_batches(const Session& s) {
  std::vector<std::pair<uint32_t, uint32_t>> out;
  const uint64_t m = s.dc.m;
  uint64_t batch_bytes = kBatchBytes;
  if (const char* e = getenv("IG_EXACT_BATCH_BYTES"))  // test knob: force batch merges
    batch_bytes = std::max<uint64_t>(1, strtoull(e, nullptr, 10));
  uint64_t q = 0;
  while (q < m) {
    const uint64_t q0 = q;
    const uint64_t b0 = s.hoff[q0];
    while (q < m && s.hoff[q + 1] - b0 <= batch_bytes) ++q;
    if (q == q0) ++q;
    if (s.hoff[q] - b0 >= (1ull << 31))
      throw Error(IG_ECONFIG, "exact GPU counter: a sequence of 2 GiB or more is not supported");
    out.emplace_back((uint32_t)q0, (uint32_t)q);
  }
  return out;
}

// Emits the hits of sequences [q0, q1) in position order into ex.keys (and
// the sequence of each into ex.vals when `vals`).  Returns the hit count.
template <int KIND>
uint64_t emit(Session& s, EmitSpec sp, uint32_t q0, uint32_t q1, bool vals) {
  sp.data = s.dc.data;
  sp.off = s.dc.off;
  sp.q0 = q0;
  sp.q1 = q1;
  sp.g0 = s.hoff[q0];
  sp.g1 = s.hoff[q1];
  if (sp.g1 <= sp.g0) return 0;
  sp.c0 = sp.g0 / kXChunk;
  const uint64_t nchunks = (sp.g1 + kXChunk - 1) / kXChunk - sp.c0;
  auto* cnt = s.ex.chunk_cnt.as<unsigned long long>(nchunks + 1);
  auto* base = s.ex.chunk_base.as<unsigned long long>(nchunks + 1);
  IGB_CUDA(cudaMemsetAsync(cnt + nchunks, 0, 8, s.stream));
  k_exact_count<KIND><<<(unsigned)nchunks, kXT, 0, s.stream>>>(sp, cnt);
  IGB_LAUNCHED(&s);
  cub_call(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt, base, (int64_t)(nchunks + 1), s.stream);
  });
  unsigned long long total = 0;
  IGB_CUDA(cudaMemcpyAsync(&total, base + nchunks, 8, cudaMemcpyDeviceToHost, s.stream));
  IGB_CUDA(cudaStreamSynchronize(s.stream));
  if (total == 0) return 0;
  uint64_t* keys = s.ex.keys.as<uint64_t>(total);
  uint32_t* v = vals ? s.ex.vals.as<uint32_t>(total) : nullptr;
  if (vals)
    k_exact_emit<KIND, true><<<(unsigned)nchunks, kXT, 0, s.stream>>>(sp, base, keys, v);
  else
    k_exact_emit<KIND, false><<<(unsigned)nchunks, kXT, 0, s.stream>>>(sp, base, keys, v);
  IGB_LAUNCHED(&s);
  return total;
}

// Exact counts of the ids a KIND emission produces over the whole corpus:
// unique ids ascending in ex.acc_keys, their counts (u64) in ex.acc_counts.
template <int KIND>
uint64_t exact_count(Session& s, const EmitSpec& sp, int mode, int id_bits) {
  const bool once = mode == IG_MODE_ONCE;
  uint64_t acc = 0;
  for (const auto& bq : make_batches(s)) {
    const uint64_t N = emit<KIND>(s, sp, bq.first, bq.second, once);
    if (N == 0) continue;
    uint64_t* k_in = s.ex.keys.as<uint64_t>(N);
    uint64_t* k_out = s.ex.keys2.as<uint64_t>(N);
    uint64_t* uniq = s.ex.uniq.as<uint64_t>(N);
    uint32_t* runs = s.ex.runs.as<uint32_t>(N);
    uint64_t* nr = s.ex.nruns.as<uint64_t>(1);
    if (once) {
      uint32_t* v_in = s.ex.vals.as<uint32_t>(N);
      uint32_t* v_out = s.ex.vals2.as<uint32_t>(N);
      cub_call(s, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, k_in, k_out, v_in, v_out, (int64_t)N, 0,
                                               id_bits, s.stream);
      });
      uint32_t* flags = s.ex.flags.as<uint32_t>(N);
      k_first_flags<<<grid_of(N), 256, 0, s.stream>>>(k_out, v_out, N, flags);
      IGB_LAUNCHED(&s);
      cub_call(s, [&](void* t, size_t& b) {
        return cub::DeviceReduce::ReduceByKey(t, b, k_out, uniq, flags, runs, nr, AddU32{},
                                              (int64_t)N, s.stream);
      });
    } else {
      cub_call(s, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortKeys(t, b, k_in, k_out, (int64_t)N, 0, id_bits,
                                              s.stream);
      });
      cub_call(s, [&](void* t, size_t& b) {
        return cub::DeviceRunLengthEncode::Encode(t, b, k_out, uniq, runs, nr, (int64_t)N,
                                                  s.stream);
      });
    }
    s.launches += 4;  // sort + reduce (cub)
    uint64_t U = 0;
    IGB_CUDA(cudaMemcpyAsync(&U, nr, 8, cudaMemcpyDeviceToHost, s.stream));
    IGB_CUDA(cudaStreamSynchronize(s.stream));
    if (acc == 0) {
      uint64_t* ak = s.ex.acc_keys.as<uint64_t>(U);
      uint64_t* ac = s.ex.acc_counts.as<uint64_t>(U);
      IGB_CUDA(cudaMemcpyAsync(ak, uniq, U * 8, cudaMemcpyDeviceToDevice, s.stream));
      k_widen<<<grid_of(U), 256, 0, s.stream>>>(runs, U, ac);
      IGB_LAUNCHED(&s);
      acc = U;
      continue;
    }
    // merge: concatenate, sort by id, sum counts of equal ids
    const uint64_t M = acc + U;
    uint64_t* mk = s.ex.mrg_keys.as<uint64_t>(M);
    uint64_t* mc = s.ex.mrg_counts.as<uint64_t>(M);
    uint64_t* mk2 = s.ex.mrg_keys2.as<uint64_t>(M);
    uint64_t* mc2 = s.ex.mrg_counts2.as<uint64_t>(M);
    IGB_CUDA(cudaMemcpyAsync(mk, s.ex.acc_keys.p, acc * 8, cudaMemcpyDeviceToDevice, s.stream));
    IGB_CUDA(cudaMemcpyAsync(mc, s.ex.acc_counts.p, acc * 8, cudaMemcpyDeviceToDevice, s.stream));
    IGB_CUDA(cudaMemcpyAsync(mk + acc, uniq, U * 8, cudaMemcpyDeviceToDevice, s.stream));
    k_widen<<<grid_of(U), 256, 0, s.stream>>>(runs, U, mc + acc);
    IGB_LAUNCHED(&s);
    cub_call(s, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, mk, mk2, mc, mc2, (int64_t)M, 0, id_bits,
                                             s.stream);
    });
    uint64_t* ak = s.ex.acc_keys.as<uint64_t>(M);
    uint64_t* ac = s.ex.acc_counts.as<uint64_t>(M);
    cub_call(s, [&](void* t, size_t& b) {
      return cub::DeviceReduce::ReduceByKey(t, b, mk2, ak, mc2, ac, nr, AddU64{}, (int64_t)M,
                                            s.stream);
    });
    s.launches += 4;
    IGB_CUDA(cudaMemcpyAsync(&acc, nr, 8, cudaMemcpyDeviceToHost, s.stream));
    IGB_CUDA(cudaStreamSynchronize(s.stream));
  }
  return acc;
}

// Canonical top-k of the U unique ids in ex.acc_keys / ex.acc_counts (ids
// ascending): stable sort by count descending.  Results on the host.
void exact_topk(Session& s, uint64_t U, uint64_t k, std::vector<uint64_t>& keys,
                std::vector<uint64_t>& counts) {
  keys.clear();
  counts.clear();
  if (U == 0) return;
  uint64_t* ck = s.ex.mrg_counts.as<uint64_t>(U);
  uint64_t* kk = s.ex.mrg_keys.as<uint64_t>(U);
  const uint64_t* ac = (const uint64_t*)s.ex.acc_counts.p;
  const uint64_t* ak = (const uint64_t*)s.ex.acc_keys.p;
  cub_call(s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairsDescending(t, b, ac, ck, ak, kk, (int64_t)U, 0, 64,
                                                     s.stream);
  });
  s.launches += 4;
  const uint64_t len = std::min<uint64_t>(k, U);
  keys.resize(len);
  counts.resize(len);
  IGB_CUDA(cudaMemcpyAsync(keys.data(), kk, len * 8, cudaMemcpyDeviceToHost, s.stream));
  IGB_CUDA(cudaMemcpyAsync(counts.data(), ck, len * 8, cudaMemcpyDeviceToHost, s.stream));
  IGB_CUDA(cudaStreamSynchronize(s.stream));
}

template <typename CT>
__global__ void k_put_counts(const uint64_t* keys, const uint64_t* counts, uint64_t n, CT* table) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) table[keys[i]] = (CT)counts[i];
}

void fill_result(ig_result* out, uint32_t n, const std::vector<uint64_t>& keys,
                 const std::vector<uint64_t>& counts, const std::vector<Row>& rows,
                 StepTimer* tm) {
  memset(out, 0, sizeof(*out));
  const uint64_t len = keys.size();
  out->len = len;
  out->gram_len = n;
  out->keys = (uint64_t*)malloc((len + 1) * 8);
  out->counts = (uint64_t*)malloc((len + 1) * 8);
  out->passes = (ig_pass_stat*)malloc((rows.size() + 1) * sizeof(ig_pass_stat));
  out->diagnostics = (char*)malloc(1);
  out->grams = (uint8_t*)malloc(len * n + 1);
  if (!out->keys || !out->counts || !out->passes || !out->diagnostics || !out->grams) {
    ig_result_free(out);
    throw Error(IG_EINTERNAL, "host allocation failed");
  }
  if (len) {
    memcpy(out->keys, keys.data(), len * 8);
    memcpy(out->counts, counts.data(), len * 8);
  }
  for (uint64_t i = 0; i < len; ++i)
    for (uint32_t b = 0; b < n; ++b) out->grams[i * n + b] = (uint8_t)(keys[i] >> (8 * (n - 1 - b)));
  for (size_t i = 0; i < rows.size(); ++i) {
    out->passes[i] = rows[i].st;
    if (tm) out->passes[i].seconds = tm->seconds(rows[i].ev);
  }
  out->num_passes = (uint32_t)rows.size();
  out->diagnostics[0] = 0;
}

template <typename F>
void with_session(const ig_corpus* corpus, int32_t device, F&& f) {
  ig_session* s = create(device, nullptr, nullptr);
  try {
    load_corpus(*s, *corpus);
    f(*s);
  } catch (...) {
    delete s;
    throw;
  }
  delete s;
}

}  // namespace

// Count-once extension pass by sorting (the fallback for survivor sets too
// large for the route path's 16-bit owners): (rank * 256 + last byte,
// sequence) pairs for every position whose prefix survived, deduplicated per
// sequence and counted, then written into the pass table (table zeroed by the
// caller).
template <typename CT>
void count_once_exact(Session& s, uint32_t L, const DevPrefixSet& ps, uint64_t cap, CT* table) {
  EmitSpec sp;
  sp.n = L;
  sp.ps = ps;
  const uint64_t U = exact_count<kEmitCandidate>(s, sp, IG_MODE_ONCE, bits_for(cap ? cap - 1 : 0));
  if (U == 0) return;
  k_put_counts<CT><<<grid_of(U), 256, 0, s.stream>>>(
      static_cast<const uint64_t*>(s.ex.acc_keys.p), static_cast<const uint64_t*>(s.ex.acc_counts.p),
      U, table);
  IGB_LAUNCHED(&s);
}
template void count_once_exact<uint32_t>(Session&, uint32_t, const DevPrefixSet&, uint64_t,
                                         uint32_t*);

// Extension pass j >= 9 (grams longer than the packed u64 keys), both count
// modes, by sorting: every position whose (j-1)-byte prefix survived emits
// (rank * 256 + last byte[, sequence]); ids, counts and selection are the
// reference's (intergrams.cpp:44-66), since ranks follow byte order.
template <typename CT>
void count_chain_exact(Session& s, uint32_t j, const DevPrefixSet& ps8,
                       const uint32_t* const* remap, int mode, uint64_t cap, CT* table) {
  EmitSpec sp;
  sp.n = j;
  sp.ps = ps8;
  sp.remap = remap;
  const uint64_t U = exact_count<kEmitChain>(s, sp, mode, bits_for(cap ? cap - 1 : 0));
  if (U == 0) return;
  k_put_counts<CT><<<grid_of(U), 256, 0, s.stream>>>(
      static_cast<const uint64_t*>(s.ex.acc_keys.p), static_cast<const uint64_t*>(s.ex.acc_counts.p),
      U, table);
  IGB_LAUNCHED(&s);
}
template void count_chain_exact<uint32_t>(Session&, uint32_t, const DevPrefixSet&,
                                          const uint32_t* const*, int, uint64_t, uint32_t*);
template void count_chain_exact<unsigned long long>(Session&, uint32_t, const DevPrefixSet&,
                                                    const uint32_t* const*, int, uint64_t,
                                                    unsigned long long*);

// remap[ids[r]] = r for the survivors sorted by id (the table was set to ~0u).
__global__ void k_scatter_rank(const uint64_t* __restrict__ ids, uint64_t n,
                               uint32_t* __restrict__ remap) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) remap[ids[i]] = (uint32_t)i;
}

void launch_scatter_rank(const uint64_t* sorted_ids, uint64_t n, uint32_t* remap,
                         cudaStream_t st) {
  if (n) k_scatter_rank<<<grid_of(n), 256, 0, st>>>(sorted_ids, n, remap);
}
template void count_once_exact<unsigned long long>(Session&, uint32_t, const DevPrefixSet&,
                                                   uint64_t, unsigned long long*);

}  // namespace igb

using namespace igb;

extern "C" {

uint64_t ig_mix64(const uint8_t* bytes, uint64_t len, uint64_t seed) {
  // MurmurHash64A exactly as mix64 (hashgram.cpp:22-59): 8-byte little-endian
  // blocks, then the tail
  const uint64_t m = 0xc6a4a7935bd1e995ull;
  const int r = 47;
  uint64_t h = seed ^ (len * m);
  const uint8_t* p = bytes;
  uint64_t rem = len;
  while (rem >= 8) {
    uint64_t k = 0;
    for (int b = 7; b >= 0; --b) k = (k << 8) | p[b];
    k *= m;
    k ^= k >> r;
    k *= m;
    h ^= k;
    h *= m;
    p += 8;
    rem -= 8;
  }
  uint64_t tail = 0;
  for (uint64_t i = rem; i-- > 0;) tail = (tail << 8) | p[i];
  if (rem > 0) {
    h ^= tail;
    h *= m;
  }
  h ^= h >> r;
  h *= m;
  h ^= h >> r;
  return h;
}

int ig_naive_topk(const ig_corpus* corpus, uint32_t n, uint64_t k, int32_t mode,
                  uint64_t max_corpus_bytes, int32_t device, ig_result* out, char* err,
                  size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!corpus || !out) throw Error(IG_ECONFIG, "null argument");
    // naive_count (oracle.cpp:7-19), then naive_topk (:37-39)
    if (n < 1) throw Error(IG_ECONFIG, "gram length must be >= 1");
    if (mode != IG_MODE_ONCE && mode != IG_MODE_ALL) throw Error(IG_ECONFIG, "bad count mode");
    {
      uint64_t total = 0;
      if (corpus->num_seqs) {
        if (corpus->location == IG_DEVICE)
          IGB_CUDA(cudaMemcpy(&total, corpus->offsets + corpus->num_seqs, 8,
                              cudaMemcpyDeviceToHost));
        else
          total = corpus->offsets[corpus->num_seqs];
      }
      if (total > max_corpus_bytes)
        throw Error(IG_ECONFIG, "oracle corpus size guard exceeded (" +
                                    std::to_string(max_corpus_bytes) + " bytes)");
    }
    if (n > IG_MAX_N)
      throw Error(IG_ECONFIG, "gram length n above 8 is not supported by the packed-u64 GPU path");
    if (k < 1) throw Error(IG_ECONFIG, "top-k requires k >= 1");
    with_session(corpus, device, [&](Session& s) {
      EmitSpec sp;
      sp.n = n;
      const uint64_t U = exact_count<kEmitGram>(s, sp, mode, 8 * (int)n);
      std::vector<uint64_t> keys, counts;
      exact_topk(s, U, k, keys, counts);
      fill_result(out, n, keys, counts, {}, nullptr);
    });
  });
}

int ig_hashgram_topk(const ig_corpus* corpus, const ig_hashgram_params* p, ig_result* out,
                     char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!corpus || !p || !out) throw Error(IG_ECONFIG, "null argument");
    // HashgramConfig::validate, hashgram.cpp:16-20
    if (p->buckets < 1) throw Error(IG_ECONFIG, "bucket count B must be >= 1");
    if (p->n < 1) throw Error(IG_ECONFIG, "gram length n must be >= 1");
    if (p->k < 1) throw Error(IG_ECONFIG, "k must be >= 1");
    if (p->mode != IG_MODE_ONCE && p->mode != IG_MODE_ALL)
      throw Error(IG_ECONFIG, "bad count mode");
    if (p->n > IG_MAX_N)
      throw Error(IG_ECONFIG, "gram length n above 8 is not supported by the packed-u64 GPU path");
    with_session(corpus, p->device, [&](Session& s) {
      StepTimer tm(s);
      std::vector<Row> rows;
      EmitSpec sp;
      sp.n = p->n;
      sp.seed = p->seed;
      sp.buckets = p->buckets;
      const int bbits = bits_for(p->buckets - 1);
      // pass 1: bucket counts (hashgram.cpp:336-351)
      size_t ev = tm.begin();
      const uint64_t U1 = exact_count<kEmitBucket>(s, sp, p->mode, bbits);
      tm.end(ev);
      rows.push_back(make_row("hash pass", p->n, s.dc.total, p->buckets, 0, false, ev));
      // top-k buckets (hashgram.cpp:353-362): count desc, bucket id asc
      ev = tm.begin();
      std::vector<uint64_t> kb, kc;
      exact_topk(s, U1, p->k, kb, kc);
      const uint64_t nk = kb.size();
      if (p->buckets <= (1ull << 33)) {
        const uint64_t words = (p->buckets + 63) / 64;
        auto* bits = s.ex.kept.as<unsigned long long>(words);
        IGB_CUDA(cudaMemsetAsync(bits, 0, words * 8, s.stream));
        if (nk) {
          // the kept ids are still on the device (ex.mrg_keys[0..nk))
          k_set_bits<<<grid_of(nk), 256, 0, s.stream>>>((const uint64_t*)s.ex.mrg_keys.p, nk,
                                                         bits);
          IGB_LAUNCHED(&s);
        }
        sp.kept_bits = (const uint64_t*)bits;
      } else {
        std::vector<uint64_t> sorted(kb);
        std::sort(sorted.begin(), sorted.end());
        uint64_t* d = s.ex.kept.as<uint64_t>(nk + 1);
        IGB_CUDA(cudaMemcpyAsync(d, sorted.data(), nk * 8, cudaMemcpyHostToDevice, s.stream));
        IGB_CUDA(cudaStreamSynchronize(s.stream));
        sp.kept_sorted = d;
        sp.nkept = nk;
      }
      tm.end(ev);
      rows.push_back(make_row("top-k buckets", p->n, 0, 0, nk, nk < p->k, ev));
      // pass 2: exact counts of grams in kept buckets (hashgram.cpp:364-375)
      ev = tm.begin();
      uint64_t U2 = 0;
      if (nk) U2 = exact_count<kEmitKeptGram>(s, sp, p->mode, 8 * (int)p->n);
      tm.end(ev);
      rows.push_back(make_row("exact pass", p->n, s.dc.total, 0, U2, false, ev));
      // final top-k (hashgram.cpp:377-380)
      ev = tm.begin();
      std::vector<uint64_t> keys, counts;
      exact_topk(s, U2, p->k, keys, counts);
      tm.end(ev);
      rows.push_back(make_row("top-k grams", p->n, 0, 0, keys.size(), false, ev));
      fill_result(out, p->n, keys, counts, rows, &tm);
    });
  });
}

int ig_featurize(const ig_corpus* corpus, const uint64_t* vocab_keys, uint64_t ncols,
                 uint32_t gram_len, int32_t device, ig_matrix* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!corpus || !out || (ncols && !vocab_keys)) throw Error(IG_ECONFIG, "null argument");
    if (ncols && gram_len > IG_MAX_N)
      throw Error(IG_ECONFIG, "featurize: gram length above 8 is not supported by the GPU path");
    if (ncols >= 0xffffffffull) throw Error(IG_ECONFIG, "featurize: vocabulary too large");
    memset(out, 0, sizeof(*out));
    std::vector<uint64_t> ent;  // (row << 32) | col, sorted
    with_session(corpus, device, [&](Session& s) {
      const uint64_t m = s.dc.m;
      out->rows = m;  // every sequence is a row (metrics.cpp:108-112)
      out->cols = ncols;
      if (ncols == 0) return;
      if (gram_len == 0) {  // the empty gram occurs in every sequence
        ent.resize(m);
        for (uint64_t r = 0; r < m; ++r) ent[r] = r << 32;
        return;
      }
      // vocabulary table: first occurrence of a gram owns it (columns.emplace)
      uint32_t lg = 4;
      while ((1ull << lg) < 2 * ncols) ++lg;
      const uint64_t cap = 1ull << lg;
      std::vector<uint64_t> hk(cap, 0);
      std::vector<uint32_t> hc(cap, 0xffffffffu);
      for (uint64_t j = 0; j < ncols; ++j) {
        const uint64_t key = vocab_keys[j];
        uint32_t slot = (uint32_t)((key * kCuckooMul1) >> (64 - lg));
        while (hc[slot] != 0xffffffffu && hk[slot] != key) slot = (slot + 1) & (uint32_t)(cap - 1);
        if (hc[slot] == 0xffffffffu) {
          hk[slot] = key;
          hc[slot] = (uint32_t)j;
        }
      }
      uint64_t* dk = s.ex.vocab_keys.as<uint64_t>(cap);
      uint32_t* dc = s.ex.vocab_cols.as<uint32_t>(cap);
      IGB_CUDA(cudaMemcpyAsync(dk, hk.data(), cap * 8, cudaMemcpyHostToDevice, s.stream));
      IGB_CUDA(cudaMemcpyAsync(dc, hc.data(), cap * 4, cudaMemcpyHostToDevice, s.stream));
      EmitSpec sp;
      sp.n = gram_len;
      sp.vkeys = dk;
      sp.vcols = dc;
      sp.vlg = lg;
      const int kbits = 32 + bits_for(m ? m - 1 : 0);
      for (const auto& bq : make_batches(s)) {
        const uint64_t N = emit<kEmitVocab>(s, sp, bq.first, bq.second, false);
        if (N == 0) continue;
        uint64_t* k_in = s.ex.keys.as<uint64_t>(N);
        uint64_t* k_out = s.ex.keys2.as<uint64_t>(N);
        uint64_t* uq = s.ex.uniq.as<uint64_t>(N);
        uint64_t* nr = s.ex.nruns.as<uint64_t>(1);
        cub_call(s, [&](void* t, size_t& b) {
          return cub::DeviceRadixSort::SortKeys(t, b, k_in, k_out, (int64_t)N, 0, kbits, s.stream);
        });
        cub_call(s, [&](void* t, size_t& b) {
          return cub::DeviceSelect::Unique(t, b, k_out, uq, nr, (int64_t)N, s.stream);
        });
        s.launches += 4;
        uint64_t U = 0;
        IGB_CUDA(cudaMemcpyAsync(&U, nr, 8, cudaMemcpyDeviceToHost, s.stream));
        IGB_CUDA(cudaStreamSynchronize(s.stream));
        const size_t at = ent.size();
        ent.resize(at + U);
        IGB_CUDA(cudaMemcpyAsync(ent.data() + at, uq, U * 8, cudaMemcpyDeviceToHost, s.stream));
        IGB_CUDA(cudaStreamSynchronize(s.stream));
      }
    });
    const uint64_t nnz = ent.size();
    out->nnz = nnz;
    out->row = (uint64_t*)malloc((nnz + 1) * 8);
    out->col = (uint32_t*)malloc((nnz + 1) * 4);
    if (!out->row || !out->col) {
      ig_matrix_free(out);
      throw Error(IG_EINTERNAL, "host allocation failed");
    }
    for (uint64_t i = 0; i < nnz; ++i) {
      out->row[i] = ent[i] >> 32;
      out->col[i] = (uint32_t)ent[i];
    }
  });
}

void ig_matrix_free(ig_matrix* m) {
  if (!m) return;
  free(m->row);
  free(m->col);
  m->row = nullptr;
  m->col = nullptr;
  m->nnz = 0;
}

}  // extern "C"
