// hot_kernels.cu — count-all passes with sampled hot-gram tables in shared
// memory.
//
// Reference semantics are those of count_kernels.cu (count-all:
// pipeline.hpp:106-113, counts[id] += 1 per occurrence; extension pass:
// proj/src/intergrams.cpp:44-66, id = p * 256 + last byte when the (j-1)-byte
// prefix is survivor p).  Only the way the additions reach the table changes:
//
//   1. sample  — every 16th to 256th 512-byte tile (~64 MiB) is counted by the
//                plain kernel into a scratch table (thrown away after step 2;
//                the sweeps count every tile, sampled ones included).
//   2. select  — per slice of the table's id range, the ids with the largest
//                sample counts become that slice's hot set (a semi-log
//                histogram picks a threshold; at most 2 candidates per slot).
//   3. build   — each slice's hot grams go into NB two-way buckets, the two
//                hottest keys of a bucket winning it (64-bit atomicMax on
//                (count << 32 | id)).  An empty slot holds a key whose own
//                bucket is a different one, so no query can ever match it.
//   4. sweep   — every tile, once per slice: the CTA keeps its slice's
//                bucket keys (16 B per bucket, one LDS.128 per lookup) and
//                u32 counters in shared memory.  A gram found there is one
//                shared-memory atomic — for an extension pass a hot gram's
//                prefix is known to be a survivor, so the L2 prefix probe is
//                skipped too.  Every other gram takes the plain path (prefix
//                probe + one RED to L2).  A slice is a contiguous id range,
//                so the REDs of one sweep touch 1/S of the table (kept under
//                the L2 knee).  CTAs flush their counters with one RED per
//                nonzero slot when they retire.
//
// Which grams are hot changes nothing but speed: every occurrence is counted
// exactly once, in shared memory or in L2, and the final table is the same
// integer table as the plain kernel's (tests/test_gpu_count_all_paths.py runs
// both against the oracle).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "ig_internal.cuh"
#include "kernels.h"

namespace igb {

constexpr uint64_t kHotMul = 0xA24BAED4963EE407ull;  // bucket hash (odd)
constexpr int kHotBins = 128;                        // semi-log count bins

// Bucket of a hot-table key: a 32-bit mix of both key halves (4 ALU ops in
// the sweep's inner loop instead of a 64-bit multiply).
constexpr uint32_t kHotMul0 = 0x9E3779B1u;  // first multiplier of the low key word
__host__ __device__ __forceinline__ uint32_t hot_bucket(uint64_t key, uint32_t lgnb,
                                                        uint32_t mul) {
  // the top bits of a sum of two odd-multiplier products: 2 IMAD + 1 shift.
  // `mul` (odd) is the table's multiplier of the low key word: a rebuild with
  // another one moves the keys apart that shared a slot.
  const uint32_t h = (uint32_t)key * mul + (uint32_t)(key >> 32) * 0x85EBCA77u;
  return h >> (32 - lgnb);
}

// Semi-log bin of a count c >= 1: 2 * floor(log2 c) + the next bit.
__device__ __forceinline__ uint32_t hot_bin(uint64_t c) {
  const uint32_t bl = 63 - __clzll(c);
  const uint32_t nx = bl ? (uint32_t)((c >> (bl - 1)) & 1) : 0;
  return 2 * bl + nx;
}

struct HotKeyFn {
  const uint64_t* pkeys;  // nullptr: key = id (dense pass)
  __device__ __forceinline__ uint64_t operator()(uint64_t id) const {
    return pkeys ? ((__ldg(pkeys + (id >> 8)) << 8) | (id & 255)) : id;
  }
};

__device__ __forceinline__ uint32_t slice_of(uint64_t id, const HotSliceIds& sl) {
  uint32_t s = 0;
#pragma unroll
  for (int i = 1; i < kMaxHotSlices; ++i)
    if (i < (int)sl.S && id >= sl.lo[i]) s = i;
  return s;
}

// ---------------------------------------------------------------- select

template <typename CT>
__global__ void k_hot_hist(const CT* __restrict__ t, uint64_t cap, HotSliceIds sl,
                           uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kMaxHotSlices * kHotBins];
  for (int i = threadIdx.x; i < kMaxHotSlices * kHotBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t[i];
    if (c) atomicAdd(&h[slice_of(i, sl) * kHotBins + hot_bin(c)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxHotSlices * kHotBins; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// One thread per slice: the lowest bin whose cumulative (from the top) stays
// within `cap` candidates, except that the top bin is always taken.
__global__ void k_hot_thresh(const uint32_t* __restrict__ hist, uint32_t S, uint32_t cap,
                             uint32_t* __restrict__ thr) {
  const uint32_t s = threadIdx.x;
  if (s >= S) return;
  uint64_t cum = 0;
  uint32_t b = kHotBins;
  while (b > 0) {
    const uint32_t n = hist[s * kHotBins + b - 1];
    if (n && cum + n > cap && cum) break;
    cum += n;
    --b;
    if (cum >= cap) break;
  }
  thr[s] = b;
}

template <typename CT>
__global__ void k_hot_collect(const CT* __restrict__ t, uint64_t cap, HotSliceIds sl,
                              const uint32_t* __restrict__ thr, uint32_t ccap,
                              uint32_t* __restrict__ ncand, unsigned long long* __restrict__ cand) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = t[i];
    if (!c) continue;
    const uint32_t s = slice_of(i, sl);
    if (hot_bin(c) < thr[s]) continue;
    const uint32_t pos = atomicAdd(&ncand[s], 1u);
    if (pos < ccap)
      cand[(uint64_t)s * ccap + pos] =
          ((unsigned long long)min(c, (uint64_t)0xffffffffu) << 32) | (uint32_t)i;
  }
}

// Pass w (0, 1): slot w of each bucket takes the best candidate not already
// in slot 0.
__global__ void k_hot_best(const unsigned long long* __restrict__ cand,
                           const uint32_t* __restrict__ ncand, uint32_t S, uint32_t ccap,
                           HotKeyFn kf, uint32_t lgnb, int way,
                           unsigned long long* __restrict__ best,
                           unsigned long long drop_above, uint32_t mul) {
  const uint32_t nb = 1u << lgnb;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < (uint64_t)S * ccap;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(g / ccap), i = (uint32_t)(g % ccap);
    if (i >= min(ncand[s], ccap)) continue;
    const unsigned long long v = cand[g];
    if ((v >> 32) > drop_above) continue;  // experiment: the hottest grams stay cold
    if (way < 0) {  // direct: the way is the next hash bit
      atomicMax(best + (uint64_t)s * nb * 2 + hot_bucket(kf(v & 0xffffffffu), lgnb + 1, mul), v);
      continue;
    }
    const uint32_t b = hot_bucket(kf(v & 0xffffffffu), lgnb, mul);
    unsigned long long* bk = best + ((uint64_t)s * nb + b) * 2;
    if (way == 1 && bk[0] == v) continue;
    atomicMax(bk + way, v);
  }
}

// Direct tables: candidates with a sample count of at least `imp` that lost
// their slot to a hotter key (they would be counted by same-address L2 REDs,
// which serialise: c3's dense pass takes 400 ms instead of 38 with its few
// hottest grams left out).  The host rebuilds two-way when any exists.
__global__ void k_hot_lost(const unsigned long long* __restrict__ cand,
                           const uint32_t* __restrict__ ncand, uint32_t S, uint32_t ccap,
                           HotKeyFn kf, uint32_t lgnb, const unsigned long long* __restrict__ best,
                           unsigned long long imp, uint32_t* __restrict__ lost, bool direct,
                           uint32_t mul) {
  const uint32_t nb = 1u << lgnb;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < (uint64_t)S * ccap;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(g / ccap), i = (uint32_t)(g % ccap);
    if (i >= min(ncand[s], ccap)) continue;
    const unsigned long long v = cand[g];
    if ((v >> 32) < imp) continue;
    const unsigned long long* bs = best + (uint64_t)s * nb * 2;
    const uint64_t key = kf(v & 0xffffffffu);
    bool in;
    if (direct) {
      in = bs[hot_bucket(key, lgnb + 1, mul)] == v;
    } else {
      const uint32_t b = hot_bucket(key, lgnb, mul);
      in = bs[2 * b] == v || bs[2 * b + 1] == v;
    }
    if (!in) atomicAdd(lost, 1u);
  }
}

__global__ void k_hot_fill(const unsigned long long* __restrict__ best, uint32_t S, HotKeyFn kf,
                           uint32_t lgnb, uint64_t* __restrict__ keys, uint32_t* __restrict__ ids,
                           uint32_t mul) {
  const uint32_t nb = 1u << lgnb;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < (uint64_t)S * nb * 2;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)((g >> 1) & (nb - 1));
    const unsigned long long v = best[g];
    if (v) {
      keys[g] = kf(v & 0xffffffffu);
      ids[g] = (uint32_t)v;
    } else {
      // a key this bucket can never be asked for
      uint64_t k = ~0ull;
      for (uint64_t c = 0; hot_bucket(k, lgnb, mul) == b; ++c) k = c;
      keys[g] = k;
      ids[g] = 0xffffffffu;
    }
  }
}

template <typename CT>
void build_hot_set(const CT* table, uint64_t cap, const HotSliceIds& sl, const uint64_t* pkeys,
                   uint32_t lgnb, HotSet& hs, DevBuf& work, int num_sms, cudaStream_t st,
                   bool direct, uint64_t important, uint32_t mul) {
  const uint32_t S = sl.S, nb = 1u << lgnb;
  const uint32_t ccap = 2 * nb * 2;  // candidates per slice: twice the slots
  // work layout: hist | thr | ncand | cand | best
  const size_t o_hist = 0, n_hist = (size_t)kMaxHotSlices * kHotBins * 4;
  const size_t o_thr = o_hist + n_hist, o_nc = o_thr + 64, o_cand = o_nc + 64;
  const size_t o_best = o_cand + (size_t)S * ccap * 8;
  const size_t need = o_best + (size_t)S * nb * 2 * 8;
  char* w = static_cast<char*>(work.get(need));
  uint32_t* hist = reinterpret_cast<uint32_t*>(w + o_hist);
  uint32_t* thr = reinterpret_cast<uint32_t*>(w + o_thr);
  uint32_t* nc = reinterpret_cast<uint32_t*>(w + o_nc);
  auto* cand = reinterpret_cast<unsigned long long*>(w + o_cand);
  auto* best = reinterpret_cast<unsigned long long*>(w + o_best);
  IGB_CUDA(cudaMemsetAsync(w, 0, o_cand, st));
  IGB_CUDA(cudaMemsetAsync(best, 0, (size_t)S * nb * 2 * 8, st));
  const unsigned gb = (unsigned)std::min<uint64_t>((cap + 255) / 256, (uint64_t)num_sms * 8);
  k_hot_hist<CT><<<gb ? gb : 1, 256, 0, st>>>(table, cap, sl, hist);
  k_hot_thresh<<<1, 32, 0, st>>>(hist, S, ccap / 2, thr);
  k_hot_collect<CT><<<gb ? gb : 1, 256, 0, st>>>(table, cap, sl, thr, ccap, nc, cand);
  const HotKeyFn kf{pkeys};
  const unsigned cb = (unsigned)std::min<uint64_t>(((uint64_t)S * ccap + 255) / 256, 4096);
  // IG_HOT_DROP_ABOVE=c (experiment): candidates with a sample count above c
  // are left out of the table, i.e. the hottest grams are counted by L2 REDs
  static const char* drop_env = getenv("IG_HOT_DROP_ABOVE");
  const unsigned long long drop = drop_env ? strtoull(drop_env, nullptr, 10) : ~0ull;
  if (direct) {
    k_hot_best<<<cb, 256, 0, st>>>(cand, nc, S, ccap, kf, lgnb, -1, best, drop, mul);
  } else {
    k_hot_best<<<cb, 256, 0, st>>>(cand, nc, S, ccap, kf, lgnb, 0, best, drop, mul);
    k_hot_best<<<cb, 256, 0, st>>>(cand, nc, S, ccap, kf, lgnb, 1, best, drop, mul);
  }
  hs.lost = nc + 15;  // (zeroed with the work header above)
  k_hot_lost<<<cb, 256, 0, st>>>(cand, nc, S, ccap, kf, lgnb, best,
                                 std::max<unsigned long long>(important, 1), hs.lost, direct, mul);
  const unsigned fb = (unsigned)std::min<uint64_t>(((uint64_t)S * nb * 2 + 255) / 256, 4096);
  k_hot_fill<<<fb, 256, 0, st>>>(best, S, kf, lgnb, hs.keys, hs.ids, mul);
  hs.S = S;
  hs.lgnb = lgnb;
  hs.direct = direct;
  hs.mul = mul;
}

template void build_hot_set<uint32_t>(const uint32_t*, uint64_t, const HotSliceIds&,
                                      const uint64_t*, uint32_t, HotSet&, DevBuf&, int,
                                      cudaStream_t, bool, uint64_t, uint32_t);
template void build_hot_set<unsigned long long>(const unsigned long long*, uint64_t,
                                                const HotSliceIds&, const uint64_t*, uint32_t,
                                                HotSet&, DevBuf&, int, cudaStream_t, bool,
                                                uint64_t, uint32_t);

// ---------------------------------------------------------------- sweep

// The 8 bytes before a lane's 16-byte segment + the segment (count_kernels.cu Seg).
struct HSeg {
  uint32_t W[7];
};

template <int T>
__device__ __forceinline__ uint64_t hkey8_at(const HSeg& s) {
  constexpr int o = T + 1;
  constexpr int wi = o / 4, sh = 8 * (o % 4);
  uint32_t lo, hi;
  if constexpr (sh == 0) {
    lo = s.W[wi];
    hi = s.W[wi + 1];
  } else {
    lo = __funnelshift_r(s.W[wi], s.W[wi + 1], sh);
    hi = __funnelshift_r(s.W[wi + 1], s.W[wi + 2], sh);
  }
  return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | (uint64_t)__byte_perm(hi, 0, 0x0123);
}

template <int L>
__device__ __forceinline__ uint64_t hgram_mask() {
  if constexpr (L >= 8) return ~0ull;
  else return (1ull << (8 * L)) - 1;
}

template <int B, int E, typename F>
__device__ __forceinline__ void hstatic_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    hstatic_for<B + 1, E>(f);
  }
}

// Validity of a segment that crosses sequence boundaries (count_kernels.cu).
template <int L>
__device__ __noinline__ uint32_t hvalid_walk(const uint64_t* __restrict__ off, uint64_t m,
                                             uint64_t total, uint64_t q, int64_t b0) {
  if (b0 >= (int64_t)total) return 0;
  int64_t s0 = (int64_t)off[q], s1 = (int64_t)off[q + 1];
  while (s1 <= b0 && q + 1 < m) {
    ++q;
    s0 = s1;
    s1 = (int64_t)off[q + 1];
  }
  uint32_t vm = 0;
  for (;;) {
    const int64_t lo = s0 + L - 1;
    int64_t a = lo - b0, b = s1 - b0;
    if (a < 0) a = 0;
    if (b > 16) b = 16;
    if (a < b) vm |= ((1u << b) - 1u) & ~((1u << a) - 1u);
    if (s1 >= b0 + 16 || q + 1 >= m) break;
    ++q;
    s0 = s1;
    s1 = (int64_t)off[q + 1];
  }
  return vm;
}

__device__ __forceinline__ uint32_t hlookup_rank(const uint64_t* __restrict__ rankbits,
                                                 uint32_t pre) {
  const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(rankbits) + (pre >> 6));
  const uint64_t bit = 1ull << (pre & 63);
  return (e.x & bit) ? (uint32_t)e.y + (uint32_t)__popcll(e.x & (bit - 1)) : 0xffffffffu;
}

__device__ __forceinline__ uint32_t hlookup_packed(const uint64_t* __restrict__ tab, uint32_t lgS,
                                                   uint32_t ib, uint64_t key) {
  const uint32_t mask = (1u << lgS) - 1;
  uint32_t h = hash_slot(key, lgS);
  for (;;) {
    const uint64_t e = __ldg(tab + h);
    if (e == kEmptyKey) return 0xffffffffu;
    if ((e >> ib) == key) return (uint32_t)(e & ((1ull << ib) - 1));
    h = (h + 1) & mask;
  }
}

__device__ __noinline__ uint32_t hlookup_packed_from(const uint64_t* __restrict__ tab,
                                                     uint32_t lgS, uint32_t ib, uint64_t key,
                                                     uint32_t h) {
  const uint32_t mask = (1u << lgS) - 1;
  for (;;) {
    const uint64_t e = __ldg(tab + h);
    if (e == kEmptyKey) return 0xffffffffu;
    if ((e >> ib) == key) return (uint32_t)(e & ((1ull << ib) - 1));
    h = (h + 1) & mask;
  }
}

__device__ __noinline__ uint32_t hlookup_wide_from(const uint64_t* __restrict__ wide,
                                                   uint32_t lgS, uint64_t key, uint32_t h) {
  const uint32_t mask = (1u << lgS) - 1;
  for (;;) {
    const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(wide) + h);
    if (e.x == key) return (uint32_t)e.y;
    if (e.x == kEmptyKey) return 0xffffffffu;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ uint32_t hlookup_wide(const uint64_t* __restrict__ wide, uint32_t lgS,
                                                 uint64_t key, uint32_t hmask) {
  const uint32_t mask = (1u << lgS) - 1;
  uint32_t h = hash_slot(key, lgS, hmask);
  for (;;) {
    const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(wide) + h);
    if (e.x == key) return (uint32_t)e.y;
    if (e.x == kEmptyKey) return 0xffffffffu;
    h = (h + 1) & mask;
  }
}

// KIND 0: dense pass (gram = id).  KIND 1: extension pass; TAB 3 packed
// global prefix set, 4 {key, p} slots, 5 rank bitmap of 3-byte prefixes.
// CT: pass table (hot flushes); CC: cold REDs (CT itself, or a u32
// per-segment scratch when CT is u64).
// Shared-memory accesses by 32-bit shared address (the extension sweep's
// branch-free inner loop): a 16-byte load, and a predicated add / stores.
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}
__device__ __forceinline__ uint64_t lds_u64_if(uint32_t a, bool p) {
  uint64_t v = 0;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.u64 %0, [%1];\n\t}"
               : "+l"(v) : "r"(a), "r"((uint32_t)p));
  return v;
}
__device__ __forceinline__ ulonglong2 lds_u64x2(uint32_t a) {
  ulonglong2 v;
  asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void red_shared_if(uint32_t a, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q red.shared.add.u32 [%0], 1;\n\t}"
               :: "r"(a), "r"((uint32_t)p) : "memory");
}
__device__ __forceinline__ void st_shared_u64_if(uint32_t a, uint64_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u64 [%0], %1;\n\t}"
               :: "r"(a), "l"(v), "r"((uint32_t)p) : "memory");
}
__device__ __forceinline__ void st_shared_u32_if(uint32_t a, uint32_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
               :: "r"(a), "r"(v), "r"((uint32_t)p) : "memory");
}
__device__ __forceinline__ void st_shared_u16_if(uint32_t a, uint16_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u16 [%0], %1;\n\t}"
               :: "r"(a), "h"(v), "r"((uint32_t)p) : "memory");
}

// A probe that reads whole buckets from the key's (4-aligned) home: TAB 3
// four packed slots (one 32-byte sector, two 16-byte loads) per step, TAB 4
// two {key, p} slots, TAB 5 the rank-bitmap word pair (no probing).  The
// first empty slot ends a miss (linear probing, no deletions).
template <int TAB>
__device__ __forceinline__ uint32_t hlookup_bucket(const uint64_t* __restrict__ ptab,
                                                   const DevPrefixSet& ps, uint64_t pk) {
  if constexpr (TAB == 5) {
    return hlookup_rank(ptab, (uint32_t)pk);
  } else if constexpr (TAB == 3) {
    const uint32_t mask = (1u << ps.lgS) - 1;
    const uint64_t pmask = (1ull << ps.ib) - 1;
    for (uint32_t h = hash_slot(pk, ps.lgS);; h = (h + 4) & mask) {
      const ulonglong2* b = reinterpret_cast<const ulonglong2*>(ptab + h);
      const ulonglong2 x = __ldg(b), y = __ldg(b + 1);
      if (x.x == kEmptyKey) return 0xffffffffu;
      if ((x.x >> ps.ib) == pk) return (uint32_t)(x.x & pmask);
      if (x.y == kEmptyKey) return 0xffffffffu;
      if ((x.y >> ps.ib) == pk) return (uint32_t)(x.y & pmask);
      if (y.x == kEmptyKey) return 0xffffffffu;
      if ((y.x >> ps.ib) == pk) return (uint32_t)(y.x & pmask);
      if (y.y == kEmptyKey) return 0xffffffffu;
      if ((y.y >> ps.ib) == pk) return (uint32_t)(y.y & pmask);
    }
  } else {
    const uint32_t mask = (1u << ps.lgS) - 1;
    for (uint32_t h = hash_slot(pk, ps.lgS, ps.hmask);; h = (h + 2) & mask) {
      const ulonglong2* b = reinterpret_cast<const ulonglong2*>(ptab) + h;
      const ulonglong2 x = __ldg(b), y = __ldg(b + 1);
      if (x.x == pk) return (uint32_t)x.y;
      if (x.x == kEmptyKey) return 0xffffffffu;
      if (y.x == pk) return (uint32_t)y.y;
      if (y.x == kEmptyKey) return 0xffffffffu;
    }
  }
}

// Resolves one cold position's probe whose first slot `e` (slot h) is
// already loaded; later slots (a collision chain, rare at load <= 0.5) are
// read in order.
template <int TAB>
__device__ __forceinline__ uint32_t hresolve(const uint64_t* __restrict__ ptab,
                                             const DevPrefixSet& ps, uint64_t pk, uint32_t h,
                                             ulonglong2 e) {
  if constexpr (TAB == 5) {
    const uint64_t bit = 1ull << (pk & 63);
    return (e.x & bit) ? (uint32_t)e.y + (uint32_t)__popcll(e.x & (bit - 1)) : 0xffffffffu;
  } else if constexpr (TAB == 3) {
    if (e.x == kEmptyKey) return 0xffffffffu;
    if ((e.x >> ps.ib) == pk) return (uint32_t)(e.x & ((1ull << ps.ib) - 1));
    return hlookup_packed_from(ptab, ps.lgS, ps.ib, pk, (h + 1) & ((1u << ps.lgS) - 1));
  } else {
    if (e.x == pk) return (uint32_t)e.y;
    if (e.x == kEmptyKey) return 0xffffffffu;
    return hlookup_wide_from(ptab, ps.lgS, pk, (h + 1) & ((1u << ps.lgS) - 1));
  }
}

// First probe slot of a cold position: TAB 5 the rank-bitmap word pair, 3 a
// packed slot, 4 a {key, p} slot.
template <int TAB>
__device__ __forceinline__ ulonglong2 hfirst(const uint64_t* __restrict__ ptab,
                                             const DevPrefixSet& ps, uint64_t pk, uint32_t& h) {
  if constexpr (TAB == 5) {
    h = 0;
    return __ldg(reinterpret_cast<const ulonglong2*>(ptab) + (pk >> 6));
  } else if constexpr (TAB == 3) {
    h = hash_slot(pk, ps.lgS);
    return make_ulonglong2(__ldg(ptab + h), 0ull);
  } else {
    h = hash_slot(pk, ps.lgS, ps.hmask);
    return __ldg(reinterpret_cast<const ulonglong2*>(ptab) + h);
  }
}

// Per-warp cold queue of the extension sweep (PH): kHotQ gram keys and
// positions, and the hit bits its drains found, per lane.
constexpr int kHotQ = 64;
constexpr size_t kHotQWarpBytes = kHotQ * 8 + kHotQ * 4 + 32 * 4;

template <bool PH>
constexpr int hot_threads() { return 1024; }

template <int KIND, int L, int TAB, typename CT, typename CC, bool PH = false, bool SP = false>
__global__ void __launch_bounds__(hot_threads<PH>(), 1)
    k_count_hot(DevCorpus c, DevPrefixSet ps, const uint64_t* __restrict__ ptab, HotSweep hw,
                CT* __restrict__ table, CC* __restrict__ cold) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t nb = 1u << hw.lgnb;
  ulonglong2* skeys = reinterpret_cast<ulonglong2*>(smem_raw);
  uint32_t* scnt = reinterpret_cast<uint32_t*>(smem_raw + (size_t)nb * 16);
  {
    const ulonglong2* gk = reinterpret_cast<const ulonglong2*>(hw.keys);
    if constexpr (PH && KIND == 1) {
      // a direct table (HotSet::direct): 2 nb slots, slot = the top
      // lgnb + 1 hash bits, one 8-byte load per lookup
      for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) skeys[i] = gk[i];
    } else {
      for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) skeys[i] = gk[i];
    }
    for (uint32_t i = threadIdx.x; i < 2 * nb; i += blockDim.x) scnt[i] = 0;
  }
  const int lane = threadIdx.x & 31;
  // this warp's cold queue (extension sweep with queued probes)
  unsigned char* qbase =
      smem_raw + ((size_t)nb * 24) + (size_t)(threadIdx.x >> 5) * kHotQWarpBytes;
  uint64_t* qkey = reinterpret_cast<uint64_t*>(qbase);
  uint32_t* qpos = reinterpret_cast<uint32_t*>(qbase + kHotQ * 8);
  uint32_t* qhit = reinterpret_cast<uint32_t*>(qbase + kHotQ * 12);
  // 32-bit shared addresses, made opaque so the compiler keeps them in
  // registers instead of rebuilding the shared window base at every use
  const uint32_t s_keys = opaque_u32((uint32_t)__cvta_generic_to_shared(skeys));
  const uint32_t s_cnt = opaque_u32((uint32_t)__cvta_generic_to_shared(scnt));
  const uint32_t s_qkey = opaque_u32((uint32_t)__cvta_generic_to_shared(qkey));
  const uint32_t s_qpos = opaque_u32((uint32_t)__cvta_generic_to_shared(qpos));
  const uint32_t lgnb_s = opaque_u32(31 - hw.lgnb);  // slot = hash >> lgnb_s (lgnb + 1 bits)
  const uint32_t hmul = opaque_u32(hw.mul);          // the table's low-word multiplier
  const uint32_t slot_sh = opaque_u32(64 - ps.lgS);  // hash_slot's shift
  const uint32_t slot_hm = TAB == 4 ? ps.hmask : ~3u;  // and its home alignment
  uint32_t qhead = 0, qtail = 0;  // warp-uniform
  const uint32_t lt_mask = (1u << lane) - 1u;
  if constexpr (PH && KIND == 1) qhit[lane] = 0;
  const bool sliced = hw.sliced;
  __syncthreads();
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t lo = hw.bounds[0], hi = hw.bounds[1];  // this slice's key range
  const bool chain = KIND == 1 && ps.hit_in != nullptr;
  const bool sparse = SP && chain;  // a sparse pass
  // Queue drains are software-pipelined: drain_issue takes 32 queued
  // positions (one per lane) and starts their first bucket loads; they are
  // resolved (compare, RED, hit bit) by drain_resolve at the next drain, a
  // few positions later, so the L2 round trip overlaps hot-path work.  A
  // position carries its tile's iteration number k: if its tile is still
  // the current one its hit bit goes to qhit (merged into the tile's
  // hit-mask store), else straight into hit_out with an atomic OR.
  const uint64_t tfirst = c.tile0 + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
  uint32_t kcur = 0;          // iteration number of the current tile
  bool pf = false;            // a probe in flight on this lane
  uint64_t pfkey = 0;
  uint32_t pfpos = 0;
  ulonglong2 pfa = make_ulonglong2(0, 0), pfb = make_ulonglong2(0, 0);
  auto drain_resolve = [&]() {
    if (pf) {
      uint32_t p;
      const uint64_t pk = pfkey >> 8;
      if constexpr (TAB == 5) {
        const uint64_t bit = 1ull << (pk & 63);
        p = (pfa.x & bit) ? (uint32_t)pfa.y + (uint32_t)__popcll(pfa.x & (bit - 1)) : 0xffffffffu;
      } else if constexpr (TAB == 3) {
        // branch-free over the 4 slots of the bucket: a slot holds
        // (key << ib) | rank, so slot ^ (pk << ib) < 2^ib is a match and its
        // low word the rank (ib < 32: ranks are u32).  Linear probing
        // without deletions: the key cannot lie beyond an empty slot, so
        // match -> hit, else any empty slot -> miss, else the next bucket.
        const uint64_t pks = pk << ps.ib, lim = 1ull << ps.ib;
        const uint64_t x0 = pfa.x ^ pks, x1 = pfa.y ^ pks, x2 = pfb.x ^ pks, x3 = pfb.y ^ pks;
        const bool m0 = x0 < lim, m1 = x1 < lim, m2 = x2 < lim, m3 = x3 < lim;
        const bool anye = (pfa.x == kEmptyKey) | (pfa.y == kEmptyKey) | (pfb.x == kEmptyKey) |
                          (pfb.y == kEmptyKey);
        const uint32_t pv = m0 ? (uint32_t)x0 : m1 ? (uint32_t)x1 : m2 ? (uint32_t)x2 : (uint32_t)x3;
        p = (m0 | m1 | m2 | m3) ? pv : (anye ? 0xffffffffu : 0xfffffffeu);
        if (p == 0xfffffffeu)  // a full bucket: continue from the next one
          p = hlookup_packed_from(ptab, ps.lgS, ps.ib, pk,
                                  (hash_slot(pk, ps.lgS) + 4) & ((1u << ps.lgS) - 1));
      } else {
        // two {key, p} slots, branch-free (same argument as the packed bucket)
        const bool m0 = pfa.x == pk, m1 = pfb.x == pk;
        const bool anye = (pfa.x == kEmptyKey) | (pfb.x == kEmptyKey);
        p = m0 ? (uint32_t)pfa.y : m1 ? (uint32_t)pfb.y : anye ? 0xffffffffu : 0xfffffffeu;
        if (p == 0xfffffffeu)  // both slots taken by other keys: the next bucket
          p = hlookup_wide_from(ptab, ps.lgS, pk,
                                (hash_slot(pk, ps.lgS, ps.hmask) + 2) & ((1u << ps.lgS) - 1));
      }
      if (p != 0xffffffffu) {
        atomicAdd(cold + ((uint64_t)p * 256 + (uint32_t)(pfkey & 0xff)), (CC)1);
        const uint32_t k = pfpos >> 9, el = (pfpos >> 4) & 31, bit = 1u << (pfpos & 15);
        if (k == kcur) {
          atomicOr(qhit + el, bit);
        } else if (ps.hit_out != nullptr) {  // its tile is done: OR into hit_out
          const uint64_t wi = (tfirst + (uint64_t)k * nwarps) * 32 + el;
          atomicOr(reinterpret_cast<unsigned int*>(ps.hit_out) + (wi >> 1), bit << (16 * (wi & 1)));
        }
      }
      pf = false;
    }
  };
  auto drain_issue = [&](uint32_t cnt) {
    if (lane < cnt) {
      const uint32_t qi = (qhead + lane) & (kHotQ - 1);
      pfkey = qkey[qi];
      pfpos = qpos[qi];
      const uint64_t pk = pfkey >> 8;
      if constexpr (TAB == 5) {  // rank bitmap: one 16-byte word pair
        pfa = __ldg(reinterpret_cast<const ulonglong2*>(ptab) + (pk >> 6));
      } else {
        // hash_slot(pk, lgS) with the shift in a register (lgS >= 3 here:
        // tables that fit shared memory take the plain kernel)
        const uint32_t hh = (uint32_t)((pk * 0x9E3779B97F4A7C15ull) >> slot_sh) & slot_hm;
        const ulonglong2* bk = TAB == 3 ? reinterpret_cast<const ulonglong2*>(ptab + hh)
                                        : reinterpret_cast<const ulonglong2*>(ptab) + hh;
        // the 32-byte bucket in one 256-bit load (homes are 32-byte aligned)
        asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(pfa.x), "=l"(pfa.y), "=l"(pfb.x), "=l"(pfb.y)
                     : "l"(bk));
      }
      pf = true;
    }
    qhead += cnt;
    __syncwarp();
  };
  auto drain = [&](uint32_t cnt) {
    drain_resolve();
    drain_issue(cnt);
  };
  uint64_t t = c.tile0 + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
  if (t < c.ntiles) {
    // the next tile's loads stay in flight while the current one is counted.
    // On a sparse pass (ps.sparse: the previous pass hit fewer than half of
    // the positions) the masks run one tile further ahead, and a tile whose
    // mask is empty (no position of it was counted by the previous pass)
    // never reads its corpus bytes: c5's 6- to 8-gram passes touch ~10 % of
    // the 64 GiB.
    auto mask_at = [&](uint64_t tt) -> uint32_t {
      uint32_t m = __ldcs(ps.hit_in + tt * 32 + lane);
      m |= (lane == 0 ? (uint32_t)__ldcs(ps.hit_in + tt * 32 - 1) : 0xffffu) << 16;
      return m;
    };
    auto live_of = [&](uint32_t m) -> bool {  // warp-uniform
      return __any_sync(0xffffffffu, (lane == 0 ? m : (m & 0xffffu)) != 0);
    };
    uint32_t mk = chain ? mask_at(t) : 0xffffffffu;
    uint4 v = make_uint4(0, 0, 0, 0);
    uint2 h = make_uint2(0, 0);
    uint32_t d = 0x80000000u;  // dead tile: "all positions valid" & an empty mask
    bool cur_live = !sparse || live_of(mk);  // warp-uniform: the tile has a live position
    if (cur_live) {
      v = __ldcs(reinterpret_cast<const uint4*>(c.data + t * kTileBytes + lane * 16));
      if (lane == 0) h = *reinterpret_cast<const uint2*>(c.data + t * kTileBytes - 8);
      d = __ldg(c.tile_seq + t);
    }
    // sparse: the mask of tile t + nwarps (else unused: loaded with its tile)
    uint32_t mkn = (sparse && t + nwarps < c.ntiles) ? mask_at(t + nwarps) : 0xffffffffu;
    for (;;) {
      const uint64_t tn = t + nwarps;
      uint4 vn = make_uint4(0, 0, 0, 0);
      uint2 hn = make_uint2(0, 0);
      uint32_t dn = 0x80000000u, mknn = 0xffffffffu;
      bool next_live = true;
      if (sparse) {
        next_live = tn < c.ntiles && live_of(mkn);
        if (next_live) {
          vn = __ldcs(reinterpret_cast<const uint4*>(c.data + tn * kTileBytes + lane * 16));
          if (lane == 0) hn = *reinterpret_cast<const uint2*>(c.data + tn * kTileBytes - 8);
          dn = __ldg(c.tile_seq + tn);
        }
        if (tn + nwarps < c.ntiles) mknn = mask_at(tn + nwarps);
      } else if (tn < c.ntiles) {
        vn = __ldcs(reinterpret_cast<const uint4*>(c.data + tn * kTileBytes + lane * 16));
        if (lane == 0) hn = *reinterpret_cast<const uint2*>(c.data + tn * kTileBytes - 8);
        dn = __ldg(c.tile_seq + tn);
        if (chain) mkn = mask_at(tn);
      }
      uint32_t hm = 0;
      if (!SP || cur_live) {  // (a dead tile of a sparse pass: only its zero hit-mask word)
      HSeg s;
      s.W[2] = v.x;
      s.W[3] = v.y;
      s.W[4] = v.z;
      s.W[5] = v.w;
      s.W[6] = 0;
      s.W[0] = __shfl_up_sync(0xffffffffu, v.z, 1);
      s.W[1] = __shfl_up_sync(0xffffffffu, v.w, 1);
      if (lane == 0) {
        s.W[0] = h.x;
        s.W[1] = h.y;
      }
      const int64_t b0 = (int64_t)t * kTileBytes + lane * 16;
      uint32_t vm = (d >> 31) ? 0xffffu : hvalid_walk<L>(c.off, c.m, c.total, d & 0x7fffffffu, b0);
      if (chain) {
        const uint32_t up = __shfl_up_sync(0xffffffffu, mk, 1);
        vm &= (mk << 1) | (((lane == 0 ? mk >> 16 : up) >> 15) & 1u);
      }
      if constexpr (PH && KIND == 1) {
        // hot grams in shared memory; the others go to this warp's queue
        // (ballot-compacted), drained 32 at a time with every lane probing
        // one position: the L2 probes of a whole tile then cost a few round
        // trips with full warps instead of one divergent round trip per T.
        // One position of every lane (v: the lane has one): branch-free, the
        // shared add and the queue stores are predicated, and shared
        // addresses are 32-bit from one base
        // (one slice only: launch_count_hot sends sliced sweeps, which need
        // tables above IG_HOT_SLICE_MB = 4 GiB, to the serial kernel)
        auto step = [&](uint64_t key, uint32_t T, bool v) {
          const uint32_t hh = (uint32_t)key * hmul + (uint32_t)(key >> 32) * 0x85EBCA77u;
          const uint32_t sl = hh >> lgnb_s;  // direct slot = 2 * hot_bucket + way bit
          // a predicated 8-byte load: lanes without a valid position add no
          // shared-memory wavefronts
          const uint64_t k0 = lds_u64_if(s_keys + sl * 8, v);
          const bool hot = v && k0 == key;
          red_shared_if(s_cnt + sl * 4, hot);
          if (hot) hm |= 1u << T;
          const bool cq = v && !hot;
          const uint32_t bal = __ballot_sync(0xffffffffu, cq);
          const uint32_t qi = (qtail + __popc(bal & lt_mask)) & (kHotQ - 1);
          st_shared_u64_if(s_qkey + qi * 8, key, cq);
          st_shared_u32_if(s_qpos + qi * 4, (kcur << 9) | (lane << 4) | T, cq);
          qtail += __popc(bal);
          if (qtail - qhead >= 32) {
            __syncwarp();
            drain(32u);
          }
        };
        bool dense_tile = true;
        if constexpr (SP) {
          // the most live positions any lane holds (hit chaining leaves few
          // on a sparse pass: c5's 6- to 8-gram passes keep ~10 % of the
          // tiles, its 5-gram pass ~9 % of the positions of the others)
          const uint32_t iters =
              sparse ? __reduce_max_sync(0xffffffffu, (uint32_t)__popc(vm)) : 16u;
          if (iters == 0) {
            dense_tile = false;  // a dead tile costs one reduction
          } else if (iters <= hw.sparse_iters) {
            // sparse tile: every lane walks its own live positions, so the
            // tile costs max-popcount steps instead of 16; the key comes out
            // of the window at a runtime offset (word selects + funnel shifts)
            dense_tile = false;
            uint32_t rem = vm;
#pragma unroll 1
            for (uint32_t it = 0; it < iters; ++it) {
              const uint32_t has = rem != 0;
              const uint32_t T = has ? (uint32_t)__ffs((int)rem) - 1u : 0u;
              rem &= rem - 1;
              const uint32_t o = T + 1, wi = o >> 2, sh = 8 * (o & 3);
              uint32_t x0 = (wi & 2) ? s.W[2] : s.W[0], x1 = (wi & 2) ? s.W[3] : s.W[1];
              uint32_t x2 = (wi & 2) ? s.W[4] : s.W[2], x3 = (wi & 2) ? s.W[5] : s.W[3];
              if (wi & 4) {
                x0 = s.W[4];
                x1 = s.W[5];
                x2 = 0;
                x3 = 0;
              }
              const uint32_t a0 = (wi & 1) ? x1 : x0, a1 = (wi & 1) ? x2 : x1,
                             a2 = (wi & 1) ? x3 : x2;
              const uint32_t klo = __funnelshift_r(a0, a1, sh), khi = __funnelshift_r(a1, a2, sh);
              const uint64_t key = (((uint64_t)__byte_perm(klo, 0, 0x0123) << 32) |
                                    (uint64_t)__byte_perm(khi, 0, 0x0123)) & hgram_mask<L>();
              step(key, T, has != 0);
            }
            __syncwarp();
            hm |= qhit[lane];
            qhit[lane] = 0;
          }
        }
        if (dense_tile) {
          // a runtime loop over 4 groups of 4 positions (the window words
          // rotate by one per group), so the drain code exists 4 times, not 16
          uint32_t q0 = s.W[0], q1 = s.W[1], q2 = s.W[2], q3 = s.W[3], q4 = s.W[4], q5 = s.W[5];
#pragma unroll 1
          for (int g = 0; g < 4; ++g) {
            hstatic_for<0, 4>([&](auto ic) {
              constexpr int I = decltype(ic)::value;
              constexpr int o = I + 1, wi = o / 4, sh = 8 * (o % 4);
              const uint32_t w0 = wi == 0 ? q0 : q1, w1 = wi == 0 ? q1 : q2, w2 = wi == 0 ? q2 : q3;
              const uint32_t klo = sh ? __funnelshift_r(w0, w1, sh) : w0;
              const uint32_t khi = sh ? __funnelshift_r(w1, w2, sh) : w1;
              const uint64_t key = (((uint64_t)__byte_perm(klo, 0, 0x0123) << 32) |
                                    (uint64_t)__byte_perm(khi, 0, 0x0123)) & hgram_mask<L>();
              const uint32_t T = 4 * g + I;
              step(key, T, ((vm >> T) & 1u) != 0);
            });
            q0 = q1;
            q1 = q2;
            q2 = q3;
            q3 = q4;
            q4 = q5;
            q5 = 0;
          }
          __syncwarp();
          hm |= qhit[lane];
          qhit[lane] = 0;
        }
      } else if (KIND == 0 && hw.direct) {
        // dense pass over a direct table (one slice), branch-free: one
        // predicated 8-byte load and compare, a predicated shared add for a
        // hot gram, a predicated RED for any other
        hstatic_for<0, 16>([&](auto tc) {
          constexpr int T = decltype(tc)::value;
          const bool v = ((vm >> T) & 1u) != 0;
          const uint64_t key = hkey8_at<T>(s) & hgram_mask<L>();
          const uint32_t hh = (uint32_t)key * hmul + (uint32_t)(key >> 32) * 0x85EBCA77u;
          const uint32_t sl = hh >> lgnb_s;
          const uint64_t k0 = lds_u64_if(s_keys + sl * 8, v);
          const bool hot = v && k0 == key;
          red_shared_if(s_cnt + sl * 4, hot);
          if (v && !hot) atomicAdd(cold + key, (CC)1);
        });
      } else if (KIND == 1 && TAB == 5 && hw.direct) {
        // the rank-bitmap (4-gram) pass over a direct table (one slice),
        // branch-free: the hot lookup as above; any other position loads its
        // 3-byte prefix's {bits, rank} pair (predicated), and a set bit is one
        // RED at rank * 256 + last byte.  The 16 positions' loads are
        // independent, so they overlap without a queue.
        hstatic_for<0, 16>([&](auto tc) {
          constexpr int T = decltype(tc)::value;
          const bool v = ((vm >> T) & 1u) != 0;
          const uint64_t key = hkey8_at<T>(s) & hgram_mask<L>();
          const uint32_t hh = (uint32_t)key * hmul + (uint32_t)(key >> 32) * 0x85EBCA77u;
          const uint32_t sl = hh >> lgnb_s;
          const uint64_t k0 = lds_u64_if(s_keys + sl * 8, v);
          const bool hot = v && k0 == key;
          red_shared_if(s_cnt + sl * 4, hot);
          const bool cq = v && !hot;
          const uint32_t pre = (uint32_t)(key >> 8);
          ulonglong2 e = make_ulonglong2(0, 0);
          if (cq) e = __ldg(reinterpret_cast<const ulonglong2*>(ptab) + (pre >> 6));
          const uint64_t bit = 1ull << (pre & 63);
          const bool hit = (e.x & bit) != 0;  // (e = 0 unless cq)
          if (hit) {
            const uint32_t p = (uint32_t)e.y + (uint32_t)__popcll(e.x & (bit - 1));
            atomicAdd(cold + ((uint64_t)p * 256 + (uint32_t)(key & 0xff)), (CC)1);
          }
          if (hot || hit) hm |= 1u << T;
        });
      } else
      hstatic_for<0, 16>([&](auto tc) {
        constexpr int T = decltype(tc)::value;
        if ((vm >> T) & 1u) {
          const uint64_t key = hkey8_at<T>(s) & hgram_mask<L>();
          const uint64_t sk = KIND == 1 ? key >> 8 : key;
          if (!sliced || (sk >= lo && sk < hi)) {
            const uint32_t b = hot_bucket(key, hw.lgnb, hmul);
            const ulonglong2 e = skeys[b];
            const uint32_t slot = e.x == key ? 2 * b : (e.y == key ? 2 * b + 1 : 0xffffffffu);
            if (slot != 0xffffffffu) {
              atomicAdd(scnt + slot, 1u);
              hm |= 1u << T;
            } else if constexpr (KIND == 0) {
              atomicAdd(cold + key, (CC)1);
            } else {
              uint32_t p;
              if constexpr (TAB == 3) p = hlookup_packed(ptab, ps.lgS, ps.ib, key >> 8);
              else if constexpr (TAB == 4) p = hlookup_wide(ptab, ps.lgS, key >> 8, ps.hmask);
              else p = hlookup_rank(ptab, (uint32_t)(key >> 8));
              if (p != 0xffffffffu) {
                atomicAdd(cold + ((uint64_t)p * 256 + (uint32_t)(key & 0xff)), (CC)1);
                hm |= 1u << T;
              }
            }
          }
        }
      });
      }
      if (KIND == 1 && ps.hit_out != nullptr) {
        uint16_t* w = ps.hit_out + t * 32 + lane;
        if (hw.first) __stcs(w, (uint16_t)hm);  // slice 0 writes every word
        else if (hm) *w = (uint16_t)(*w | hm);  // later slices add their bits
      }
      if (tn >= c.ntiles) break;
      t = tn;
      v = vn;
      h = hn;
      d = dn;
      mk = mkn;
      if (sparse) mkn = mknn;
      cur_live = next_live;
      ++kcur;
    }
  }
  if constexpr (PH && KIND == 1) {  // the warp's last probes: every tile is done
    __syncwarp();
    ++kcur;
    drain_resolve();
    while (qtail != qhead) {
      const uint32_t n = qtail - qhead < 32u ? qtail - qhead : 32u;
      drain_issue(n);
      drain_resolve();
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 2 * nb; i += blockDim.x) {
    const uint32_t n = scnt[i];
    if (n) atomicAdd(table + hw.ids[i], (CT)n);
  }
}

size_t hot_smem(uint32_t lgnb) { return ((size_t)1 << lgnb) * 24; }

bool hot_sweep_queued(const DevPrefixSet& ps, bool dense, uint32_t L, bool sliced) {
  static const bool off = getenv("IG_HOT_SERIAL") != nullptr || getenv("IG_HOT_TWOWAY") != nullptr;
  if (off || sliced) return false;
  if (dense) return true;  // the dense sweep's branch-free path reads a direct table too
  // the rank-bitmap (4-gram) pass: the serial kernel's branch-free path (the
  // queued sweep only with IG_HOT_Q5: slower)
  if (L == 4 && ps.rankbits) return true;
  return ps.packed != nullptr || ps.wide != nullptr;
}
static size_t hot_smem_q(uint32_t lgnb, int threads) {
  return hot_smem(lgnb) + (size_t)(threads / 32) * kHotQWarpBytes;
}

template <typename CT, typename CC>
void launch_count_hot(const DevCorpus& c, const DevPrefixSet& ps, bool dense, uint32_t L,
                      const HotSweep& hw, CT* table, CC* cold, int num_sms, cudaStream_t st) {
  if (c.ntiles <= c.tile0) return;
  auto go = [&](auto kern, const uint64_t* ptab, bool queued = false) {
    const int threads = 1024;
    const size_t smem = queued ? hot_smem_q(hw.lgnb, threads) : hot_smem(hw.lgnb);
    IGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 0;
    IGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem));
    const uint64_t want = ((c.ntiles - c.tile0) * 32 + threads - 1) / threads;
    const uint64_t capb = (uint64_t)num_sms * (per > 0 ? per : 1);
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min(want, capb));
    kern<<<blocks, threads, smem, st>>>(c, ps, ptab, hw, table, cold);
  };
  if (dense) {
    switch (L) {
      case 1: go(k_count_hot<0, 1, 0, CT, CC>, nullptr); break;
      case 2: go(k_count_hot<0, 2, 0, CT, CC>, nullptr); break;
      default: go(k_count_hot<0, 3, 0, CT, CC>, nullptr); break;
    }
    return;
  }
  // queued cold probes (ballot-compacted per warp, probed 32 at a time);
  // the one-position-at-a-time kernel stays behind IG_HOT_SERIAL=1
  static const bool serial_env = getenv("IG_HOT_SERIAL") != nullptr;
  static const bool q5 = getenv("IG_HOT_Q5") != nullptr;  // queued rank-bitmap pass (experiment)
  // the sparse variant (dead / sparse tiles, mask-gated corpus loads) is a
  // second kernel, so the dense sweep's loop stays inside the instruction
  // cache; only u32 tables (every chained pass of a < 2^32-count corpus)
  constexpr bool kSparseTypes = sizeof(CT) == 4 && sizeof(CC) == 4;
  // the queued sweep handles one slice and reads a direct table
  const bool serial = serial_env || hw.sliced || !hw.direct;
  const bool sp = ps.sparse && ps.hit_in != nullptr && kSparseTypes && !serial;
#define IGB_HOT_J(J)                                                                     \
  case J:                                                                                \
    if (J == 4 && ps.rankbits) {  /* one load per probe: the serial kernel is faster */ \
      if constexpr (J == 4) {                                                            \
        if (q5 && !serial) {                                                             \
          go(k_count_hot<1, 4, 5, CT, CC, true>, ps.rankbits, true);                     \
          break;                                                                         \
        }                                                                                \
      }                                                                                  \
      go(k_count_hot<1, J, 5, CT, CC>, ps.rankbits);                                     \
    } else if (ps.packed) {                                                              \
      if constexpr (kSparseTypes && J >= 5) {                                            \
        if (sp) {                                                                        \
          go(k_count_hot<1, J, 3, CT, CC, true, true>, ps.packed, true);                 \
          break;                                                                         \
        }                                                                                \
      }                                                                                  \
      if (serial) go(k_count_hot<1, J, 3, CT, CC>, ps.packed);                           \
      else go(k_count_hot<1, J, 3, CT, CC, true>, ps.packed, true);                      \
    } else {                                                                             \
      if constexpr (kSparseTypes && J >= 5) {                                            \
        if (sp) {                                                                        \
          go(k_count_hot<1, J, 4, CT, CC, true, true>, ps.wide, true);                   \
          break;                                                                         \
        }                                                                                \
      }                                                                                  \
      if (serial) go(k_count_hot<1, J, 4, CT, CC>, ps.wide);                             \
      else go(k_count_hot<1, J, 4, CT, CC, true>, ps.wide, true);                        \
    }                                                                                    \
    break;
  switch (L) {
    IGB_HOT_J(2) IGB_HOT_J(3) IGB_HOT_J(4) IGB_HOT_J(5) IGB_HOT_J(6) IGB_HOT_J(7) IGB_HOT_J(8)
    default: throw Error(IG_ECONFIG, "gram length above 8 is not supported");
  }
#undef IGB_HOT_J
}

template void launch_count_hot<uint32_t, uint32_t>(const DevCorpus&, const DevPrefixSet&, bool,
                                                   uint32_t, const HotSweep&, uint32_t*,
                                                   uint32_t*, int, cudaStream_t);
template void launch_count_hot<unsigned long long, uint32_t>(
    const DevCorpus&, const DevPrefixSet&, bool, uint32_t, const HotSweep&, unsigned long long*,
    uint32_t*, int, cudaStream_t);
template void launch_count_hot<unsigned long long, unsigned long long>(
    const DevCorpus&, const DevPrefixSet&, bool, uint32_t, const HotSweep&, unsigned long long*,
    unsigned long long*, int, cudaStream_t);

}  // namespace igb
