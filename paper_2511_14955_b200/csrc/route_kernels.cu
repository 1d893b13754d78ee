// route_kernels.cu — count-once passes as route-then-count (sm_100a).
//
// Reference semantics: counting.hpp:48-74 + counting.cpp:27-50 (a gram adds 1
// per sequence containing it), over the candidates of the dense pass
// (intergrams.cpp:79-100) or of an extension pass (intergrams.cpp:44-66).
//
// Design.  Per-sequence dedup needs a bitmap over the whole
// candidate space (2 MiB for the 2^24 dense 3-grams), far more than one SM's
// shared memory.  Every candidate occurrence is therefore computed once and
// routed to the owner of its id slice:
//   dense:     id' = (id * M) mod 2^24 (odd M: a bijection that spreads hot
//              grams), owner = id' >> 14, local = id' & 16383
//   extension: owner = hash(prefix) (<= 64 prefixes per owner), prefixes are
//              numbered owner by owner, local = (p - ostart[owner])*256 + last
// Work unit = <= 1 MiB of gram ends of one sequence.
//   1. k_route_count    per unit: owner histogram in smem -> cnt[o][u] (for
//                       extension passes an upper bound: no prefix lookup)
//   2. exclusive scan   cnt -> base: unit u owns [base[o][u], base[o][u+1]) of
//                       owner o's region (owner-major, no reservation atomics)
//   3. k_route_scatter  per unit, 8K positions at a time: drop repeats of the
//                       same gram inside the chunk (smem cache, before any
//                       lookup; an optimisation only, the consumer is exact),
//                       look the prefix up, counting-sort by owner in smem, copy
//                       each owner's run out coalesced; actual[o][u] = written
//   4. k_consume_once   CTA per (owner, block of sequences): a warp streams one
//                       sequence's runs (uint4 = 8 entries per load), dedups in
//                       a warp-private smem bitmap, counts first occurrences in
//                       smem u16 counters; the CTA flushes nonzero counters with
//                       coalesced REDs.
// Extension prefixes live in a host-built CHD perfect-hash table: a lookup is
// one 16-bit displacement load and one 8-byte slot load, with no divergence.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "ig_internal.cuh"
#include "kernels.h"

namespace igb {

namespace {

template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

template <int T>
__device__ __forceinline__ uint64_t key8(const uint32_t (&W)[7]) {
  constexpr int o = T + 1;
  constexpr int wi = o / 4, sh = 8 * (o % 4);
  uint32_t lo, hi;
  if constexpr (sh == 0) {
    lo = W[wi];
    hi = W[wi + 1];
  } else {
    lo = __funnelshift_r(W[wi], W[wi + 1], sh);
    hi = __funnelshift_r(W[wi + 1], W[wi + 2], sh);
  }
  return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | (uint64_t)__byte_perm(hi, 0, 0x0123);
}

template <int L>
__device__ __forceinline__ uint64_t gmask() {
  if constexpr (L >= 8) return ~0ull;
  else return (1ull << (8 * L)) - 1;
}

// CHD perfect-hash prefix set (host-built): bucket b = hash1(key) of nb,
// slot = range(s + d[b] * t) of nslots with (s, t) = hash2(key); every survivor
// owns exactly one slot.  Keys of <= 4 bytes (NARROW) hash with 32-bit
// multiplies (bijections of the key).  A slot packs the key with what the
// scatter needs, by prefix length (layout is a function of the pass):
//   <= 4 bytes   (key << 32) | owner << 16 | index in owner << 8
//      5 bytes   (key << 24) | v          v = owner << 6 | index in owner
//   6..7 bytes   (key << 8)  | index      owner recomputed from the key
// empty = ~0 (an impossible v / index).  A lookup is one u16 and one u64
// shared-memory load: no probing, no divergence.
struct MphfHash {
  uint32_t b, s, t;
};
template <bool NARROW>
__host__ __device__ __forceinline__ MphfHash mphf_hash(uint64_t key, uint32_t nb) {
  MphfHash h;
  if constexpr (NARROW) {
    const uint32_t k = (uint32_t)key;
    h.b = (uint32_t)(((uint64_t)(k * kNarrowMul1) * nb) >> 32);
    h.s = k * kNarrowMul2;
    h.t = (k * kNarrowMul3) | 1u;
  } else {
    const uint64_t x = key * kCuckooMul1;
    const uint64_t y = key * kCuckooMul2;
    h.b = (uint32_t)(((x >> 32) * (uint64_t)nb) >> 32);
    h.s = (uint32_t)(y >> 32);
    h.t = (uint32_t)y | 1u;
  }
  return h;
}

__host__ __device__ __forceinline__ uint32_t mphf_place(const MphfHash& h, uint32_t d,
                                                        uint32_t nslots) {
  return (uint32_t)(((uint64_t)(h.s + d * h.t) * nslots) >> 32);
}

// Returns the route base of a survivor prefix, (owner << 16) | (index in
// owner << 8), or 0xffffffff when the prefix is not a survivor.
template <int PLEN>
__device__ __forceinline__ uint32_t prefix_lookup_v(const uint64_t* slots, const uint16_t* disp,
                                                    uint32_t nb, uint32_t nslots, uint32_t lgno,
                                                    uint64_t key) {
  const MphfHash h = mphf_hash<(PLEN <= 4)>(key, nb);
  const uint32_t sl = mphf_place(h, disp[h.b], nslots);
  const uint64_t e = slots[sl];
  if constexpr (PLEN <= 4) {  // the base itself is stored
    const uint32_t v = (uint32_t)e;
    return ((uint32_t)(e >> 32) == (uint32_t)key) ? v : 0xffffffffu;  // empty: v = ~0
  } else if constexpr (PLEN == 5) {
    const uint32_t v = (uint32_t)e & 0xffffffu;
    return ((e >> 24) == key && v != 0xffffffu) ? (((v >> 6) << 16) | ((v & 63u) << 8))
                                                : 0xffffffffu;
  } else {
    const uint32_t idx = (uint32_t)e & 0xffu;
    return ((e >> 8) == key && idx != 0xffu) ? ((owner_hash(key, PLEN, lgno) << 16) | (idx << 8))
                                             : 0xffffffffu;
  }
}

constexpr int kRouteThreads = 1024;
constexpr int kChunk = kRouteThreads * 16;  // positions per scatter chunk
constexpr int kDedupSlots = 4096;

// The 16-byte segment at b0 plus its 8-byte halo (full warp, consecutive lanes).
__device__ __forceinline__ void seg_load(const uint8_t* __restrict__ data, int64_t b0, int lane,
                                         uint32_t (&W)[7]) {
  const uint4 v = __ldcs(reinterpret_cast<const uint4*>(data + b0));
  W[2] = v.x;
  W[3] = v.y;
  W[4] = v.z;
  W[5] = v.w;
  W[6] = 0;
  uint32_t h0 = __shfl_up_sync(0xffffffffu, v.z, 1);
  uint32_t h1 = __shfl_up_sync(0xffffffffu, v.w, 1);
  if (lane == 0) {
    const uint2 h = *reinterpret_cast<const uint2*>(data + b0 - 8);
    h0 = h.x;
    h1 = h.y;
  }
  W[0] = h0;
  W[1] = h1;
}

__device__ __forceinline__ uint32_t vmask(int64_t b0, int64_t lo, int64_t hi) {
  int64_t a = lo - b0, b = hi - b0;
  if (a < 0) a = 0;
  if (b > 16) b = 16;
  if (a >= b) return 0;
  return ((1u << b) - 1u) & ~((1u << a) - 1u);
}

// Dense: (owner << 16 | local) of a dense id via the odd-multiplier
// permutation (dense ids have <= 24 bits, so 32-bit arithmetic is exact).
__device__ __forceinline__ uint32_t dense_route(uint64_t id, const RouteParams& rp) {
  const uint32_t idp = ((uint32_t)id * (uint32_t)rp.mult) & (uint32_t)rp.cmask;
  return ((idp >> rp.lgl) << 16) | (idp & ((1u << rp.lgl) - 1));
}

// Count pass owner of the gram ending at T (no prefix lookup: an upper bound
// for extension passes, exact for the dense pass).
template <int KIND, int L, int T>
__device__ __forceinline__ uint32_t count_owner(const uint32_t (&W)[7], const RouteParams& rp) {
  const uint64_t key = key8<T>(W) & gmask<L>();
  if constexpr (KIND == 0) return dense_route(key, rp) >> 16;
  else return owner_hash(key >> 8, L - 1, rp.lgno);
}

// Scatter pass: (owner << 16 | local) of a gram key, or ~0 (prefix miss).
// Extension: the lookup yields (owner << 16 | index of the prefix inside its
// owner << 8), so the route is that | last byte, with no second lookup.
template <int KIND, int L>
__device__ __forceinline__ uint32_t scatter_route(uint64_t key, const RouteParams& rp,
                                                  const uint64_t* slots, const uint16_t* disp) {
  if constexpr (KIND == 0) {
    return dense_route(key, rp);
  } else {
    const uint32_t base =
        prefix_lookup_v<L - 1>(slots, disp, rp.nb, rp.nslots, rp.lgno, key >> 8);
    return base == 0xffffffffu ? base : base | (uint32_t)(key & 0xff);
  }
}

// Stages the perfect-hash prefix set (slots, then displacements) in smem
// (TAB == 1) or points at global memory.
template <int TAB>
__device__ __forceinline__ const uint64_t* stage_table(const RouteParams& rp, uint64_t* s_slots,
                                                       const uint16_t*& disp) {
  if constexpr (TAB == 1) {
    for (uint32_t i = threadIdx.x; i < rp.nslots; i += blockDim.x) s_slots[i] = rp.slots[i];
    uint16_t* s_disp = reinterpret_cast<uint16_t*>(s_slots + rp.nslots);
    for (uint32_t i = threadIdx.x; i < rp.nb; i += blockDim.x) s_disp[i] = rp.disp[i];
    __syncthreads();
    disp = s_disp;
    return s_slots;
  } else {
    disp = rp.disp;
    return rp.slots;
  }
}

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

}  // namespace

// ------------------------------------------------------------------ 1. count

template <int KIND, int L>
__global__ void __launch_bounds__(kRouteThreads) k_route_count(DevCorpus c, RouteView uv,
                                                               RouteParams rp,
                                                               uint32_t* __restrict__ cnt) {
  extern __shared__ uint4 smem4[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem4);
  const int lane = threadIdx.x & 31;
  for (uint32_t ui = blockIdx.x; ui < uv.nb; ui += gridDim.x) {
    const uint32_t u = uv.u0 + ui;
    for (uint32_t i = threadIdx.x; i < rp.NO; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const RouteUnit U = uv.units[u];
    const int64_t s0 = (int64_t)c.off[U.q];
    const int64_t lo = max((int64_t)U.b0, s0 + L - 1), hi = (int64_t)U.b1;
    const int64_t first = (int64_t)U.b0 & ~int64_t(15);
    const int64_t nseg = (hi - first + 15) >> 4;
    const int64_t nseg_r = (nseg + 31) & ~int64_t(31);  // whole warps
    for (int64_t sgi = threadIdx.x; sgi < nseg_r; sgi += blockDim.x) {
      const int64_t b0 = first + sgi * 16;
      uint32_t W[7];
      seg_load(c.data, b0, lane, W);
      const uint32_t vm = sgi < nseg ? vmask(b0, lo, hi) : 0u;
      static_for<0, 16>([&](auto tc) {
        constexpr int T = decltype(tc)::value;
        if ((vm >> T) & 1u) atomicAdd(hist + count_owner<KIND, L, T>(W, rp), 1u);
      });
    }
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < rp.NO; o += blockDim.x)
      cnt[(size_t)o * uv.nb + ui] = hist[o];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ 3. scatter

constexpr int kScatterThreads = 512;      // default scatter CTA
constexpr int kScatterThreadsBig = 768;   // smem-staged table: one CTA per SM
constexpr int kSChunk = kScatterThreads * 16;  // positions per chunk (default CTA)

// TAB: 0 dense (no table), 1 perfect-hash table staged in smem (768-thread
// CTA), 4 the same with a 512-thread CTA (smaller staging, bigger tables),
// 2 table in global memory.
template <int KIND, int L, int TAB, int NT, int DSLOTS>
__global__ void __launch_bounds__(NT) k_route_scatter(
    DevCorpus c, RouteView uv, RouteParams rp, const unsigned long long* __restrict__ base,
    uint32_t* __restrict__ actual, uint16_t* __restrict__ entries) {
  extern __shared__ uint4 smem4[];
  char* sp = reinterpret_cast<char*>(smem4);
  uint32_t* staging = reinterpret_cast<uint32_t*>(sp);  // kSChunk x (owner<<16|local)
  sp += (size_t)NT * 16 * 4;
  // dedup cache: DSLOTS * 8 bytes of gram keys.  Grams of <= 4 bytes are
  // kept as u32 (twice the slots); 5-byte grams as the low 40 - lg bits of a
  // bijection h = key * odd mod 2^40 whose top lg bits pick the slot (slot +
  // tag identify the key exactly, and a tag < 2^31 never equals the marker).
  using CK = std::conditional_t<(L <= 5), uint32_t, uint64_t>;
  constexpr int kSlots = DSLOTS * (int)(8 / sizeof(CK));
  constexpr CK kEmpty = (CK)~(CK)0;
  CK* cache = reinterpret_cast<CK*>(sp);
  sp += (size_t)DSLOTS * 8;
  unsigned long long* res = reinterpret_cast<unsigned long long*>(sp);  // NO
  sp += align16((size_t)rp.NO * 8);
  uint32_t* lhist = reinterpret_cast<uint32_t*>(sp);  // NO
  sp += align16((size_t)rp.NO * 4);
  // copy-out delta of each owner: global index of its staging slot 0
  unsigned long long* delta = reinterpret_cast<unsigned long long*>(sp);  // NO
  sp += align16((size_t)rp.NO * 8);
  const bool nextc = rp.next_lgno >= 0;
  const uint32_t nno = nextc ? (1u << rp.next_lgno) : 0u;
  uint32_t* nhist = reinterpret_cast<uint32_t*>(sp);  // next pass's owner histogram
  sp += align16((size_t)nno * 4);
  uint64_t* s_slots = reinterpret_cast<uint64_t*>(sp);
  __shared__ uint32_t s_total;
  using BlockScan = cub::BlockScan<uint32_t, NT>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  const uint16_t* disp = nullptr;
  const uint64_t* slots = KIND == 1 ? stage_table<(TAB == 1 || TAB == 4) ? 1 : 2>(rp, s_slots, disp) : nullptr;
  const bool dedup = rp.dedup;
  const int lane = threadIdx.x & 31;
  const uint32_t s_cache = smem_u32(cache), s_lhist = smem_u32(lhist), s_nhist = smem_u32(nhist),
                 s_staging = smem_u32(staging);
  for (uint32_t ui = blockIdx.x; ui < uv.nb; ui += gridDim.x) {
    const uint32_t u = uv.u0 + ui;
    const RouteUnit U = uv.units[u];
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < rp.NO; o += blockDim.x) res[o] = base[(size_t)o * uv.nb + ui];
    for (uint32_t o = threadIdx.x; o < nno; o += blockDim.x) nhist[o] = 0;
    const int64_t s0 = (int64_t)c.off[U.q];
    const int64_t lo = max((int64_t)U.b0, s0 + L - 1), hi = (int64_t)U.b1;
    const int64_t first = (int64_t)U.b0 & ~int64_t(15);
    const int64_t nseg = (hi - first + 15) >> 4;
    const bool next_in_seq = nextc && hi < (int64_t)c.off[U.q + 1];
    // the dedup cache lives for the whole unit: every chunk of a unit belongs to
    // the same sequence, so a gram seen anywhere earlier in it adds nothing
    for (uint32_t i = threadIdx.x; i < kSlots; i += blockDim.x) cache[i] = kEmpty;
    for (uint32_t i = threadIdx.x; i < rp.NO; i += blockDim.x) lhist[i] = 0;
    // four barriers per chunk: the scan phase also turns counts into bases,
    // copy-out deltas and advanced cursors (each owner belongs to one
    // thread), and the copy-out phase zeroes the histogram for the next chunk
    for (int64_t cs = 0; cs < nseg; cs += NT) {
      __syncthreads();
      const int64_t sgi = cs + threadIdx.x;
      const int64_t b0 = first + sgi * 16;
      uint32_t W[7] = {0, 0, 0, 0, 0, 0, 0};
      if (cs + (int64_t)(threadIdx.x & ~31u) < nseg) seg_load(c.data, b0, lane, W);  // warp-uniform
      const uint32_t vm = sgi < nseg ? vmask(b0, lo, hi) : 0u;
      // the next pass's gram ending at b0+T+1 is in this unit iff T < lim
      const int64_t lim64 = hi - b0 - 1;
      const int32_t lim = (int32_t)(lim64 < 0 ? -1 : lim64 > 16 ? 16 : lim64);
      uint32_t r[16];
      static_for<0, 16>([&](auto tc) {
        constexpr int T = decltype(tc)::value;
        // branch-free: a warp almost never has all 32 lanes on the cheap side
        // of a test, so every step is computed and the results predicated
        const bool valid = (vm >> T) & 1u;
        const uint64_t key = key8<T>(W) & gmask<L>();
        // a gram already routed from this unit adds nothing (count-once):
        // drop it.  Races only cost a duplicate.
        constexpr int kLgSlots = kSlots == 16384 ? 14 : kSlots == 8192 ? 13 : kSlots == 4096 ? 12 : 11;
        uint32_t slot;
        CK tag;
        if constexpr (L == 5) {
          const uint64_t h = (key * 0x9E3779B97F4A7C15ull) & ((1ull << 40) - 1);
          slot = (uint32_t)(h >> (40 - kLgSlots));
          tag = (CK)(h & ((1ull << (40 - kLgSlots)) - 1));
        } else if constexpr (L <= 4) {
          slot = ((uint32_t)key * 0x9E3779B1u) >> (32 - kLgSlots);
          tag = (CK)key;
        } else {
          slot = (((uint32_t)key ^ ((uint32_t)(key >> 32) * 0x85EBCA6Bu)) * 0x9E3779B1u) >> (32 - kLgSlots);
          tag = (CK)key;
        }
        const CK seen = cache[slot];
        const bool fresh = valid && (!dedup || (L != 5 && tag == kEmpty) || seen != tag);  // kEmpty: marker
        if constexpr (sizeof(CK) == 8) st_shared_u64_at(fresh, s_cache + slot * 8, key);
        else st_shared_u32_at(fresh, s_cache + slot * 4, (uint32_t)tag);
        uint32_t v = scatter_route<KIND, L>(key, rp, slots, disp);
        v = fresh ? v : 0xffffffffu;
        red_inc_shared_at(v != 0xffffffffu, s_lhist + (v >> 16) * 4);
        if (nextc) {
          // the next pass's gram ending at b0+T+1 has this gram as its prefix;
          // it can be routed only if this gram is a candidate: a lookup hit,
          // or a repeat (counted conservatively: the count is an upper bound)
          const bool cand = valid && (KIND == 0 || v != 0xffffffffu || !fresh);
          const uint32_t no = owner_hash(key, L, rp.next_lgno);
          red_inc_shared_at(cand && T < lim, s_nhist + no * 4);
          // a valid position with T >= lim is the unit's last: its successor is
          // the first position of unit u+1 when that unit is in this sequence
          if (cand && T >= lim && next_in_seq)
            atomicAdd(rp.next_cnt + (size_t)no * uv.nunits + u + 1, 1u);
        }
        r[T] = v;
      });
      __syncthreads();
      {  // exclusive scan of lhist; each thread owns a contiguous run of owners
        const uint32_t per = (rp.NO + NT - 1) / NT;
        const uint32_t a = threadIdx.x * per, e = min(rp.NO, a + per);
        uint32_t sum = 0;
        for (uint32_t o = a; o < e; ++o) sum += lhist[o];
        uint32_t ex, tot;
        BlockScan(scan_tmp).ExclusiveSum(sum, ex, tot);
        for (uint32_t o = a; o < e; ++o) {
          const uint32_t cnt = lhist[o];
          lhist[o] = ex;               // placement cursor (staging base of o)
          delta[o] = res[o] - ex;      // staging slot i of o -> entries[delta + i]
          res[o] += cnt;               // o's global cursor after this chunk
          ex += cnt;
        }
        if (threadIdx.x == 0) s_total = tot;
      }
      __syncthreads();
      static_for<0, 16>([&](auto tc) {
        constexpr int T = decltype(tc)::value;
        const bool h = r[T] != 0xffffffffu;
        const uint32_t at = atom_inc_shared_at(h, s_lhist + (r[T] >> 16) * 4);
        st_shared_u32_at(h, s_staging + at * 4, r[T]);
      });
      __syncthreads();
      const uint32_t total = s_total;
      for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
        const uint32_t e = staging[i];
        const uint32_t o = e >> 16;
        entries[delta[o] + i] = (uint16_t)(e & 0xffffu);
      }
      for (uint32_t i = threadIdx.x; i < rp.NO; i += blockDim.x) lhist[i] = 0;
    }
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < rp.NO; o += blockDim.x)
      actual[(size_t)o * uv.nb + ui] = (uint32_t)(res[o] - base[(size_t)o * uv.nb + ui]);
    for (uint32_t o = threadIdx.x; o < nno; o += blockDim.x)
      if (nhist[o]) atomicAdd(rp.next_cnt + (size_t)o * uv.nunits + u, nhist[o]);
  }
}

// ------------------------------------------------------------------ 4. consume

constexpr int kConsumeThreads = 512;
constexpr int kConsumeWarps = kConsumeThreads / 32;

// Words of a warp's bitmap / packing region: the bitmap of ipo ids, at least
// 16 rounds x 32 packed entries, a multiple of 4 words.
__host__ __device__ inline uint32_t consume_region_words(uint32_t ipo) {
  const uint32_t w = ((ipo + 31) / 32 + 3) & ~3u;
  return w < 512u ? 512u : w;
}

__device__ __forceinline__ void consume_entry(uint32_t local, uint32_t* bm, uint32_t* cnt) {
  const uint32_t bit = 1u << (local & 31);
  uint32_t* w = bm + (local >> 5);
  if (!(*(volatile uint32_t*)w & bit)) {
    if (!(atomicOr(w, bit) & bit)) atomicAdd(cnt + (local >> 1), 1u << (16 * (local & 1)));
  }
}

// One sequence's runs for owner o through the warp's bitmap (then cleared).
__device__ __forceinline__ void consume_bitmap(const RouteView& uv, uint32_t o, uint64_t q,
                                               const unsigned long long* __restrict__ base,
                                               const uint32_t* __restrict__ actual,
                                               const uint16_t* __restrict__ entries,
                                               uint32_t* bm, uint32_t bmw4, uint32_t* cnt,
                                               int lane) {
  const uint32_t u0 = uv.unit_first[q], u1 = uv.unit_first[q + 1];
  for (uint32_t u = u0; u < u1; ++u) {
    const size_t ix = (size_t)o * uv.nb + (u - uv.u0);
    const uint64_t e0 = base[ix], e1 = e0 + actual[ix];
    // uint4-aligned body: 8 entries per lane per load
    const uint64_t a0 = (e0 + 7) & ~7ull, a1 = e1 & ~7ull;
    if (a0 >= a1) {
      for (uint64_t e = e0 + lane; e < e1; e += 32) consume_entry(entries[e], bm, cnt);
    } else {
      if (e0 + lane < a0) consume_entry(entries[e0 + lane], bm, cnt);
      if (a1 + lane < e1) consume_entry(entries[a1 + lane], bm, cnt);
      const uint4* v4 = reinterpret_cast<const uint4*>(entries + a0);
      const uint64_t nv = (a1 - a0) >> 3;
      for (uint64_t i = lane; i < nv; i += 32) {
        const uint4 v = __ldcs(v4 + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          consume_entry(w[k] & 0xffffu, bm, cnt);
          consume_entry(w[k] >> 16, bm, cnt);
        }
      }
    }
  }
  __syncwarp();
  for (uint32_t i = lane; i < bmw4 / 4; i += 32) reinterpret_cast<uint4*>(bm)[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();
}

// Consume: CTA per (owner, block of sequences).  A warp walks a contiguous
// range of the block's sequences 16 at a time: lanes fetch the 16 sequences'
// run metadata in parallel; runs of more than 32 entries (and sequences of
// several units) go through the warp's bitmap one sequence at a time; short
// runs are packed whole into rounds of 32 lanes and deduplicated with
// MATCH.ANY on (run, local) -- no bitmap to set or clear, which is what
// dominates when sequences are a few KiB.  The bitmap region doubles as the
// packing buffer (it is zero again afterwards).
template <typename CT>
__global__ void __launch_bounds__(kConsumeThreads) k_consume_once(
    RouteView uv, RouteParams rp, uint32_t seq_block, uint32_t nblocks,
    const unsigned long long* __restrict__ base, const uint32_t* __restrict__ actual,
    const uint16_t* __restrict__ entries, CT* __restrict__ table,
    const uint32_t* __restrict__ owner_order, uint32_t* __restrict__ work) {
  extern __shared__ uint4 smem4[];
  const uint32_t ipo = 1u << rp.lgl;                   // ids per owner
  const uint32_t cntw = (uint32_t)(align16((size_t)(ipo + 1) / 2 * 4) / 4);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem4);  // u16 pairs
  uint32_t* bms = cnt + cntw;                          // kConsumeWarps x bmw4 words
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t bmw4 = consume_region_words(ipo);
  uint32_t* bm = bms + warp * bmw4;
  const uint32_t nitems = rp.NO * nblocks;
  for (uint32_t i = threadIdx.x; i < bmw4 * kConsumeWarps; i += blockDim.x) bms[i] = 0;
  // items are claimed dynamically, owners heaviest first (Zipf corpora route
  // most entries to a few owners; a static split leaves SMs idle at the end)
  __shared__ uint32_t s_item;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= nitems) break;
    const uint32_t o = owner_order[item / nblocks], b = item % nblocks;
    for (uint32_t i = threadIdx.x; i < cntw; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const uint64_t q0 = uv.q0 + (uint64_t)b * seq_block;
    const uint64_t q1 = min((uint64_t)uv.q1, q0 + seq_block);
    const uint64_t per_w = (q1 - q0 + kConsumeWarps - 1) / kConsumeWarps;
    const uint64_t wq0 = min(q1, q0 + warp * per_w), wq1 = min(q1, wq0 + per_w);
    for (uint64_t qw = wq0; qw < wq1; qw += 16) {
      const uint64_t q = qw + (lane & 15);
      uint64_t e0 = 0;
      uint32_t len = 0;
      bool big = false;
      if (lane < 16 && q < wq1) {
        const uint32_t ua = uv.unit_first[q], ub = uv.unit_first[q + 1];
        if (ub == ua + 1) {
          const size_t ix = (size_t)o * uv.nb + (ua - uv.u0);
          e0 = base[ix];
          len = actual[ix];
          big = len > 32;
        } else {
          big = ub > ua + 1;  // zero units: a short sequence (k_once_short)
        }
      }
      uint32_t bigm = __ballot_sync(0xffffffffu, big);
      while (bigm) {
        const int l = __ffs(bigm) - 1;
        bigm &= bigm - 1;
        consume_bitmap(uv, o, qw + l, base, actual, entries, bm, bmw4, cnt, lane);
      }
      // greedy packing of whole short runs into rounds of 32 entries
      const uint32_t mylen = (lane < 16 && !big) ? len : 0u;
      uint32_t mypos = 0, round = 0, off = 0;
      for (int i = 0; i < 16; ++i) {
        const uint32_t l = __shfl_sync(0xffffffffu, mylen, i);
        if (l == 0) continue;
        if (off + l > 32) {
          ++round;
          off = 0;
        }
        if (lane == i) mypos = round * 32 + off;
        off += l;
      }
      const uint32_t nr = off ? round + 1 : 0;
      if (!nr) continue;
      for (uint32_t r = 0; r < nr; ++r) bm[r * 32 + lane] = 0xffffffffu;
      __syncwarp();
      for (uint32_t t2 = 0; t2 < mylen; ++t2)
        bm[mypos + t2] = ((uint32_t)lane << 16) | entries[e0 + t2];
      __syncwarp();
      for (uint32_t r = 0; r < nr; ++r) {
        const uint32_t v = bm[r * 32 + lane];
        const uint32_t grp = __match_any_sync(0xffffffffu, v);
        if (v != 0xffffffffu && (__ffs(grp) - 1) == lane) {
          const uint32_t local = v & 0xffffu;
          atomicAdd(cnt + (local >> 1), 1u << (16 * (local & 1)));
        }
      }
      __syncwarp();
      for (uint32_t r = 0; r < nr; ++r) bm[r * 32 + lane] = 0u;
      __syncwarp();
    }
    __syncthreads();
    // owner o's ids start at o << lgl (dense, permuted) or ostart[o]*256 (extension)
    CT* dst = table + (rp.ext ? (size_t)rp.ostart[o] * 256 : ((size_t)o << rp.lgl));
    const uint32_t lim = rp.ext ? (rp.ostart[o + 1] - rp.ostart[o]) * 256 : ipo;
    for (uint32_t i = threadIdx.x; i < (lim + 1) / 2; i += blockDim.x) {
      const uint32_t v = cnt[i];
      if (v & 0xffffu) atomicAdd(dst + 2 * i, (CT)(v & 0xffffu));
      if ((v >> 16) && 2 * i + 1 < lim) atomicAdd(dst + 2 * i + 1, (CT)(v >> 16));
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ 5. short sequences

// Count-once over short sequences (the route path's per-unit and
// per-(owner, sequence) costs do not amortise over a few hundred bytes): a
// group of G threads (a warp, or a whole CTA) takes one sequence of <= LMAX
// gram ends, dedups its candidate table indices exactly in a shared-memory
// hash set sized to the sequence, and adds 1 per distinct index to the pass
// table.  Table indices are the route path's (dense: the permuted id;
// extension: (ostart[owner] + index in owner) * 256 + last byte), so both
// paths count into one table.
constexpr int kShortThreads = 512;
static size_t table_bytes(const RouteParams& rp);

template <int KIND, int L, int TAB, int G, int LMAX, typename CT>
__global__ void __launch_bounds__(kShortThreads) k_once_short(
    DevCorpus c, RouteParams rp, const uint32_t* __restrict__ seqs, uint32_t nseqs,
    CT* __restrict__ table) {
  extern __shared__ uint4 smem4[];
  constexpr int NG = kShortThreads / G;  // groups per CTA
  constexpr int HS = 2 * LMAX;           // hash slots per group (power of two)
  uint32_t* hs_all = reinterpret_cast<uint32_t*>(smem4);
  uint32_t* hs = hs_all + (threadIdx.x / G) * HS;
  uint64_t* s_slots = reinterpret_cast<uint64_t*>(hs_all + NG * HS);
  const uint16_t* disp = nullptr;
  const uint64_t* slots = KIND == 1 ? stage_table<TAB>(rp, s_slots, disp) : nullptr;
  const uint32_t gl = threadIdx.x % G;
  const uint32_t ngroups = gridDim.x * NG;
  auto group_sync = [] {
    if constexpr (G == 32) __syncwarp();
    else __syncthreads();
  };
  for (uint32_t i = blockIdx.x * NG + threadIdx.x / G; i < nseqs; i += ngroups) {
    const uint32_t q = seqs[i];
    const uint64_t s0 = c.off[q], s1 = c.off[q + 1];
    const int64_t npos = (int64_t)(s1 - s0) - (L - 1);  // gram ends (group-uniform)
    if (npos <= 0) continue;
    uint32_t lg = 4;
    while ((1 << lg) < 2 * npos) ++lg;
    const uint32_t mask = (1u << lg) - 1;
    for (uint32_t j = gl; j <= mask; j += G) hs[j] = 0xffffffffu;
    group_sync();
    // each thread: a contiguous run of gram ends, key rolled byte by byte
    const uint32_t per = (uint32_t)((npos + G - 1) / G);
    const int64_t p0 = (int64_t)gl * per;
    const int64_t p1 = p0 + per < npos ? p0 + per : npos;
    if (p0 < p1) {
      const uint8_t* d = c.data + s0;
      uint64_t key = 0;
      for (int b = 0; b < L - 1; ++b) key = (key << 8) | d[p0 + b];
      for (int64_t p = p0; p < p1; ++p) {
        key = ((key << 8) | d[p + L - 1]) & gmask<L>();
        uint32_t tidx;
        if constexpr (KIND == 0) {
          const uint32_t r = dense_route(key, rp);
          tidx = ((r >> 16) << rp.lgl) | (r & 0xffffu);
        } else {
          const uint32_t base =
              prefix_lookup_v<L - 1>(slots, disp, rp.nb, rp.nslots, rp.lgno, key >> 8);
          if (base == 0xffffffffu) continue;
          tidx = (rp.ostart[base >> 16] + ((base >> 8) & 63u)) * 256u + (uint32_t)(key & 0xff);
        }
        uint32_t h = (tidx * 0x9E3779B1u) >> (32 - lg);
        for (;;) {
          const uint32_t old = atomicCAS(hs + h, 0xffffffffu, tidx);
          if (old == 0xffffffffu) {
            atomicAdd(table + tidx, (CT)1);
            break;
          }
          if (old == tidx) break;
          h = (h + 1) & mask;
        }
      }
    }
    group_sync();
  }
}

template <int KIND, int L, int TAB, int G, int LMAX, typename CT>
static void launch_short_t(const DevCorpus& c, const RouteParams& rp, const uint32_t* seqs,
                           uint32_t n, CT* table, int num_sms, cudaStream_t st) {
  if (!n) return;
  constexpr int NG = kShortThreads / G;
  const size_t smem = (size_t)NG * 2 * LMAX * 4 + (TAB == 1 ? table_bytes(rp) : 0);
  auto k = k_once_short<KIND, L, TAB, G, LMAX, CT>;
  IGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  IGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kShortThreads, smem));
  if (per < 1) throw Error(IG_EINTERNAL, "short-sequence count does not fit in shared memory");
  const uint64_t want = (n + NG - 1) / NG;
  const unsigned grid = (unsigned)std::min<uint64_t>(want, (uint64_t)num_sms * per);
  k<<<grid, kShortThreads, smem, st>>>(c, rp, seqs, n, table);
}

template <int KIND, int L, typename CT>
static void launch_short_l(const DevCorpus& c, const RouteParams& rp, const uint32_t* sw,
                           uint32_t nw, const uint32_t* sc, uint32_t nc, CT* table, int num_sms,
                           cudaStream_t st) {
  if constexpr (KIND == 0) {
    launch_short_t<0, L, 0, 32, kShortWarpLen, CT>(c, rp, sw, nw, table, num_sms, st);
    launch_short_t<0, L, 0, kShortThreads, kShortCtaLen, CT>(c, rp, sc, nc, table, num_sms, st);
  } else {
    // the perfect-hash table in smem next to the hash sets when it fits
    const bool fits = (size_t)2 * kShortCtaLen * 4 + table_bytes(rp) <= kMaxOnceSmem &&
                      (size_t)(kShortThreads / 32) * 2 * kShortWarpLen * 4 + table_bytes(rp) <=
                          kMaxOnceSmem;
    if (fits) {
      launch_short_t<1, L, 1, 32, kShortWarpLen, CT>(c, rp, sw, nw, table, num_sms, st);
      launch_short_t<1, L, 1, kShortThreads, kShortCtaLen, CT>(c, rp, sc, nc, table, num_sms, st);
    } else {
      launch_short_t<1, L, 2, 32, kShortWarpLen, CT>(c, rp, sw, nw, table, num_sms, st);
      launch_short_t<1, L, 2, kShortThreads, kShortCtaLen, CT>(c, rp, sc, nc, table, num_sms, st);
    }
  }
}

template <typename CT>
void count_once_short(int kind, uint32_t L, const DevCorpus& c, const RouteParams& rp,
                      const uint32_t* sw, uint32_t nw, const uint32_t* sc, uint32_t nc, CT* table,
                      int num_sms, cudaStream_t st) {
  if (!nw && !nc) return;
  if (kind == 0) {
    switch (L) {
      case 1: launch_short_l<0, 1, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      case 2: launch_short_l<0, 2, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      default: launch_short_l<0, 3, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
    }
  } else {
    switch (L) {
      case 2: launch_short_l<1, 2, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      case 3: launch_short_l<1, 3, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      case 4: launch_short_l<1, 4, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      case 5: launch_short_l<1, 5, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      case 6: launch_short_l<1, 6, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      case 7: launch_short_l<1, 7, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      case 8: launch_short_l<1, 8, CT>(c, rp, sw, nw, sc, nc, table, num_sms, st); break;
      default: throw Error(IG_ECONFIG, "gram length above 8 is not supported");
    }
  }
  IGB_CUDA(cudaGetLastError());
}

template void count_once_short<uint32_t>(int, uint32_t, const DevCorpus&, const RouteParams&,
                                         const uint32_t*, uint32_t, const uint32_t*, uint32_t,
                                         uint32_t*, int, cudaStream_t);
template void count_once_short<unsigned long long>(int, uint32_t, const DevCorpus&,
                                                   const RouteParams&, const uint32_t*, uint32_t,
                                                   const uint32_t*, uint32_t,
                                                   unsigned long long*, int, cudaStream_t);

// Routed entries per owner (one CTA per owner row of `actual`).
__global__ void k_owner_totals(const uint32_t* __restrict__ actual, uint32_t nb,
                               uint32_t* __restrict__ tot) {
  uint64_t t = 0;
  const uint32_t* row = actual + (size_t)blockIdx.x * nb;
  for (uint32_t u = threadIdx.x; u < nb; u += blockDim.x) t += row[u];
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __shared__ uint64_t ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) s += ws[w];
    tot[blockIdx.x] = (uint32_t)(s < 0xfffffffeull ? s : 0xfffffffeull);
  }
}

// Owners heaviest first (one CTA, block radix sort on ~total).  work[0] = 0
// (the item counter).
constexpr int kOrderThreads = 1024, kOrderItems = 8;  // <= 8192 owners
// Owners in index order (the consume fallback for > kOrderThreads *
// kOrderItems owners or IG_CONSUME_NO_ORDER) and a zeroed item counter.
__global__ void k_identity_order(uint32_t* __restrict__ ord, uint32_t n,
                                 uint32_t* __restrict__ work) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ord[i] = i;
  if (i == 0) work[0] = 0;
}

__global__ void __launch_bounds__(kOrderThreads) k_owner_order(const uint32_t* __restrict__ tot,
                                                                uint32_t NO,
                                                                uint32_t* __restrict__ order,
                                                                uint32_t* __restrict__ work) {
  using Sort = cub::BlockRadixSort<uint32_t, kOrderThreads, kOrderItems, uint32_t>;
  __shared__ typename Sort::TempStorage tmp;
  uint32_t keys[kOrderItems], vals[kOrderItems];
#pragma unroll
  for (int i = 0; i < kOrderItems; ++i) {
    const uint32_t o = threadIdx.x * kOrderItems + i;
    keys[i] = o < NO ? ~tot[o] : 0xffffffffu;
    vals[i] = o;
  }
  Sort(tmp).Sort(keys, vals);
#pragma unroll
  for (int i = 0; i < kOrderItems; ++i) {
    const uint32_t r = threadIdx.x * kOrderItems + i;
    if (r < NO) order[r] = vals[i];
  }
  if (threadIdx.x == 0) work[0] = 0;
}

// ------------------------------------------------------------------ direct

// Count-once over a small alphabet.  When the corpus uses
// A <= 16 distinct bytes, an extension pass has at most K' * A candidates
// that can occur (prefix ordinal p, rank r of the last byte in the alphabet).
// When that fits a shared-memory bitmap, a CTA takes one whole sequence at a
// time: every position's candidate bit is set (test first, then an atomic OR),
// and at the end of the sequence each set bit adds 1 to compact[p * A + r]
// and is cleared.  No routing, no dedup cache, no consume pass.
// Gram ends [lo, hi) of a direct work item: part `part` of `nparts` equal
// byte ranges of sequence q (the first part starts at the sequence's first
// complete gram).
__device__ __forceinline__ void direct_part(const DevCorpus& c, const DirectItem& it, uint32_t L,
                                            int64_t& lo, int64_t& hi) {
  const int64_t s0 = (int64_t)c.off[it.q], s1 = (int64_t)c.off[it.q + 1];
  const int64_t len = s1 - s0;
  const int64_t a = s0 + (int64_t)((__int128)len * it.part / it.nparts);
  hi = s0 + (int64_t)((__int128)len * (it.part + 1) / it.nparts);
  lo = a > s0 + (int64_t)L - 1 ? a : s0 + (int64_t)L - 1;
  if (lo > hi) lo = hi;
}

// End of a work item: every set bit of the CTA bitmap counts one sequence.
// A part of a split sequence ORs its bits into the sequence's global bitmap
// instead; the last of its parts to arrive (threadfence-reduction order)
// counts the union and leaves the slot zeroed.
__device__ __forceinline__ void direct_flush(uint32_t* bm, uint32_t nwords, const DirectItem& it,
                                             const DirectWork& w, uint32_t* compact,
                                             uint32_t* s_last) {
  __syncthreads();
  if (it.nparts == 1) {
    for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) {
      uint32_t x = bm[i];
      if (x) {
        bm[i] = 0;
        do {
          atomicAdd(compact + i * 32 + (__ffs(x) - 1), 1u);
          x &= x - 1;
        } while (x);
      }
    }
  } else {
    uint32_t* g = w.gbm + (size_t)it.slot * nwords;
    for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) {
      const uint32_t x = bm[i];
      if (x) {
        bm[i] = 0;
        atomicOr(g + i, x);
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) *s_last = atomicAdd(w.done + it.slot, 1u) == it.nparts - 1;
    __syncthreads();
    if (*s_last) {
      __threadfence();
      for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) {
        uint32_t x = __ldcg(g + i);
        if (x) {
          g[i] = 0;
          do {
            atomicAdd(compact + i * 32 + (__ffs(x) - 1), 1u);
            x &= x - 1;
          } while (x);
        }
      }
    }
  }
  __syncthreads();
}

constexpr int kDirectThreads = 1024;

template <int L>
__global__ void __launch_bounds__(kDirectThreads, 1) k_once_direct(
    DevCorpus c, RouteParams rp, DirectWork w, const uint8_t* __restrict__ arank, uint32_t A,
    uint32_t nwords, uint32_t* __restrict__ compact) {
  extern __shared__ uint4 smem4[];
  char* sp = reinterpret_cast<char*>(smem4);
  uint32_t* bm = reinterpret_cast<uint32_t*>(sp);
  sp += align16((size_t)nwords * 4);
  uint32_t* s_ostart = reinterpret_cast<uint32_t*>(sp);
  sp += align16((size_t)rp.NO * 4);
  uint8_t* s_arank = reinterpret_cast<uint8_t*>(sp);
  sp += 256;
  uint64_t* s_slots = reinterpret_cast<uint64_t*>(sp);
  for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) bm[i] = 0;
  for (uint32_t i = threadIdx.x; i < rp.NO; i += blockDim.x) s_ostart[i] = rp.ostart[i];
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) s_arank[i] = arank[i];
  const uint16_t* disp = nullptr;
  const uint64_t* slots = stage_table<1>(rp, s_slots, disp);  // ends with a barrier
  const int lane = threadIdx.x & 31;
  __shared__ uint32_t s_last;
  for (uint32_t qi = blockIdx.x; qi < w.nitems; qi += gridDim.x) {
    const DirectItem it = w.items[qi];
    int64_t lo, hi;
    direct_part(c, it, L, lo, hi);
    const int64_t first = (lo - (L - 1)) & ~int64_t(15);
    const int64_t nseg = (hi - first + 15) >> 4;
    const int64_t nseg_r = (nseg + 31) & ~int64_t(31);  // whole warps (seg_load shuffles)
    for (int64_t sgi = threadIdx.x; sgi < nseg_r; sgi += blockDim.x) {
      const int64_t b0 = first + sgi * 16;
      uint32_t W[7];
      seg_load(c.data, b0, lane, W);
      const uint32_t vm = sgi < nseg ? vmask(b0, lo, hi) : 0u;
      static_for<0, 16>([&](auto tc) {
        constexpr int T = decltype(tc)::value;
        if ((vm >> T) & 1u) {
          const uint64_t key = key8<T>(W) & gmask<L>();
          const uint32_t v = scatter_route<1, L>(key, rp, slots, disp);
          if (v != 0xffffffffu) {
            const uint32_t id = (s_ostart[v >> 16] + ((v >> 8) & 0xffu)) * A + s_arank[v & 0xffu];
            uint32_t* w = bm + (id >> 5);
            const uint32_t bit = 1u << (id & 31);
            if (!(*(volatile uint32_t*)w & bit)) atomicOr(w, bit);
          }
        }
      });
    }
    direct_flush(bm, nwords, it, w, compact, &s_last);
  }
}

// The same with the prefix looked up in a direct table (alphabet of <= 16
// bytes, `bits` per rank, bits * (L - 1) <= 16): the 24 window bytes of a lane
// are translated to ranks once, the rank-packed prefix rolls from position to
// position, and lut[prefix] is the ordinal p (0xffff: not a survivor).
template <int L>
__global__ void __launch_bounds__(1024, 1) k_once_direct_lut(
    DevCorpus c, const uint16_t* __restrict__ lut, uint32_t lut_n, uint32_t bits, DirectWork w,
    const uint8_t* __restrict__ arank, uint32_t A, uint32_t nwords,
    uint32_t* __restrict__ compact) {
  extern __shared__ uint4 smem4[];
  char* sp = reinterpret_cast<char*>(smem4);
  uint32_t* bm = reinterpret_cast<uint32_t*>(sp);
  sp += align16((size_t)nwords * 4);
  uint8_t* s_arank = reinterpret_cast<uint8_t*>(sp);
  sp += 256;
  uint16_t* s_lut = reinterpret_cast<uint16_t*>(sp);
  for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) bm[i] = 0;
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) s_arank[i] = arank[i];
  for (uint32_t i = threadIdx.x; i < lut_n; i += blockDim.x) s_lut[i] = lut[i];
  __syncthreads();
  constexpr int PL = L - 1;
  const uint32_t pmask = (1u << (bits * PL)) - 1u;
  const int lane = threadIdx.x & 31;
  __shared__ uint32_t s_last;
  for (uint32_t qi = blockIdx.x; qi < w.nitems; qi += gridDim.x) {
    const DirectItem it = w.items[qi];
    int64_t lo, hi;
    direct_part(c, it, L, lo, hi);
    const int64_t first = (lo - (L - 1)) & ~int64_t(15);
    const int64_t nseg = (hi - first + 15) >> 4;
    const int64_t nseg_r = (nseg + 31) & ~int64_t(31);
    for (int64_t sgi = threadIdx.x; sgi < nseg_r; sgi += blockDim.x) {
      const int64_t b0 = first + sgi * 16;
      uint32_t W[7];
      seg_load(c.data, b0, lane, W);
      const uint32_t vm = sgi < nseg ? vmask(b0, lo, hi) : 0u;
      // ranks of window bytes 0..23 (bytes 8 + T are the segment's)
      uint32_t R[3] = {0u, 0u, 0u};
      static_for<0, 24>([&](auto kc) {
        constexpr int K = decltype(kc)::value;
        const uint32_t by = (W[K >> 2] >> (8 * (K & 3))) & 0xffu;
        R[K >> 3] |= (uint32_t)s_arank[by] << (4 * (K & 7));
      });
      auto rk = [&](auto kc) -> uint32_t {
        constexpr int K = decltype(kc)::value;
        return (R[K >> 3] >> (4 * (K & 7))) & 0xfu;
      };
      uint32_t pre = 0;  // prefix of the gram ending at T = 0: bytes 9-L .. 7
      static_for<9 - L, 8>([&](auto kc) { pre = (pre << bits) | rk(kc); });
      static_for<0, 16>([&](auto tc) {
        constexpr int T = decltype(tc)::value;
        if ((vm >> T) & 1u) {
          const uint32_t p = s_lut[pre & pmask];
          if (p != 0xffffu) {
            const uint32_t id = p * A + rk(std::integral_constant<int, 8 + T>{});
            uint32_t* w = bm + (id >> 5);
            const uint32_t bit = 1u << (id & 31);
            if (!(*(volatile uint32_t*)w & bit)) atomicOr(w, bit);
          }
        }
        pre = (pre << bits) | rk(std::integral_constant<int, 8 + T>{});
      });
    }
    direct_flush(bm, nwords, it, w, compact, &s_last);
  }
}

// table[p * 256 + alpha[r]] += compact[p * A + r]
template <typename CT>
__global__ void k_expand_compact(const uint32_t* __restrict__ compact, uint64_t n, uint32_t A,
                                 const uint8_t* __restrict__ alpha, CT* __restrict__ table) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = compact[i];
    if (v) {
      const uint64_t p = i / A, r = i - p * A;
      table[p * 256 + alpha[r]] += (CT)v;
    }
  }
}

// Bytes present in the corpus (256-bit mask): 16-byte loads, flags in smem.
__global__ void k_byte_presence(const uint8_t* __restrict__ data, uint64_t n,
                                uint32_t* __restrict__ mask) {
  __shared__ uint32_t sm[8];
  if (threadIdx.x < 8) sm[threadIdx.x] = 0;
  __syncthreads();
  uint32_t local[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint64_t n16 = n / 16;
  // only "at most 16 distinct bytes" matters to the caller: every 64 steps a
  // warp checks its bytes so far and the global verdict (mask[8] = 1: more)
  uint32_t step = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if ((++step & 63) == 0) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) c += __popc(__reduce_or_sync(__activemask(), local[q]));
      if (c > 16) atomicExch(mask + 8, 1u);
      if (*(volatile uint32_t*)(mask + 8)) break;
    }
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(data) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t by = (w[k >> 2] >> (8 * (k & 3))) & 0xffu;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if ((by >> 5) == (uint32_t)q) local[q] |= 1u << (by & 31);
    }
  }
  for (uint64_t i = n16 * 16 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t by = data[i];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if ((by >> 5) == (uint32_t)q) local[q] |= 1u << (by & 31);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t x = local[q];
    for (int o = 16; o; o >>= 1) x |= __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicOr(sm + q, x);
  }
  __syncthreads();
  if (threadIdx.x < 8 && sm[threadIdx.x]) atomicOr(mask + threadIdx.x, sm[threadIdx.x]);
}

// Dense count-once over a small alphabet: compact[(r0 * A + r1) * A + r2]
// counts the 3-gram alpha[r0] alpha[r1] alpha[r2]; added into the dense
// table at its route permutation (index = key * mult & cmask).
template <typename CT>
__global__ void k_expand_dense(const uint32_t* __restrict__ compact, uint32_t A,
                               const uint8_t* __restrict__ alpha, uint64_t mult, uint64_t cmask,
                               CT* __restrict__ table) {
  const uint32_t n = A * A * A;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = compact[i];
    if (v) {
      const uint32_t r2 = i % A, r1 = (i / A) % A, r0 = i / (A * A);
      const uint64_t key = ((uint64_t)alpha[r0] << 16) | ((uint64_t)alpha[r1] << 8) | alpha[r2];
      table[(key * mult) & cmask] += (CT)v;
    }
  }
}

// Byte alphabet of a corpus from its dense count-once n0-gram table: every
// byte that can end an extension-pass gram lies in some counted n0-gram.
// index -> key = (index * minv) & cmask (the dense route permutation).
template <typename CT>
__global__ void k_alphabet(const CT* __restrict__ table, uint64_t cap, uint64_t minv,
                           uint64_t cmask, uint32_t n0, uint32_t* __restrict__ mask) {
  __shared__ uint32_t sm[8];
  if (threadIdx.x < 8) sm[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (table[i]) {
      const uint64_t key = minv ? ((i * minv) & cmask) : i;
      for (uint32_t b = 0; b < n0; ++b) {
        const uint32_t by = (uint32_t)(key >> (8 * b)) & 0xffu;
        if (!(sm[by >> 5] & (1u << (by & 31)))) atomicOr(sm + (by >> 5), 1u << (by & 31));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 8 && sm[threadIdx.x]) atomicOr(mask + threadIdx.x, sm[threadIdx.x]);
}

// ------------------------------------------------------------------ host

static size_t table_bytes(const RouteParams& rp) {
  return align16((size_t)rp.nslots * 8 + (size_t)rp.nb * 2);
}

// Exclusive prefix sum of u32 region sizes into u64 offsets, accumulated in 64
// bits (a corpus can route more than 2^32 positions).
struct WidenU64 {
  __host__ __device__ unsigned long long operator()(uint32_t v) const { return v; }
};
static void scan_u32_to_u64(RouteCtx& x, const uint32_t* cnt, unsigned long long* base, size_t n,
                            cudaStream_t st) {
  cub::TransformInputIterator<unsigned long long, WidenU64, const uint32_t*> in(cnt, WidenU64{});
  size_t need = 0;
  IGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, in, base, (int64_t)n, st));
  void* tmp = x.cub_tmp.get(need);
  IGB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, in, base, (int64_t)n, st));
}

// Folds a fused owner histogram built at 2^d times this pass's owner count:
// owner_hash keeps the top bits of one hash, so owner o at the narrower width
// covers owners [o << d, (o + 1) << d) of the wider one.
__global__ void k_fold_counts(const uint32_t* __restrict__ wide, uint32_t d, uint32_t NO,
                              uint32_t nunits, uint32_t* __restrict__ cnt) {
  const uint64_t n = (uint64_t)NO * nunits;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t o = i / nunits, u = i - o * nunits;
    uint32_t sum = 0;
    for (uint32_t w = 0; w < (1u << d); ++w) sum += wide[((o << d) + w) * nunits + u];
    cnt[i] = sum;
  }
}

// Stage 1: count kernel + owner-major scan (needs only the owner function).
template <int KIND, int L>
static void route_stage1_t(RouteCtx& x, const DevCorpus& c, const RouteParams& rp, int num_sms,
                           cudaStream_t st) {
  const RouteView uv = x.view();
  const size_t ncnt = (size_t)rp.NO * uv.nb + 1;
  x.actual.as<uint32_t>(ncnt);
  unsigned long long* base = x.base.as<unsigned long long>(ncnt);
  if (KIND == 1 && x.have_next && x.next_lgno == (int32_t)rp.lgno) {
    // the previous pass's scatter already histogrammed this pass's owners
    x.cnt.swap(x.cnt_next);
    x.have_next = false;
    uint32_t* cnt = x.cnt.as<uint32_t>(ncnt);
    scan_u32_to_u64(x, cnt, base, ncnt, st);
    return;
  }
  if (KIND == 1 && x.have_next && x.next_lgno > (int32_t)rp.lgno && uv.u0 == 0 &&
      uv.nb == x.nunits) {
    // the survivors came out fewer than the fused width was sized for (a
    // small alphabet): fold the fused histogram instead of recounting
    uint32_t* cnt = x.cnt.as<uint32_t>(ncnt);
    const uint64_t n = (uint64_t)rp.NO * uv.nb;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 4096);
    IGB_CUDA(cudaMemsetAsync(cnt + ncnt - 1, 0, 4, st));
    if (n) {
      k_fold_counts<<<grid, 256, 0, st>>>(x.cnt_next.as<uint32_t>(1), x.next_lgno - rp.lgno,
                                          rp.NO, uv.nb, cnt);
      x.launches++;
    }
    x.have_next = false;
    scan_u32_to_u64(x, cnt, base, ncnt, st);
    IGB_CUDA(cudaGetLastError());
    return;
  }
  x.have_next = false;
  uint32_t* cnt = x.cnt.as<uint32_t>(ncnt);
  const size_t smem = align16((size_t)rp.NO * 4);
  auto k = k_route_count<KIND, L>;
  IGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  IGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kRouteThreads, smem));
  if (per < 1) throw Error(IG_EINTERNAL, "route count does not fit in shared memory");
  const unsigned grid = (unsigned)std::min<uint64_t>(uv.nb, (uint64_t)num_sms * per);
  IGB_CUDA(cudaMemsetAsync(cnt + ncnt - 1, 0, 4, st));
  const size_t ev = x.kt ? x.kt->begin(IG_KF_ROUTE_COUNT, st) : 0;
  k<<<grid, kRouteThreads, smem, st>>>(c, uv, rp, cnt);
  if (x.kt) x.kt->end(ev, st);
  x.launches++;
  scan_u32_to_u64(x, cnt, base, ncnt, st);
  IGB_CUDA(cudaGetLastError());
}

// Stage 2: scatter + consume (needs the prefix table for extension passes).
template <int KIND, int L, int TAB, typename CT>
static void route_stage2_t(RouteCtx& x, const DevCorpus& c, const RouteParams& rp, CT* table,
                           int num_sms, cudaStream_t st) {
  const RouteView uv = x.view();
  const size_t tab = (TAB == 1 || TAB == 4) ? table_bytes(rp) : 0;
  const size_t ncnt = (size_t)rp.NO * uv.nb + 1;
  uint32_t* act = x.actual.as<uint32_t>(ncnt);  // TAB 10/11: dense with 1024/768 threads
  unsigned long long* base = x.base.as<unsigned long long>(ncnt);
  uint16_t* ent = x.entries.as<uint16_t>(c.total + 64);
  RouteParams rq = rp;
  if (rp.next_lgno >= 0) {
    const size_t nn = ((size_t)1 << rp.next_lgno) * x.nunits + 1;
    rq.next_cnt = x.cnt_next.as<uint32_t>(nn);
    // batched (pipelined) dense passes accumulate into one next-pass histogram
    if (x.u0 == 0) IGB_CUDA(cudaMemsetAsync(rq.next_cnt, 0, nn * 4, st));
    x.have_next = true;
    x.next_lgno = rp.next_lgno;
  }
  {
    constexpr int NT = TAB == 1 || TAB == 11 ? kScatterThreadsBig
                       : (TAB == 10 || TAB == 12) ? 1024 : kScatterThreads;
    constexpr int DS = (TAB == 1 || TAB == 4) ? 2048 : TAB == 12 ? 8192 : kDedupSlots;
    constexpr int KT = TAB >= 10 ? 0 : TAB;  // dense variants carry no table
    const size_t nxt = rp.next_lgno >= 0 ? align16(((size_t)1 << rp.next_lgno) * 4) : 0;
    const size_t smem = (size_t)NT * 16 * 4 + (size_t)DS * 8 + align16((size_t)rp.NO * 8) +
                        align16((size_t)rp.NO * 4) + align16((size_t)rp.NO * 8) + nxt + tab;
    auto k = k_route_scatter<KIND, L, KT, NT, DS>;
    IGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 0;
    IGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, NT, smem));
    if (per < 1) throw Error(IG_EINTERNAL, "route scatter does not fit in shared memory");
    const unsigned grid = (unsigned)std::min<uint64_t>(uv.nb, (uint64_t)num_sms * per);
    const size_t ev = x.kt ? x.kt->begin(IG_KF_ROUTE_SCATTER, st) : 0;
    k<<<grid, NT, smem, st>>>(c, uv, rq, base, act, ent);
    if (x.kt) x.kt->end(ev, st);
    x.launches++;
  }
  {
    const uint32_t ipo = 1u << rp.lgl;
    const uint32_t bmw4 = consume_region_words(ipo);
    const size_t smem = align16((size_t)(ipo + 1) / 2 * 4) + (size_t)kConsumeWarps * bmw4 * 4;
    auto k = k_consume_once<CT>;
    IGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 0;
    IGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kConsumeThreads, smem));
    if (per < 1) throw Error(IG_EINTERNAL, "route consume does not fit in shared memory");
    const uint64_t slots = (uint64_t)num_sms * per;
    const uint64_t mq = uv.q1 - uv.q0;
    static const char* cg = getenv("IG_CONSUME_GRAIN");
    const uint64_t grain = cg ? std::max<uint64_t>(1, strtoull(cg, nullptr, 10)) : 8;
    uint64_t nblocks = (slots * grain + rp.NO - 1) / rp.NO;
    if (nblocks > mq) nblocks = mq;
    if (nblocks < 1) nblocks = 1;
    uint64_t sb = (mq + nblocks - 1) / nblocks;
    if (sb > 65535) sb = 65535;  // u16 smem counters: <= 65535 sequences per item
    if (sb < 1) sb = 1;
    nblocks = (mq + sb - 1) / sb;
    if (nblocks < 1) nblocks = 1;
    const uint64_t nitems = (uint64_t)rp.NO * nblocks;
    const unsigned grid = (unsigned)std::min<uint64_t>(nitems, slots);
    uint32_t* ord = x.consume_order.as<uint32_t>(2 * (size_t)rp.NO + 8);
    uint32_t* work = ord + rp.NO + 4;
    uint32_t* tot = work + 4;
    const size_t ev = x.kt ? x.kt->begin(IG_KF_ROUTE_CONSUME, st) : 0;
    static const bool no_order = getenv("IG_CONSUME_NO_ORDER") != nullptr;
    if (!no_order && rp.NO <= (uint32_t)(kOrderThreads * kOrderItems)) {
      k_owner_totals<<<rp.NO, 256, 0, st>>>(act, uv.nb, tot);
      k_owner_order<<<1, kOrderThreads, 0, st>>>(tot, rp.NO, ord, work);
      x.launches++;
    } else {  // identity order, written on the stream (no host stall)
      k_identity_order<<<(rp.NO + 255) / 256, 256, 0, st>>>(ord, rp.NO, work);
    }
    x.launches++;
    k<<<grid, kConsumeThreads, smem, st>>>(uv, rp, (uint32_t)sb, (uint32_t)nblocks, base, act,
                                            ent, table, ord, work);
    if (x.kt) x.kt->end(ev, st);
    x.launches++;
  }
  IGB_CUDA(cudaGetLastError());
}

template <int KIND, int L, typename CT>
static void route_stage_l(int stage, RouteCtx& x, const DevCorpus& c, const RouteParams& rp,
                          CT* table, int num_sms, cudaStream_t st) {
  if (stage == 1) {
    route_stage1_t<KIND, L>(x, c, rp, num_sms, st);
  } else if constexpr (KIND == 0) {
    // dense: one 1024-thread CTA per SM with an 8192-slot dedup cache
    // (measured best of 512/768/1024 threads and 4096/8192 slots)
    route_stage2_t<0, L, 12, CT>(x, c, rp, table, num_sms, st);
  } else {
    auto fixed = [&](size_t nt) {  // + static smem
      const size_t nxt = rp.next_lgno >= 0 ? align16(((size_t)1 << rp.next_lgno) * 4) : 0;
      return nt * 64 + 2048 * 8 + (size_t)rp.NO * 20 + 256 + nxt + 8 * 1024;
    };
    // the table is staged in shared memory when it fits (one 768-thread CTA
    // per SM: measured 1.2x faster than L1-cached global loads with two
    // 512-thread CTAs); IG_SCATTER_TABLE_GLOBAL=1 forces the global variant
    static const bool force_global = getenv("IG_SCATTER_TABLE_GLOBAL") != nullptr;
    if (!force_global && fixed(kScatterThreadsBig) + table_bytes(rp) <= kMaxOnceSmem)
      route_stage2_t<1, L, 1, CT>(x, c, rp, table, num_sms, st);
    else if (!force_global && fixed(kScatterThreads) + table_bytes(rp) <= kMaxOnceSmem)
      route_stage2_t<1, L, 4, CT>(x, c, rp, table, num_sms, st);
    else
      route_stage2_t<1, L, 2, CT>(x, c, rp, table, num_sms, st);
  }
}

template <typename CT>
void route_count_once(int stage, RouteCtx& x, const DevCorpus& c, int kind, uint32_t L,
                      const RouteParams& rp, CT* table, int num_sms, cudaStream_t st) {
  if (!c.m || !x.nunits || x.u1 <= x.u0) return;
  if (kind == 0) {
    switch (L) {
      case 1: route_stage_l<0, 1, CT>(stage, x, c, rp, table, num_sms, st); break;
      case 2: route_stage_l<0, 2, CT>(stage, x, c, rp, table, num_sms, st); break;
      default: route_stage_l<0, 3, CT>(stage, x, c, rp, table, num_sms, st); break;
    }
  } else {
    switch (L) {
      case 2: route_stage_l<1, 2, CT>(stage, x, c, rp, table, num_sms, st); break;
      case 3: route_stage_l<1, 3, CT>(stage, x, c, rp, table, num_sms, st); break;
      case 4: route_stage_l<1, 4, CT>(stage, x, c, rp, table, num_sms, st); break;
      case 5: route_stage_l<1, 5, CT>(stage, x, c, rp, table, num_sms, st); break;
      case 6: route_stage_l<1, 6, CT>(stage, x, c, rp, table, num_sms, st); break;
      case 7: route_stage_l<1, 7, CT>(stage, x, c, rp, table, num_sms, st); break;
      case 8: route_stage_l<1, 8, CT>(stage, x, c, rp, table, num_sms, st); break;
      default: throw Error(IG_ECONFIG, "gram length above 8 is not supported");
    }
  }
}

template void route_count_once<uint32_t>(int, RouteCtx&, const DevCorpus&, int, uint32_t,
                                         const RouteParams&, uint32_t*, int, cudaStream_t);
template void route_count_once<unsigned long long>(int, RouteCtx&, const DevCorpus&, int, uint32_t,
                                                   const RouteParams&, unsigned long long*, int,
                                                   cudaStream_t);

// ------------------------------------------------------------------ prefix set (host)

// CHD construction: buckets by decreasing size, each takes the first
// displacement that sends all its keys to free slots.  Per-key hashes are
// computed once; buckets are a counting sort.  False on failure.
static bool mphf_try(const std::vector<uint64_t>& keys, uint32_t nb, uint32_t nslots, bool narrow,
                     std::vector<uint16_t>& disp, std::vector<uint32_t>& slot_of_key) {
  const uint32_t K = (uint32_t)keys.size();
  std::vector<uint32_t> kb(K), ks(K), kt(K), boff(nb + 1, 0), idx(K);
  for (uint32_t i = 0; i < K; ++i) {
    const MphfHash h = narrow ? mphf_hash<true>(keys[i], nb) : mphf_hash<false>(keys[i], nb);
    kb[i] = h.b;
    ks[i] = h.s;
    kt[i] = h.t;
    ++boff[kb[i] + 1];
  }
  uint32_t maxsz = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    maxsz = std::max(maxsz, boff[b + 1]);
    boff[b + 1] += boff[b];
  }
  {
    std::vector<uint32_t> cur(boff.begin(), boff.end() - 1);
    for (uint32_t i = 0; i < K; ++i) idx[cur[kb[i]]++] = i;
  }
  // buckets ordered by decreasing size (counting sort on size)
  std::vector<uint32_t> szoff(maxsz + 2, 0), order(nb);
  for (uint32_t b = 0; b < nb; ++b) ++szoff[maxsz - (boff[b + 1] - boff[b]) + 1];
  for (uint32_t z = 0; z <= maxsz; ++z) szoff[z + 1] += szoff[z];
  for (uint32_t b = 0; b < nb; ++b) order[szoff[maxsz - (boff[b + 1] - boff[b])]++] = b;
  // occupancy bitset (fits L1); a bucket's hashes gathered once, contiguous
  std::vector<uint64_t> used((nslots + 63) / 64, 0);
  disp.assign(nb, 0);
  slot_of_key.assign(K, 0);
  uint32_t cand[64], bs[64], bt[64];
  for (uint32_t b : order) {
    const uint32_t a0 = boff[b], n = boff[b + 1] - a0;
    if (n == 0) break;
    if (n > 64) return false;
    for (uint32_t t = 0; t < n; ++t) {
      bs[t] = ks[idx[a0 + t]];
      bt[t] = kt[idx[a0 + t]];
    }
    auto place = [&](uint32_t t, uint32_t d) {
      return (uint32_t)(((uint64_t)(bs[t] + d * bt[t]) * nslots) >> 32);
    };
    auto is_used = [&](uint32_t sl) { return (uint32_t)(used[sl >> 6] >> (sl & 63)) & 1u; };
    if (n <= 2) {  // most buckets: branch-free tests, one mispredict per bucket
      uint32_t d = 0;
      if (n == 1) {
        while (d < 65536 && is_used(place(0, d))) ++d;
      } else {
        for (; d < 65536; ++d) {
          const uint32_t s0 = place(0, d), s1 = place(1, d);
          if (!(is_used(s0) | is_used(s1) | (uint32_t)(s0 == s1))) break;
        }
      }
      if (d >= 65536) return false;
      disp[b] = (uint16_t)d;
      for (uint32_t t = 0; t < n; ++t) {
        const uint32_t sl = place(t, d);
        used[sl >> 6] |= 1ull << (sl & 63);
        slot_of_key[idx[a0 + t]] = sl;
      }
      continue;
    }
    bool ok = false;
    for (uint32_t d = 0; d < 65536 && !ok; ++d) {
      // every test of a trial, then one branch (the loop trip counts repeat)
      uint32_t bad = 0;
      for (uint32_t t = 0; t < n; ++t) {
        cand[t] = place(t, d);
        bad |= is_used(cand[t]);
      }
      for (uint32_t t = 1; t < n; ++t)
        for (uint32_t u = 0; u < t; ++u) bad |= (uint32_t)(cand[u] == cand[t]);
      ok = !bad;
      if (ok) disp[b] = (uint16_t)d;
    }
    if (!ok) return false;
    for (uint32_t t = 0; t < n; ++t) {
      used[cand[t] >> 6] |= 1ull << (cand[t] & 63);
      slot_of_key[idx[a0 + t]] = cand[t];
    }
  }
  return true;
}

void build_prefix_mphf(const std::vector<uint64_t>& keys, bool narrow,
                       std::vector<uint32_t>& slot_of_key, std::vector<uint16_t>& disp,
                       uint32_t& nb, uint32_t& nslots) {
  const uint64_t K = keys.size();
  nb = (uint32_t)std::max<uint64_t>(1, (K + 2) / 3);
  nslots = (uint32_t)std::max<uint64_t>(1, K + K / 8 + 1);  // ~89% load
  while (!mphf_try(keys, nb, nslots, narrow, disp, slot_of_key)) {
    nslots += nslots / 20 + 1;
    nb += nb / 10 + 1;
  }
}

// Host: the permuted id space of a candidate space of `cap` ids.
size_t direct_smem(const RouteParams& rp, uint64_t nbits) {
  return align16((nbits + 31) / 32 * 4) + align16((size_t)rp.NO * 4) + 256 + table_bytes(rp);
}

template <typename CT>
void alphabet_mask(const CT* table, uint64_t cap, uint64_t minv, uint64_t cmask, uint32_t n0,
                   uint32_t* mask, int num_sms, cudaStream_t st) {
  IGB_CUDA(cudaMemsetAsync(mask, 0, 8 * sizeof(uint32_t), st));
  const unsigned grid = (unsigned)std::min<uint64_t>((cap + 255) / 256, (uint64_t)num_sms * 8);
  k_alphabet<CT><<<grid ? grid : 1, 256, 0, st>>>(table, cap, minv, cmask, n0, mask);
  IGB_CUDA(cudaGetLastError());
}

template <typename CT>
void count_once_direct(const DevCorpus& c, uint32_t L, const RouteParams& rp,
                       const DirectWork& w, const uint8_t* arank,
                       const uint8_t* alpha, uint32_t A, uint64_t K, uint32_t* compact, CT* table,
                       int num_sms, cudaStream_t st, const uint16_t* lut, uint32_t lut_n,
                       uint32_t bits, bool expand) {
  const uint64_t nbits = K * A;
  const uint32_t nwords = (uint32_t)((nbits + 31) / 32);
  IGB_CUDA(cudaMemsetAsync(compact, 0, nbits * 4, st));
  if (w.nsplit) {
    IGB_CUDA(cudaMemsetAsync(w.gbm, 0, (size_t)w.nsplit * nwords * 4, st));
    IGB_CUDA(cudaMemsetAsync(w.done, 0, (size_t)w.nsplit * 4, st));
  }
  const uint32_t nseqs = w.nitems;
  if (nseqs && lut) {
    const size_t smem = align16((size_t)nwords * 4) + 256 + (size_t)lut_n * 2;
    auto go = [&](auto k) {
      IGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const unsigned grid = (unsigned)std::min<uint64_t>(nseqs, (uint64_t)num_sms);
      k<<<grid, 1024, smem, st>>>(c, lut, lut_n, bits, w, arank, A, nwords, compact);
    };
    switch (L) {
      case 3: go(k_once_direct_lut<3>); break;
      case 4: go(k_once_direct_lut<4>); break;
      case 5: go(k_once_direct_lut<5>); break;
      case 6: go(k_once_direct_lut<6>); break;
      case 7: go(k_once_direct_lut<7>); break;
      case 8: go(k_once_direct_lut<8>); break;
      default: throw Error(IG_EINTERNAL, "direct lookup table needs 3 <= j <= 8");
    }
  } else if (nseqs) {
    const size_t smem = direct_smem(rp, nbits);
    auto go = [&](auto k) {
      IGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const unsigned grid = (unsigned)std::min<uint64_t>(nseqs, (uint64_t)num_sms);
      k<<<grid, kDirectThreads, smem, st>>>(c, rp, w, arank, A, nwords, compact);
    };
    switch (L) {
      case 2: go(k_once_direct<2>); break;
      case 3: go(k_once_direct<3>); break;
      case 4: go(k_once_direct<4>); break;
      case 5: go(k_once_direct<5>); break;
      case 6: go(k_once_direct<6>); break;
      case 7: go(k_once_direct<7>); break;
      case 8: go(k_once_direct<8>); break;
      default: throw Error(IG_ECONFIG, "gram length above 8 is not supported");
    }
  }
  if (!expand) return;
  const unsigned g2 = (unsigned)std::min<uint64_t>((nbits + 255) / 256, (uint64_t)num_sms * 8);
  k_expand_compact<CT><<<g2 ? g2 : 1, 256, 0, st>>>(compact, nbits, A, alpha, table);
  IGB_CUDA(cudaGetLastError());
}

void byte_presence(const uint8_t* data, uint64_t n, uint32_t* mask, int num_sms,
                   cudaStream_t st) {
  IGB_CUDA(cudaMemsetAsync(mask, 0, 9 * sizeof(uint32_t), st));
  if (!n) return;
  const unsigned grid =
      (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n / 16 + 255) / 256, (uint64_t)num_sms * 8));
  k_byte_presence<<<grid, 256, 0, st>>>(data, n, mask);
  IGB_CUDA(cudaGetLastError());
}

template <typename CT>
void expand_dense(const uint32_t* compact, uint32_t A, const uint8_t* alpha, uint64_t mult,
                  uint64_t cmask, CT* table, cudaStream_t st) {
  k_expand_dense<CT><<<16, 256, 0, st>>>(compact, A, alpha, mult, cmask, table);
  IGB_CUDA(cudaGetLastError());
}
template void expand_dense<uint32_t>(const uint32_t*, uint32_t, const uint8_t*, uint64_t, uint64_t,
                                     uint32_t*, cudaStream_t);
template void expand_dense<unsigned long long>(const uint32_t*, uint32_t, const uint8_t*, uint64_t,
                                               uint64_t, unsigned long long*, cudaStream_t);

template void alphabet_mask<uint32_t>(const uint32_t*, uint64_t, uint64_t, uint64_t, uint32_t,
                                      uint32_t*, int, cudaStream_t);
template void alphabet_mask<unsigned long long>(const unsigned long long*, uint64_t, uint64_t,
                                                uint64_t, uint32_t, uint32_t*, int, cudaStream_t);
template void count_once_direct<uint32_t>(const DevCorpus&, uint32_t, const RouteParams&,
                                          const DirectWork&, const uint8_t*,
                                          const uint8_t*, uint32_t, uint64_t, uint32_t*,
                                          uint32_t*, int, cudaStream_t, const uint16_t*, uint32_t,
                                          uint32_t, bool);
template void count_once_direct<unsigned long long>(const DevCorpus&, uint32_t,
                                                    const RouteParams&, const DirectWork&,
                                                    const uint8_t*, const uint8_t*, uint32_t,
                                                    uint64_t, uint32_t*, unsigned long long*, int,
                                                    cudaStream_t, const uint16_t*, uint32_t,
                                                    uint32_t, bool);

void make_route_params(uint64_t cap, RouteParams& rp) {
  uint32_t lgc = 0;
  while ((1ull << lgc) < cap) ++lgc;
  if (lgc < 2) lgc = 2;
  rp.lgc = lgc;
  rp.lgl = lgc < 14 ? lgc : 14;
  rp.NO = 1u << (lgc - rp.lgl);
  rp.cmask = lgc >= 64 ? ~0ull : ((1ull << lgc) - 1);
  rp.mult = (0x9E3779B97F4A7C15ull & rp.cmask) | 1ull;
  uint64_t inv = rp.mult;  // Newton: inv = inv * (2 - mult * inv) mod 2^64
  for (int i = 0; i < 6; ++i) inv *= 2ull - rp.mult * inv;
  rp.minv = inv & rp.cmask;
}

}  // namespace igb
