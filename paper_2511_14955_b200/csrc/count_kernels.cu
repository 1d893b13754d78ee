// count_kernels.cu — the count-all counting passes of Intergrams on sm_100a
// (count-once passes route through route_kernels.cu), tile descriptors and
// the count-all prefix set.
//
// Reference semantics:
//   dense pass     proj/src/intergrams.cpp:79-100 (= dense_pass.cpp:21-39):
//                  every n0-gram of every sequence, id = big-endian bytes.
//   extension pass proj/src/intergrams.cpp:44-66: every j-gram whose (j-1)-byte
//                  prefix is a survivor p; id = p*256 + last byte.
//   count-all      pipeline.hpp:106-113: counts[id] += 1 per occurrence.
//   count-once     counting.hpp:48-74 + counting.cpp:27-50: counts[id] += 1 per
//                  sequence that contains id.
// n-grams never cross sequence boundaries (intergrams.cpp:53-57).
//
// B200 design:
//   * every lane owns a 16-byte segment, read with one 128-bit load; a warp
//     covers 512 contiguous bytes, so a 32-lane load is one fully coalesced
//     512 B transaction.  The 8 bytes before a segment (the n-gram halo) come
//     from the neighbouring lane by shuffle, never from a second HBM read.
//   * n-gram keys are assembled in registers with funnel shifts / byte perms
//     at compile-time byte offsets (the gram length is a template parameter).
//   * count-all: one L2 reduction (RED) per occurrence, except for the ids a
//     CTA's shared-memory hot cache owns (counted with shared atomics and
//     flushed once), so hot Zipf grams do not serialise on one L2 slice.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ig_internal.cuh"
#include "kernels.h"

namespace igb {

// ------------------------------------------------------------------ helpers

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// W[0..1] = the 8 bytes before the segment, W[2..5] = the segment, W[6] = 0.
struct Seg {
  uint32_t W[7];
};

// Loads lane's 16-byte segment at byte index b0 (16-aligned, may be past the
// end: padding is readable) and its 8-byte halo from lane-1 (lane 0 loads it).
// Requires the full warp, with lanes holding consecutive segments.
__device__ __forceinline__ void load_seg(const uint8_t* __restrict__ data, int64_t b0, Seg& s) {
  const uint4 v = __ldcs(reinterpret_cast<const uint4*>(data + b0));
  s.W[2] = v.x;
  s.W[3] = v.y;
  s.W[4] = v.z;
  s.W[5] = v.w;
  s.W[6] = 0;
  uint32_t h0 = __shfl_up_sync(0xffffffffu, v.z, 1);
  uint32_t h1 = __shfl_up_sync(0xffffffffu, v.w, 1);
  if ((threadIdx.x & 31) == 0) {
    const uint2 h = *reinterpret_cast<const uint2*>(data + b0 - 8);
    h0 = h.x;
    h1 = h.y;
  }
  s.W[0] = h0;
  s.W[1] = h1;
}

// Word q of the segment shifted back by D bytes: byte r = b[b0 + 4q + r - D].
template <int Q, int D>
__device__ __forceinline__ uint32_t shifted(const Seg& s) {
  constexpr int o = 8 + 4 * Q - D;
  constexpr int wi = o / 4, sh = 8 * (o % 4);
  if constexpr (sh == 0) return s.W[wi];
  else return __funnelshift_r(s.W[wi], s.W[wi + 1], sh);
}

// Big-endian key of the 8 bytes ending at segment position T.
template <int T>
__device__ __forceinline__ uint64_t key8_at(const Seg& s) {
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
__device__ __forceinline__ uint64_t gram_mask() {
  if constexpr (L >= 8) return ~0ull;
  else return (1ull << (8 * L)) - 1;
}

// Per-byte zero test of y (bytes < 0x80) -> 4-bit mask, bit r = byte r == 0.
__device__ __forceinline__ uint32_t zero_bytes4(uint32_t y) {
  const uint32_t z = ~(((y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | y) & 0x80808080u;
  return (((z >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// 16-bit mask of segment positions whose window belongs to owner o.
// KIND 0 (dense, L = 3): owner = (b[i-2] ^ b[i-1] ^ b[i]) & (G-1).
// KIND 1 (extension, prefix = b[i-L+1 .. i-1]): owner = prefix_owner(prefix).
template <int KIND, int L, int Q>
__device__ __forceinline__ uint32_t owner_word(const Seg& s, uint32_t gm4, uint32_t o4) {
  uint32_t x;
  if constexpr (KIND == 0) {
    x = shifted<Q, 0>(s) ^ shifted<Q, 1>(s) ^ shifted<Q, 2>(s);
  } else {
    constexpr int P = L - 1;  // prefix length
    if constexpr (P >= 2) x = shifted<Q, 1>(s) ^ shifted<Q, P>(s);
    else x = shifted<Q, 1>(s);
  }
  return zero_bytes4((x & gm4) ^ o4) << (4 * Q);
}

template <int KIND, int L>
__device__ __forceinline__ uint32_t owner_mask(const Seg& s, uint32_t gm4, uint32_t o4) {
  return owner_word<KIND, L, 0>(s, gm4, o4) | owner_word<KIND, L, 1>(s, gm4, o4) |
         owner_word<KIND, L, 2>(s, gm4, o4) | owner_word<KIND, L, 3>(s, gm4, o4);
}

// 16-bit mask of valid gram ends in [b0, b0+16) for one sequence [s0, s1).
template <int L>
__device__ __forceinline__ uint32_t valid_mask_one(int64_t b0, int64_t s0, int64_t s1) {
  const int64_t lo = s0 + L - 1;  // first valid gram end
  int64_t a = lo - b0;
  int64_t b = s1 - b0;
  if (a < 0) a = 0;
  if (b > 16) b = 16;
  if (a >= b) return 0;
  return ((1u << b) - 1u) & ~((1u << a) - 1u);
}

// Open-addressing lookup of a prefix key in owner slice `o` (global/L2).
// Returns p or 0xffffffff.  Slices: keys[o*S .. o*S+S).
__device__ __forceinline__ uint32_t prefix_lookup(const uint64_t* __restrict__ hkeys,
                                                  const uint32_t* __restrict__ hidx, uint32_t S,
                                                  uint32_t lgS, uint32_t o, uint64_t key,
                                                  uint32_t hmask = ~3u) {
  const uint64_t* kk = hkeys + (size_t)o * S;
  uint32_t h = hash_slot(key, lgS, hmask);
  for (;;) {
    const uint64_t k = __ldg(kk + h);
    if (k == key) return __ldg(hidx + (size_t)o * S + h);
    if (k == kEmptyKey) return 0xffffffffu;
    h = (h + 1) & (S - 1);
  }
}

// Packed prefix-set slice: entry = (key << ib) | local index, kEmptyKey = empty.
// Returns the local index (p - owner_start) or 0xffffffff.
// GLOBAL: the slice lives in global memory (read-only path), else in smem.
template <bool GLOBAL = false>
__device__ __forceinline__ uint32_t lookup_packed(const uint64_t* tab, uint32_t lgS, uint32_t ib,
                                                  uint64_t key) {
  const uint32_t mask = (1u << lgS) - 1;
  uint32_t h = hash_slot(key, lgS);
  for (;;) {
    const uint64_t e = GLOBAL ? __ldg(tab + h) : tab[h];
    if (e == kEmptyKey) return 0xffffffffu;
    if ((e >> ib) == key) return (uint32_t)(e & ((1ull << ib) - 1));
    h = (h + 1) & mask;
  }
}

// The same probe over {key, p} 16-byte slots: one 16-byte load per probe.
__device__ __forceinline__ uint32_t lookup_wide(const uint64_t* __restrict__ wide, uint32_t lgS,
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

// 3-byte prefix p in the rank bitmap: one 16-byte load, no probing.
__device__ __forceinline__ uint32_t lookup_rank(const uint64_t* __restrict__ rankbits,
                                                uint32_t pre) {
  const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(rankbits) + (pre >> 6));
  const uint64_t bit = 1ull << (pre & 63);
  return (e.x & bit) ? (uint32_t)e.y + (uint32_t)__popcll(e.x & (bit - 1)) : 0xffffffffu;
}

// ------------------------------------------------------------------ tiles

// tile_desc[t]: bit 31 = "fast" (the 512-byte tile lies inside one sequence
// and starts >= 7 bytes after its start, so every position is a valid gram end
// for any n <= 8); bits 0..30 = sequence containing byte t*512.
__global__ void k_tile_desc(const uint64_t* __restrict__ off, uint64_t m, uint64_t ntiles,
                            uint32_t* __restrict__ desc) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = t * kTileBytes;
    uint64_t lo = 0, hi = m + 1;  // first index with off > b
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (off[mid] <= b) lo = mid + 1;
      else hi = mid;
    }
    uint64_t s = lo ? lo - 1 : 0;
    if (s >= m) s = m ? m - 1 : 0;
    const bool fast = m && off[s + 1] >= b + kTileBytes && b >= off[s] + 7;
    desc[t] = (uint32_t)s | (fast ? 0x80000000u : 0u);
  }
}

void launch_tile_seq(const uint64_t* off, uint64_t m, uint64_t ntiles, uint32_t* desc,
                     cudaStream_t st) {
  if (!ntiles) return;
  const int threads = 256;
  const uint64_t blocks = (ntiles + threads - 1) / threads;
  k_tile_desc<<<(unsigned)(blocks < 65535 ? blocks : 65535), threads, 0, st>>>(off, m, ntiles,
                                                                             desc);
}

// Packs owner slices of the open-addressing prefix set for shared-memory staging.
__global__ void k_pack_prefix(const uint64_t* __restrict__ hkeys, const uint32_t* __restrict__ hidx,
                              const uint32_t* __restrict__ owner_start, uint32_t S, uint32_t ib,
                              uint64_t total, uint64_t* __restrict__ packed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = hkeys[i];
    const uint32_t o = (uint32_t)(i / S);
    packed[i] = k == kEmptyKey ? kEmptyKey : ((k << ib) | (uint64_t)(hidx[i] - owner_start[o]));
  }
}

void launch_pack_prefix(const DevPrefixSet& ps, uint64_t* packed, cudaStream_t st) {
  const uint64_t total = (uint64_t)ps.G * ps.S;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  k_pack_prefix<<<blocks < 4096 ? blocks : 4096, 256, 0, st>>>(ps.hkeys, ps.hidx, ps.owner_start,
                                                               ps.S, ps.ib, total, packed);
}

__global__ void k_pack_wide(const uint64_t* __restrict__ hkeys, const uint32_t* __restrict__ hidx,
                            uint64_t total, uint64_t* __restrict__ wide) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = hkeys[i];
    reinterpret_cast<ulonglong2*>(wide)[i] =
        make_ulonglong2(k, k == kEmptyKey ? 0ull : (unsigned long long)hidx[i]);
  }
}

void launch_pack_wide(const DevPrefixSet& ps, uint64_t* wide, cudaStream_t st) {
  const uint64_t total = (uint64_t)ps.G * ps.S;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  k_pack_wide<<<blocks < 4096 ? blocks : 4096, 256, 0, st>>>(ps.hkeys, ps.hidx, total, wide);
}

constexpr uint32_t kRankWords = 1u << 18;  // 2^24 prefixes / 64

__global__ void k_rank_set(const uint64_t* __restrict__ keys, uint32_t K,
                           unsigned long long* __restrict__ rankbits) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) {
    const uint32_t pre = (uint32_t)keys[i];
    atomicOr(rankbits + 2 * (pre >> 6), 1ull << (pre & 63));
  }
}

// One CTA: rank[w] = set bits in words [0, w).
__global__ void __launch_bounds__(1024) k_rank_scan(uint64_t* __restrict__ rankbits) {
  using BlockScan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename BlockScan::TempStorage tmp;
  constexpr uint32_t per = kRankWords / 1024;
  const uint32_t w0 = threadIdx.x * per;
  uint32_t sum = 0;
  for (uint32_t w = 0; w < per; ++w) sum += (uint32_t)__popcll(rankbits[2 * (w0 + w)]);
  uint32_t ex;
  BlockScan(tmp).ExclusiveSum(sum, ex);
  for (uint32_t w = 0; w < per; ++w) {
    rankbits[2 * (w0 + w) + 1] = ex;
    ex += (uint32_t)__popcll(rankbits[2 * (w0 + w)]);
  }
}

__global__ void k_rank_fill(const uint64_t* __restrict__ keys, uint32_t K,
                            const uint64_t* __restrict__ rankbits, uint64_t* __restrict__ pkeys,
                            uint32_t* __restrict__ rank_of_p) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    const uint32_t p = lookup_rank(rankbits, (uint32_t)key);
    pkeys[p] = key;
    rank_of_p[p] = i;
  }
}

void launch_rank_prefix(const uint64_t* keys, uint32_t K, uint64_t* rankbits, uint64_t* pkeys,
                        uint32_t* rank_of_p, cudaStream_t st) {
  IGB_CUDA(cudaMemsetAsync(rankbits, 0, (size_t)2 * kRankWords * 8, st));
  const unsigned blocks = std::max(1u, std::min(4096u, (K + 255) / 256));
  k_rank_set<<<blocks, 256, 0, st>>>(keys, K, reinterpret_cast<unsigned long long*>(rankbits));
  k_rank_scan<<<1, 1024, 0, st>>>(rankbits);
  k_rank_fill<<<blocks, 256, 0, st>>>(keys, K, rankbits, pkeys, rank_of_p);
}

// Slow path: validity of a segment that crosses sequence boundaries.
template <int L>
__device__ __noinline__ uint32_t valid_mask_walk(const uint64_t* __restrict__ off, uint64_t m,
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
    vm |= valid_mask_one<L>(b0, s0, s1);
    if (s1 >= b0 + 16 || q + 1 >= m) break;
    ++q;
    s0 = s1;
    s1 = (int64_t)off[q + 1];
  }
  return vm;
}

// ------------------------------------------------------------------ count-all

// Flat scan of all 512-byte tiles; one count per valid gram end (dense) or per
// prefix hit (extension).  Each warp keeps the next tile's 128-bit loads in
// flight while it counts the current one.  TAB: 0 none (dense), 1 prefix set
// staged in shared memory (packed), 2 prefix set read from global/L2 (key and
// index arrays), 3 packed prefix set read from global/L2 (one load per probe),
// 4 {key, p} 16-byte slots read from global/L2 (one load per probe), 5 rank
// bitmap of 3-byte prefixes (one 16-byte load, L2-resident 4 MiB).
//
// Hot grams: a Zipf corpus sends a few percent of all occurrences to single
// ids, and one L2 address absorbs only ~0.1 G reductions/s.  Every CTA
// therefore keeps a direct-mapped shared-memory count cache (kHotSlots ids):
// the first id to claim a slot owns it for the CTA's lifetime and is counted
// with shared-memory atomics; everything else is a RED to L2.  The cache is
// flushed with one RED per claimed slot when the CTA retires.
constexpr int kHotSlots = 4096;
constexpr uint32_t kNoId = 0xffffffffu;

template <typename CT>
__device__ __forceinline__ void count_one(uint32_t id, uint32_t* tag, uint32_t* hcnt,
                                          CT* __restrict__ table) {
  const uint32_t h = (id * 0x9E3779B1u) >> (32 - 12);
  uint32_t t = tag[h];
  if (t == kNoId) {
    t = atomicCAS(tag + h, kNoId, id);
    if (t == kNoId) t = id;
  }
  if (t == id) atomicAdd(hcnt + h, 1u);
  else atomicAdd(table + id, (CT)1);
}

template <int KIND, int L, typename CT, int TAB, bool AGG>
__global__ void __launch_bounds__(512, 3) k_count_all(DevCorpus c, DevPrefixSet ps,
                                                   const uint64_t* __restrict__ packed,
                                                   CT* __restrict__ table) {
  extern __shared__ uint64_t s_tab[];
  __shared__ uint32_t tag[kHotSlots];
  __shared__ uint32_t hcnt[kHotSlots];
  for (uint32_t i = threadIdx.x; i < kHotSlots; i += blockDim.x) {
    tag[i] = kNoId;
    hcnt[i] = 0;
  }
  if constexpr (TAB == 1) {
    for (uint32_t i = threadIdx.x; i < ps.S; i += blockDim.x) s_tab[i] = packed[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (((uint64_t)gridDim.x * blockDim.x) >> 5) * c.tstride;
  uint64_t t = c.tile0 + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * c.tstride;
  if (t < c.ntiles) {
    uint4 v = __ldcs(reinterpret_cast<const uint4*>(c.data + t * kTileBytes + lane * 16));
    uint2 h = make_uint2(0, 0);
    if (lane == 0) h = *reinterpret_cast<const uint2*>(c.data + t * kTileBytes - 8);
    uint32_t d = __ldg(c.tile_seq + t);
    // hit chaining: this lane's word and the previous segment's word of the
    // previous pass's hit mask (the prefix of the gram ending at e is the
    // gram that pass counted ending at e - 1)
    const bool chain = KIND == 1 && ps.hit_in != nullptr;
    // mk = this segment's word | the previous segment's word << 16 (lane 0)
    uint32_t mk = 0xffffffffu;
    if (chain) {
      mk = __ldcs(ps.hit_in + t * 32 + lane);
      mk |= (lane == 0 ? (uint32_t)__ldcs(ps.hit_in + t * 32 - 1) : 0xffffu) << 16;
    }
    for (;;) {
      const uint64_t tn = t + nwarps;
      uint4 vn = make_uint4(0, 0, 0, 0);
      uint2 hn = make_uint2(0, 0);
      uint32_t dn = 0, mkn = 0xffffffffu;
      if (tn < c.ntiles) {
        vn = __ldcs(reinterpret_cast<const uint4*>(c.data + tn * kTileBytes + lane * 16));
        if (lane == 0) hn = *reinterpret_cast<const uint2*>(c.data + tn * kTileBytes - 8);
        dn = __ldg(c.tile_seq + tn);
        if (chain) {
          mkn = __ldcs(ps.hit_in + tn * 32 + lane);
          mkn |= (lane == 0 ? (uint32_t)__ldcs(ps.hit_in + tn * 32 - 1) : 0xffffu) << 16;
        }
      }
      Seg s;
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
      uint32_t vm = (d >> 31) ? 0xffffu : valid_mask_walk<L>(c.off, c.m, c.total, d & 0x7fffffffu, b0);
      if (chain) {
        const uint32_t up = __shfl_up_sync(0xffffffffu, mk, 1);
        vm &= (mk << 1) | (((lane == 0 ? mk >> 16 : up) >> 15) & 1u);
      }
      uint32_t hm = 0;  // this pass's hits (extension passes)
      static_for<0, 16>([&](auto tc) {
        constexpr int T = decltype(tc)::value;
        if ((vm >> T) & 1u) {
          const uint64_t key = key8_at<T>(s) & gram_mask<L>();
          if constexpr (KIND == 0) {
            count_one<CT>((uint32_t)key, tag, hcnt, table);
          } else {
            uint32_t p;
            if constexpr (TAB == 1) p = lookup_packed(s_tab, ps.lgS, ps.ib, key >> 8);
            else if constexpr (TAB == 3) p = lookup_packed<true>(packed, ps.lgS, ps.ib, key >> 8);
            else if constexpr (TAB == 4) p = lookup_wide(packed, ps.lgS, key >> 8, ps.hmask);
            else if constexpr (TAB == 5) p = lookup_rank(packed, (uint32_t)(key >> 8));
            else p = prefix_lookup(ps.hkeys, ps.hidx, ps.S, ps.lgS, 0, key >> 8, ps.hmask);
            if (p != 0xffffffffu) {
              count_one<CT>(p * 256 + (uint32_t)(key & 0xff), tag, hcnt, table);
              hm |= 1u << T;
            }
          }
        }
      });
      if (KIND == 1 && ps.hit_out != nullptr) __stcs(ps.hit_out + t * 32 + lane, (uint16_t)hm);
      if (tn >= c.ntiles) break;
      t = tn;
      v = vn;
      h = hn;
      d = dn;
      mk = mkn;
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kHotSlots; i += blockDim.x)
    if (tag[i] != kNoId && hcnt[i]) atomicAdd(table + tag[i], (CT)hcnt[i]);
}

// Copies between device memory and mapped pinned host memory with SM loads
// and stores (zero-copy): the session's small transfers then never queue
// behind a large DMA (another session's corpus upload) in a copy engine.
__global__ void k_copy_bytes(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                             uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const uint64_t n16 = n / 16;
    for (uint64_t i = i0; i < n16; i += stride)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (uint64_t i = n16 * 16 + i0; i < n; i += stride) dst[i] = src[i];
  } else {
    for (uint64_t i = i0; i < n; i += stride) dst[i] = src[i];
  }
}

void launch_copy(void* dst, const void* src, uint64_t n, cudaStream_t st) {
  if (!n) return;
  const uint64_t blocks = std::min<uint64_t>((n / 16 + 255) / 256 + 1, 1024);
  k_copy_bytes<<<(unsigned)blocks, 256, 0, st>>>(static_cast<uint8_t*>(dst),
                                                 static_cast<const uint8_t*>(src), n);
}

// table64[i] += scratch32[i] (count-all segments of < 2^32 positions).
__global__ void k_widen_add(const uint32_t* __restrict__ src, unsigned long long* __restrict__ dst,
                            uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(src)[i];
    ulonglong2* d = reinterpret_cast<ulonglong2*>(dst) + 2 * i;
    ulonglong2 a = d[0], b = d[1];
    a.x += v.x;
    a.y += v.y;
    b.x += v.z;
    b.y += v.w;
    d[0] = a;
    d[1] = b;
  }
}

void launch_widen_add(const uint32_t* src, unsigned long long* dst, uint64_t n, int num_sms,
                      cudaStream_t st) {
  const uint64_t n4 = n / 4;  // table capacities are multiples of 256
  if (!n4) return;
  const unsigned blocks = (unsigned)std::min<uint64_t>((n4 + 255) / 256, (uint64_t)num_sms * 16);
  k_widen_add<<<blocks, 256, 0, st>>>(src, dst, n4);
}

// Narrowed all-reduce of a u64 table: the largest entry, the
// u64 -> u32 narrowing and the widening back (n % 4 == 0).
__global__ void k_max_u64(const unsigned long long* __restrict__ t, uint64_t n,
                          unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, t[i]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void k_narrow_u64(const unsigned long long* __restrict__ src, uint32_t* __restrict__ dst,
                             uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = reinterpret_cast<const ulonglong2*>(src)[2 * i];
    const ulonglong2 b = reinterpret_cast<const ulonglong2*>(src)[2 * i + 1];
    reinterpret_cast<uint4*>(dst)[i] =
        make_uint4((uint32_t)a.x, (uint32_t)a.y, (uint32_t)b.x, (uint32_t)b.y);
  }
}

__global__ void k_widen_set(const uint32_t* __restrict__ src, unsigned long long* __restrict__ dst,
                            uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(src)[i];
    reinterpret_cast<ulonglong2*>(dst)[2 * i] = make_ulonglong2(v.x, v.y);
    reinterpret_cast<ulonglong2*>(dst)[2 * i + 1] = make_ulonglong2(v.z, v.w);
  }
}

void launch_max_u64(const unsigned long long* t, uint64_t n, unsigned long long* out,
                    int num_sms, cudaStream_t st) {
  IGB_CUDA(cudaMemsetAsync(out, 0, sizeof(*out), st));
  if (!n) return;
  const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 8);
  k_max_u64<<<blocks, 256, 0, st>>>(t, n, out);
}

void launch_narrow_u64(const unsigned long long* src, uint32_t* dst, uint64_t n, int num_sms,
                      cudaStream_t st) {
  const uint64_t n4 = n / 4;
  if (!n4) return;
  const unsigned blocks = (unsigned)std::min<uint64_t>((n4 + 255) / 256, (uint64_t)num_sms * 16);
  k_narrow_u64<<<blocks, 256, 0, st>>>(src, dst, n4);
}

void launch_widen_set(const uint32_t* src, unsigned long long* dst, uint64_t n, int num_sms,
                      cudaStream_t st) {
  const uint64_t n4 = n / 4;
  if (!n4) return;
  const unsigned blocks = (unsigned)std::min<uint64_t>((n4 + 255) / 256, (uint64_t)num_sms * 16);
  k_widen_set<<<blocks, 256, 0, st>>>(src, dst, n4);
}

// ------------------------------------------------------------------ launchers

template <int KIND, int L, typename CT>
static void launch_all_t(const DevCorpus& c, const DevPrefixSet& ps, CT* table, int num_sms,
                         cudaStream_t st) {
  if (c.ntiles <= c.tile0) return;
  const int threads = 512;
  const uint64_t want = ((c.ntiles - c.tile0 + c.tstride - 1) / c.tstride * 32 + threads - 1) / threads;
  auto go = [&](auto kern, size_t smem, const uint64_t* pk) {
    IGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 0;
    IGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem));
    const uint64_t cap = (uint64_t)num_sms * (per > 0 ? per : 1);  // persistent
    unsigned blocks = (unsigned)(want < cap ? want : cap);
    if (!blocks) blocks = 1;
    kern<<<blocks, threads, smem, st>>>(c, ps, pk, table);
  };
  if constexpr (KIND == 0) {
    go(k_count_all<0, L, CT, 0, false>, 0, nullptr);
  } else {
    // key and index packed in one 8-byte slot: one load per probe (staged in
    // smem when small); otherwise the key and index arrays (two loads on a hit)
    static const bool no_packed = getenv("IG_NO_PACKED_GLOBAL") != nullptr;
    if constexpr (L == 4) {
      if (ps.rankbits && !no_packed) {
        go(k_count_all<1, L, CT, 5, false>, 0, ps.rankbits);
        return;
      }
    }
    if (ps.packed && (size_t)ps.S * 8 <= 64 * 1024) go(k_count_all<1, L, CT, 1, false>, ps.S * 8, ps.packed);
    else if (ps.packed && !no_packed) go(k_count_all<1, L, CT, 3, false>, 0, ps.packed);
    else if (ps.wide && !no_packed) go(k_count_all<1, L, CT, 4, false>, 0, ps.wide);
    else go(k_count_all<1, L, CT, 2, false>, 0, nullptr);
  }
}

template <typename CT>
void launch_count_dense(const DevCorpus& c, uint32_t n0, int mode, CT* table, uint32_t* /*work*/,
                        int num_sms, cudaStream_t st) {
  DevPrefixSet none{};
  if (mode == IG_MODE_ALL) {
    switch (n0) {
      case 1: launch_all_t<0, 1, CT>(c, none, table, num_sms, st); break;
      case 2: launch_all_t<0, 2, CT>(c, none, table, num_sms, st); break;
      default: launch_all_t<0, 3, CT>(c, none, table, num_sms, st); break;
    }
  } else {
    // count-once counts through the route path (route_kernels.cu)
    throw Error(IG_EINTERNAL, "count_dense kernel is count-all only");
  }
}

template <typename CT>
void launch_count_extend(const DevCorpus& c, const DevPrefixSet& ps, uint32_t j, int mode,
                         CT* table, uint32_t* /*work*/, int num_sms, cudaStream_t st) {
  if (mode != IG_MODE_ALL) throw Error(IG_EINTERNAL, "count_extend kernel is count-all only");
#define IGB_J(J)                                             \
  case J:                                                    \
    launch_all_t<1, J, CT>(c, ps, table, num_sms, st);       \
    break;
  switch (j) {
    IGB_J(2) IGB_J(3) IGB_J(4) IGB_J(5) IGB_J(6) IGB_J(7) IGB_J(8)
    default: throw Error(IG_ECONFIG, "gram length above 8 is not supported");
  }
#undef IGB_J
}

template void launch_count_dense<uint32_t>(const DevCorpus&, uint32_t, int, uint32_t*, uint32_t*,
                                           int, cudaStream_t);
template void launch_count_dense<unsigned long long>(const DevCorpus&, uint32_t, int,
                                                     unsigned long long*, uint32_t*, int,
                                                     cudaStream_t);
template void launch_count_extend<uint32_t>(const DevCorpus&, const DevPrefixSet&, uint32_t, int,
                                            uint32_t*, uint32_t*, int, cudaStream_t);
template void launch_count_extend<unsigned long long>(const DevCorpus&, const DevPrefixSet&,
                                                      uint32_t, int, unsigned long long*,
                                                      uint32_t*, int, cudaStream_t);

// ------------------------------------------------------------------ prefix set build

// Survivor keys in ascending key order with their selection ranks (count-all
// prefix numbering p = rank in key order: deterministic on every GPU, and the
// slices of a hot-gram sweep are then contiguous p ranges).
__global__ void k_iota(uint32_t* __restrict__ v, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[i] = i;
}

void sort_keys_by_value(const uint64_t* keys, uint32_t K, uint32_t key_bits, uint64_t* out_keys,
                        uint32_t* out_ranks, uint32_t* tmp_ranks, DevBuf& tmp, cudaStream_t st) {
  if (!K) return;
  k_iota<<<std::min(4096u, (K + 255) / 256), 256, 0, st>>>(tmp_ranks, K);
  size_t bytes = 0;
  IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, out_keys, tmp_ranks, out_ranks,
                                           (int)K, 0, (int)key_bits, st));
  void* t = tmp.get(bytes);
  IGB_CUDA(cub::DeviceRadixSort::SortPairs(t, bytes, keys, out_keys, tmp_ranks, out_ranks, (int)K,
                                           0, (int)key_bits, st));
}

// bounds[s] = pkeys[K * s / S] (s in 1..S-1), bounds[0] = 0, bounds[S] = ~0.
__global__ void k_slice_bounds(const uint64_t* __restrict__ pkeys, uint32_t K, uint32_t S,
                               uint64_t* __restrict__ bounds) {
  const uint32_t s = threadIdx.x;
  if (s > S) return;
  bounds[s] = s == 0 ? 0ull : (s == S ? ~0ull : pkeys[(uint64_t)K * s / S]);
}

void launch_slice_bounds(const uint64_t* pkeys, uint32_t K, uint32_t S, uint64_t* bounds,
                         cudaStream_t st) {
  k_slice_bounds<<<1, 32, 0, st>>>(pkeys, K, S, bounds);
}

// Pass 1: owner of every survivor key and per-owner sizes.
__global__ void k_prefix_owner(const uint64_t* __restrict__ keys, uint32_t K, uint32_t plen,
                               uint32_t G, uint32_t* __restrict__ owner,
                               uint32_t* __restrict__ owner_count) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) {
    const uint32_t o = prefix_owner(keys[i], plen, G);
    owner[i] = o;
    atomicAdd(owner_count + o, 1u);
  }
}

// Pass 2: place survivor i at p = owner_start[o] + cursor (order inside a
// slice is irrelevant to results: selection orders by gram key), and insert it
// into owner o's open-addressing slice.
__global__ void k_prefix_insert(const uint64_t* __restrict__ keys, uint32_t K,
                                const uint32_t* __restrict__ owner,
                                const uint32_t* __restrict__ owner_start,
                                uint32_t* __restrict__ cursor, uint32_t S, uint32_t lgS,
                                uint64_t* __restrict__ hkeys, uint32_t* __restrict__ hidx,
                                uint64_t* __restrict__ pkeys, uint32_t* __restrict__ rank_of_p,
                                bool S_single, const uint32_t* __restrict__ ranks,
                                uint32_t hmask) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) {
    const uint32_t o = owner[i];
    // single slice (count-all): p = rank, identical on every rank of a
    // multi-GPU run so per-rank tables can be summed element-wise
    const uint32_t p = S_single ? i : owner_start[o] + atomicAdd(cursor + o, 1u);
    const uint64_t key = keys[i];
    pkeys[p] = key;
    rank_of_p[p] = ranks ? ranks[i] : i;
    unsigned long long* kk = reinterpret_cast<unsigned long long*>(hkeys + (size_t)o * S);
    uint32_t h = hash_slot(key, lgS, hmask);
    for (;;) {
      const unsigned long long prev = atomicCAS(kk + h, (unsigned long long)kEmptyKey,
                                                (unsigned long long)key);
      if (prev == kEmptyKey) {
        hidx[(size_t)o * S + h] = p;
        break;
      }
      h = (h + 1) & (S - 1);
    }
  }
}

void launch_prefix_owner(const uint64_t* keys, uint32_t K, uint32_t plen, uint32_t G,
                         uint32_t* owner, uint32_t* owner_count, cudaStream_t st) {
  if (!K) return;
  const unsigned blocks = (K + 255) / 256;
  k_prefix_owner<<<blocks < 4096 ? blocks : 4096, 256, 0, st>>>(keys, K, plen, G, owner,
                                                               owner_count);
}

void launch_prefix_insert(const uint64_t* keys, uint32_t K, const uint32_t* owner,
                          const uint32_t* owner_start, uint32_t* cursor, uint32_t S, uint32_t lgS,
                          uint64_t* hkeys, uint32_t* hidx, uint64_t* pkeys, uint32_t* rank_of_p,
                          cudaStream_t st, const uint32_t* ranks, uint32_t hmask) {
  if (!K) return;
  const unsigned blocks = (K + 255) / 256;
  k_prefix_insert<<<blocks < 4096 ? blocks : 4096, 256, 0, st>>>(
      keys, K, owner, owner_start, cursor, S, lgS, hkeys, hidx, pkeys, rank_of_p,
      owner_start == nullptr, ranks, hmask);
}

}  // namespace igb
