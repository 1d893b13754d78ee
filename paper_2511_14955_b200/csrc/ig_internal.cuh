// ig_internal.cuh — shared internals of the B200 Intergrams library.
//
// Layout in HBM (one session = one device):
//   corpus   d_data  : u8[total + pad], 16 B of zero front padding so a segment's
//                       8-byte halo load at base-8 never leaves the allocation
//            d_off   : u64[m+1] sequence offsets (CSR)
//            d_tile  : u32[ceil(total/512)] sequence index of each 512-byte tile
//            d_order : u32[m] sequences by length, longest first (count-once LPT)
//   tables   counts  : CT[capacity] (u32 when every count provably fits, else u64)
//   prefixes pkeys   : u64[K]   survivor keys in bucket order (p = index)
//            hkeys   : u64[G*S] open-addressing prefix set, G owner slices
//            hidx    : u32[G*S] p of each occupied slot
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/intergrams_b200.h"

namespace igb {

// Exceptions carried to the C boundary and turned into IG_* codes there.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    throw Error(IG_EINTERNAL, std::string("CUDA error in ") + what + " at " + file + ":" +
                                  std::to_string(line) + ": " + cudaGetErrorString(e));
  }
}
#define IGB_CUDA(x) ::igb::cuda_check((x), #x, __FILE__, __LINE__)
#define IGB_LAUNCHED(sess) \
  do {                     \
    (sess)->launches++;    \
    IGB_CUDA(cudaGetLastError()); \
  } while (0)

constexpr uint64_t kEmptyKey = ~0ull;
constexpr uint64_t kCuckooMul1 = 0x9E3779B97F4A7C15ull;  // prefix-set hashes
constexpr uint64_t kCuckooMul2 = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t kOwnerMul = 0xD6E8FEB86659FD93ull;    // count-once owner of a prefix  // never a key: keys have <= 56 bits in a prefix set
constexpr uint32_t kOwnerMul32 = 0x9E3779B1u;       // ... of a prefix of <= 4 bytes
constexpr uint32_t kNarrowMul1 = 0x85EBCA6Bu;       // perfect-hash hashes of <= 4-byte keys
constexpr uint32_t kNarrowMul2 = 0xC2B2AE35u;
constexpr uint32_t kNarrowMul3 = 0x27D4EB2Fu;
constexpr int kTileBytes = 512;        // one warp x 16 B per lane
constexpr int kFrontPad = 16;
constexpr int kBackPad = 1024;
constexpr size_t kMaxOnceSmem = 227 * 1024;  // dynamic smem per CTA (sm_100a)

// Guarded allocation (IG_GUARD=1; the stand-in for compute-sanitizer, which
// this GPU pool does not allow): every DevBuf gets kGuardBytes of 0xA5 in
// front of and behind its bytes, and check_guards() (after every run / load /
// exact call in this mode) throws when a kernel wrote into one.
constexpr size_t kGuardBytes = 4096;
struct DevBuf;
inline bool guard_mode() {
  static const bool g = getenv("IG_GUARD") != nullptr;
  return g;
}
struct GuardRegistry {
  std::mutex mu;
  std::set<DevBuf*> live;
  static GuardRegistry& get() {
    static GuardRegistry* r = new GuardRegistry();  // outlives every DevBuf
    return *r;
  }
};

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* base = nullptr;  // allocation start (p - kGuardBytes in guard mode)
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void swap(DevBuf& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    std::swap(base, o.base);
  }
  void release() {
    if (base) cudaFree(base);
    if (base && guard_mode()) {
      std::lock_guard<std::mutex> lk(GuardRegistry::get().mu);
      GuardRegistry::get().live.erase(this);
    }
    p = base = nullptr;
    bytes = 0;
  }
  void* get(size_t need) {
    if (need > bytes) {
      release();
      const size_t n = need ? need : 16;
      if (guard_mode()) {
        IGB_CUDA(cudaMalloc(&base, n + 2 * kGuardBytes));
        IGB_CUDA(cudaMemset(base, 0xA5, kGuardBytes));
        IGB_CUDA(cudaMemset(static_cast<char*>(base) + kGuardBytes + n, 0xA5, kGuardBytes));
        p = static_cast<char*>(base) + kGuardBytes;
        std::lock_guard<std::mutex> lk(GuardRegistry::get().mu);
        GuardRegistry::get().live.insert(this);
      } else {
        IGB_CUDA(cudaMalloc(&base, n));
        p = base;
      }
      bytes = n;
    }
    return p;
  }
  template <typename T>
  T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
  ~DevBuf() { release(); }
};

// Throws when any live guarded buffer's guard bytes changed (a device write
// out of bounds).  Synchronises the device.  No-op unless IG_GUARD is set.
inline void check_guards(const char* where) {
  if (!guard_mode()) return;
  IGB_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(GuardRegistry::get().mu);
  std::vector<unsigned char> h(kGuardBytes);
  for (DevBuf* b : GuardRegistry::get().live) {
    for (int side = 0; side < 2; ++side) {
      const char* g = side == 0 ? static_cast<const char*>(b->base)
                                : static_cast<const char*>(b->p) + b->bytes;
      IGB_CUDA(cudaMemcpy(h.data(), g, kGuardBytes, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < kGuardBytes; ++i)
        if (h[i] != 0xA5)
          throw Error(IG_EINTERNAL, std::string("guard bytes overwritten ") +
                                        (side ? "behind" : "in front of") + " a device buffer of " +
                                        std::to_string(b->bytes) + " bytes (" + where + ", offset " +
                                        std::to_string(i) + ")");
    }
  }
}

// Grow-only mapped pinned host staging.  Every small host<->device transfer
// of a run goes through it and is moved by a kernel (zero-copy), not a copy
// engine: a DMA queues behind any large copy already in flight (another
// session's corpus upload) and would serialise the run with that upload.
// Chunks are reused after reset() (called when the stream is idle).
struct PinnedArena {
  std::vector<std::pair<char*, size_t>> chunks;
  size_t chunk = 0, used = 0;
  void* get(size_t n) {
    n = (n + 15) & ~size_t(15);
    while (chunk < chunks.size() && used + n > chunks[chunk].second) {
      ++chunk;
      used = 0;
    }
    if (chunk == chunks.size()) {
      const size_t sz = std::max<size_t>(n, 16u << 20);
      void* p = nullptr;
      IGB_CUDA(cudaHostAlloc(&p, sz, cudaHostAllocMapped));
      chunks.emplace_back(static_cast<char*>(p), sz);
      used = 0;
    }
    void* r = chunks[chunk].first + used;
    used += n;
    return r;
  }
  void reset() {
    chunk = 0;
    used = 0;
  }
  PinnedArena() = default;
  PinnedArena(const PinnedArena&) = delete;
  PinnedArena& operator=(const PinnedArena&) = delete;
  ~PinnedArena() {
    for (auto& c : chunks) cudaFreeHost(c.first);
  }
};

// Optional per-kernel-family device timing (CUDA events on the launching
// stream), for the roofline numbers.  Families: see IG_KF_* in the C header.
struct KernelTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, size_t>> pending;  // family, index of the begin event
  size_t used = 0;
  double ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  size_t begin(int fam, cudaStream_t st) {
    if (!on) return 0;
    while (used + 2 > pool.size()) {
      cudaEvent_t e;
      IGB_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    IGB_CUDA(cudaEventRecord(pool[used], st));
    pending.emplace_back(fam, used);
    used += 2;
    return used - 2;
  }
  void end(size_t i, cudaStream_t st) {
    if (on) IGB_CUDA(cudaEventRecord(pool[i + 1], st));
  }
  void collect() {  // after a stream sync
    for (auto& p : pending) {
      float t = 0;
      IGB_CUDA(cudaEventElapsedTime(&t, pool[p.second], pool[p.second + 1]));
      ms[p.first] += t;
      n[p.first] += 1;
    }
    pending.clear();
    used = 0;
  }
  void reset() {
    for (int i = 0; i < 8; ++i) {
      ms[i] = 0;
      n[i] = 0;
    }
  }
  ~KernelTimer() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// Device-side corpus view.
struct DevCorpus {
  const uint8_t* data = nullptr;  // first byte of sequence 0
  const uint64_t* off = nullptr;  // m+1
  const uint32_t* tile_seq = nullptr;
  const uint32_t* order = nullptr;
  uint64_t m = 0;
  uint64_t total = 0;      // bytes
  uint64_t ntiles = 0;     // tiles [tile0, ntiles) are counted by count-all kernels
  uint64_t tile0 = 0;
  uint32_t tstride = 1;    // count-all: visit tiles tile0, tile0 + tstride, ... (sampling)
};

// Device prefix set for an extension pass.
struct DevPrefixSet {
  const uint64_t* pkeys = nullptr;   // [K] keys by p
  const uint64_t* hkeys = nullptr;   // [G*S]
  const uint32_t* hidx = nullptr;    // [G*S]
  const uint32_t* owner_start = nullptr;  // [G+1] p range of each owner slice
  uint32_t K = 0;
  uint32_t G = 1, lgG = 0;
  uint32_t S = 0;          // slots per owner slice (power of two)
  uint32_t lgS = 0;
  uint32_t plen = 0;       // prefix length (j-1)
  uint32_t max_owner = 0;  // largest owner slice size
  uint32_t ib = 0;         // local-index bits of a packed entry
  uint32_t hmask = ~3u;    // home alignment of the open-addressing slots (hash_slot)
  const uint64_t* packed = nullptr;  // [G*S] (key << ib) | local, or null
  const uint64_t* wide = nullptr;    // [2*S] {key, p} slots (G == 1), or null
  // 3-byte prefixes (the first extension pass): {bits, rank} pairs over the
  // 2^24 prefix space, p = rank of the prefix in key order (pkeys sorted), or null
  const uint64_t* rankbits = nullptr;  // [2 * 2^18]
  // count-all hit chaining: one u16 per 16-byte segment
  // (index = tile * 32 + lane), bit T = the gram ending at byte 16*index + T
  // was counted by the pass that wrote it.  hit_in[-1] is readable (zero).
  const uint16_t* hit_in = nullptr;  // previous extension pass's hits, or null
  uint16_t* hit_out = nullptr;       // this pass's hits (read by the next pass), or null
  // hot sweeps (hot_kernels.cu): the previous pass hit fewer than half of the
  // positions, so this one takes the sparse kernel (mask-gated corpus loads,
  // dead tiles skipped, sparse tiles walked live position by live position)
  bool sparse = false;
};

// Home slot of a key in an open-addressing table of 2^lgS slots: always a
// multiple of 4, so a probe can read whole 4-slot (32-byte) buckets while a
// slot-by-slot linear probe from the same home stays valid.
// hmask: ~3u (4-aligned homes: packed 8-byte slots, a 32-byte bucket holds 4)
// or ~1u (2-aligned: {key, p} 16-byte slots, a 32-byte bucket holds 2).
__host__ __device__ inline uint32_t hash_slot(uint64_t key, uint32_t lgS, uint32_t hmask = ~3u) {
  return lgS <= 2 ? 0u : (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - lgS)) & hmask;
}

// Owner slice of a prefix key (count-once passes): first byte xor last byte.
__host__ __device__ inline uint32_t prefix_owner(uint64_t key, uint32_t plen, uint32_t G) {
  uint32_t last = (uint32_t)(key & 0xff);
  uint32_t first = (uint32_t)((key >> (8 * (plen - 1))) & 0xff);
  uint32_t x = plen >= 2 ? (first ^ last) : last;
  return x & (G - 1);
}

// Owner slice of a count-once extension prefix of plen bytes (host and
// device agree on it): multiplicative hash (top bits of key * odd constant,
// in 32-bit arithmetic for prefixes of <= 4 bytes).
__host__ __device__ inline uint32_t owner_hash(uint64_t pkey, uint32_t plen, uint32_t lgno) {
#ifdef __CUDA_ARCH__
  if (plen <= 4)  // clamped funnel shift: a shift by 32 (lgno == 0) gives owner 0
    return __funnelshift_rc((uint32_t)pkey * kOwnerMul32, 0u, 32 - lgno);
#else
  if (plen <= 4) return (uint32_t)((uint64_t)((uint32_t)pkey * kOwnerMul32) >> (32 - lgno));
#endif
  return lgno ? (uint32_t)((pkey * kOwnerMul) >> (64 - lgno)) : 0u;
}

// Predicated shared-memory operations.  `if (p) atomicAdd(smem, 1)` compiles
// to a branch around the ATOMS (BSSY/BRA/BSYNC, ~7 issue slots); these emit
// a single predicated instruction instead.
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// The same, on 32-bit shared-window addresses (base converted once per
// kernel: the generic->shared conversion is not free per access).
__device__ __forceinline__ void red_inc_shared_at(bool p, uint32_t sa) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q red.shared.add.u32 [%1], 1;\n}"
               :: "r"((uint32_t)p), "r"(sa) : "memory");
}
__device__ __forceinline__ uint32_t atom_inc_shared_at(bool p, uint32_t sa) {
  uint32_t old = 0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %1, 0;\n @q atom.shared.add.u32 %0, [%2], 1;\n}"
               : "+r"(old) : "r"((uint32_t)p), "r"(sa) : "memory");
  return old;
}
__device__ __forceinline__ void st_shared_u32_at(bool p, uint32_t sa, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.u32 [%1], %2;\n}"
               :: "r"((uint32_t)p), "r"(sa), "r"(v) : "memory");
}
__device__ __forceinline__ void st_shared_u64_at(bool p, uint32_t sa, uint64_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.u64 [%1], %2;\n}"
               :: "r"((uint32_t)p), "r"(sa), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_shared_if(bool p, const uint32_t* a, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q red.shared.add.u32 [%1], %2;\n}"
               :: "r"((uint32_t)p), "r"(smem_u32(a)), "r"(v) : "memory");
}
__device__ __forceinline__ void red_inc_shared_if(bool p, const uint32_t* a) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q red.shared.add.u32 [%1], 1;\n}"
               :: "r"((uint32_t)p), "r"(smem_u32(a)) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_shared_if(bool p, const uint32_t* a, uint32_t v) {
  uint32_t old = 0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %1, 0;\n @q atom.shared.add.u32 %0, [%2], %3;\n}"
               : "+r"(old) : "r"((uint32_t)p), "r"(smem_u32(a)), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_or_shared_if(bool p, const uint32_t* a, uint32_t v) {
  uint32_t old = 0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %1, 0;\n @q atom.shared.or.b32 %0, [%2], %3;\n}"
               : "+r"(old) : "r"((uint32_t)p), "r"(smem_u32(a)), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_shared_u32_if(bool p, const uint32_t* a, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.u32 [%1], %2;\n}"
               :: "r"((uint32_t)p), "r"(smem_u32(a)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_shared_u64_if(bool p, const uint64_t* a, uint64_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.u64 [%1], %2;\n}"
               :: "r"((uint32_t)p), "r"(smem_u32(a)), "l"(v) : "memory");
}
#endif

// Session (the C handle).
struct Session;

}  // namespace igb
