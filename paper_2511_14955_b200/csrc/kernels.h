// kernels.h — host-side launchers of the sm_100a kernels (one translation
// unit per family: count_kernels.cu, select_kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "ig_internal.cuh"

namespace igb {

// --- corpus / counting (count_kernels.cu)
void launch_tile_seq(const uint64_t* off, uint64_t m, uint64_t ntiles, uint32_t* tile_seq,
                     cudaStream_t st);

template <typename CT>
void launch_count_dense(const DevCorpus& c, uint32_t n0, int mode, CT* table, uint32_t* work,
                        int num_sms, cudaStream_t st);

template <typename CT>
void launch_count_extend(const DevCorpus& c, const DevPrefixSet& ps, uint32_t j, int mode,
                         CT* table, uint32_t* work, int num_sms, cudaStream_t st);

void launch_prefix_owner(const uint64_t* keys, uint32_t K, uint32_t plen, uint32_t G,
                         uint32_t* owner, uint32_t* owner_count, cudaStream_t st);
void launch_prefix_insert(const uint64_t* keys, uint32_t K, const uint32_t* owner,
                          const uint32_t* owner_start, uint32_t* cursor, uint32_t S, uint32_t lgS,
                          uint64_t* hkeys, uint32_t* hidx, uint64_t* pkeys, uint32_t* rank_of_p,
                          cudaStream_t st, const uint32_t* ranks = nullptr,
                          uint32_t hmask = ~3u);
// keys[0..K) ascending (key_bits significant bits) with their input indices
void sort_keys_by_value(const uint64_t* keys, uint32_t K, uint32_t key_bits, uint64_t* out_keys,
                        uint32_t* out_ranks, uint32_t* tmp_ranks, DevBuf& tmp, cudaStream_t st);
// bounds[0..S]: 0, pkeys[K*s/S] for 0 < s < S, ~0
void launch_slice_bounds(const uint64_t* pkeys, uint32_t K, uint32_t S, uint64_t* bounds,
                         cudaStream_t st);

void launch_widen_add(const uint32_t* src, unsigned long long* dst, uint64_t n, int num_sms,
                      cudaStream_t st);
// narrowed all-reduce of u64 tables (n % 4 == 0)
void launch_max_u64(const unsigned long long* t, uint64_t n, unsigned long long* out,
                    int num_sms, cudaStream_t st);
void launch_narrow_u64(const unsigned long long* src, uint32_t* dst, uint64_t n, int num_sms,
                       cudaStream_t st);
void launch_widen_set(const uint32_t* src, unsigned long long* dst, uint64_t n, int num_sms,
                      cudaStream_t st);
// SM copy to/from mapped pinned host memory (no copy engine)
void launch_copy(void* dst, const void* src, uint64_t n, cudaStream_t st);
void launch_pack_prefix(const DevPrefixSet& ps, uint64_t* packed, cudaStream_t st);
// {key, index} 16-byte slots (prefixes too long for the packed 8-byte slot)
void launch_pack_wide(const DevPrefixSet& ps, uint64_t* wide, cudaStream_t st);
// Rank bitmap of K distinct 3-byte prefixes (rankbits: 2^19 u64, {bits, rank}
// pairs): p = rank in key order; writes pkeys[p] = key, rank_of_p[p] = i.
void launch_rank_prefix(const uint64_t* keys, uint32_t K, uint64_t* rankbits, uint64_t* pkeys,
                        uint32_t* rank_of_p, cudaStream_t st);

// --- count-all with sampled hot-gram tables (hot_kernels.cu)
constexpr uint32_t kHotSampleStrideMin = 16, kHotSampleStrideMax = 256;  // sample tiles: t % stride == 0
constexpr int kMaxHotSlices = 8;
// Slices of a pass table's id range: slice s = ids [lo[s], lo[s+1]).
struct HotSliceIds {
  uint32_t S = 1;
  uint64_t lo[kMaxHotSlices] = {};
};
// Per slice: 2^lgnb two-way buckets of gram keys and their table ids.
struct HotSet {
  uint32_t S = 1, lgnb = 0;
  // direct: a key may only sit in way (next hash bit) of its bucket, i.e. the
  // table is 2 << lgnb direct-mapped slots (the queued sweep reads one slot);
  // two-way lookups still find every key
  bool direct = false;
  // direct: device count of important candidates (sample count >= the
  // builder's `important`) that lost their slot; the caller rebuilds two-way
  // when it is not zero
  uint32_t* lost = nullptr;
  uint32_t mul = 0x9E3779B1u;  // the table's multiplier of the low key word (hot_bucket)
  uint64_t* keys = nullptr;  // [S][2 << lgnb]
  uint32_t* ids = nullptr;   // [S][2 << lgnb] (~0u: empty slot)
};
// One sweep (one slice): its bucket keys/ids, the slice's key range
// bounds[0] <= key < bounds[1] (the prefix key for extension passes, the
// gram for the dense pass), and whether this is the first slice (it writes
// every hit-mask word; later ones OR).
struct HotSweep {
  const uint64_t* keys = nullptr;
  const uint32_t* ids = nullptr;
  uint32_t lgnb = 0;
  const uint64_t* bounds = nullptr;  // device, 2 values
  bool first = true;
  bool sliced = false;  // more than one slice: check the key range
  // queued extension sweep: a tile whose lanes hold at most this many live
  // positions each is walked live position by live position (0: never)
  uint32_t sparse_iters = 10;
  bool direct = false;  // HotSet::direct
  uint32_t mul = 0x9E3779B1u;  // HotSet::mul
};
// Whether this pass's sweep reads a direct table: the queued extension sweep
// (launch_count_hot takes it exactly then) and the one-slice dense sweep.
bool hot_sweep_queued(const DevPrefixSet& ps, bool dense, uint32_t L, bool sliced);
size_t hot_smem(uint32_t lgnb);
// Hot set of each slice from the (sample) counts in table[0, cap).  pkeys:
// gram key of id = (pkeys[id >> 8] << 8) | (id & 255), or null (key = id).
template <typename CT>
void build_hot_set(const CT* table, uint64_t cap, const HotSliceIds& sl, const uint64_t* pkeys,
                   uint32_t lgnb, HotSet& hs, DevBuf& work, int num_sms, cudaStream_t st,
                   bool direct = false, uint64_t important = ~0ull, uint32_t mul = 0x9E3779B1u);
template <typename CT, typename CC>
void launch_count_hot(const DevCorpus& c, const DevPrefixSet& ps, bool dense, uint32_t L,
                      const HotSweep& hw, CT* table, CC* cold, int num_sms, cudaStream_t st);

// --- count-once route-then-count (route_kernels.cu)
struct RouteUnit {  // <= 1 MiB of gram ends of one sequence: byte range [b0, b1)
  uint32_t q;
  uint32_t pad;
  uint64_t b0, b1;
};

struct RouteView {
  const RouteUnit* units;
  const uint32_t* unit_first;  // [m+1] first unit of each sequence
  uint32_t nunits;             // all units (layout of fused next-pass counts)
  uint32_t u0, nb;             // units [u0, u0+nb) of this launch
  uint32_t q0, q1;             // their sequences [q0, q1)
};

struct RouteParams {
  uint32_t lgc = 2, lgl = 2, NO = 1;  // dense: permuted id space 2^lgc; 2^lgl ids per owner
  uint64_t cmask = 3, mult = 1, minv = 1;
  // extension passes: owner = hash(prefix) >> (64-lgno); p numbered owner by
  // owner (ostart[o] .. ostart[o+1]); CHD perfect-hash prefix set
  bool ext = false;
  bool dedup = true;    // scatter drops repeats inside a chunk (optimisation only)
  uint32_t lgno = 0;
  uint32_t nb = 0, nslots = 0;         // perfect-hash buckets / slots
  const uint64_t* slots = nullptr;     // [nslots]
  const uint16_t* disp = nullptr;      // [nb]
  const uint32_t* ostart = nullptr;
  // fused count of the NEXT pass (owner = hash(this pass's gram) >> (64 - next_lgno));
  // -1: not requested
  int32_t next_lgno = -1;
  uint32_t* next_cnt = nullptr;
};

struct RouteCtx {
  const RouteUnit* units = nullptr;
  const uint32_t* unit_first = nullptr;
  uint32_t nunits = 0;
  DevBuf cnt, actual, base, entries, cub_tmp, cnt_next;
  DevBuf consume_order;  // consume: owners heaviest first + the work counter
  uint64_t launches = 0;
  KernelTimer* kt = nullptr;
  bool have_next = false;   // cnt_next holds the next pass's counts (fused in the scatter)
  int32_t next_lgno = -1;
  // range of the current launch (whole corpus unless a pipelined load batches it)
  uint32_t u0 = 0, u1 = 0, q0 = 0, q1 = 0;
  RouteView view() const { return RouteView{units, unit_first, nunits, u0, u1 - u0, q0, q1}; }
};

void make_route_params(uint64_t cap, RouteParams& rp);
// narrow: keys of <= 4 bytes (32-bit hashes, (key << 32) | v slots)
void build_prefix_mphf(const std::vector<uint64_t>& keys, bool narrow,
                       std::vector<uint32_t>& slot_of_key, std::vector<uint16_t>& disp,
                       uint32_t& nb, uint32_t& nslots);
// stage 1: count + scan (owner function only); stage 2: scatter + consume.
template <typename CT>
void route_count_once(int stage, RouteCtx& x, const DevCorpus& c, int kind, uint32_t L,
                      const RouteParams& rp, CT* table, int num_sms, cudaStream_t st);

// Count-once over short sequences (no routing): sw / sc list the sequences
// of <= kShortWarpLen / <= kShortCtaLen gram ends (a warp / a CTA each).
constexpr int kShortWarpLen = 512;
constexpr int kShortCtaLen = 8192;
template <typename CT>
void count_once_short(int kind, uint32_t L, const DevCorpus& c, const RouteParams& rp,
                      const uint32_t* sw, uint32_t nw, const uint32_t* sc, uint32_t nc, CT* table,
                      int num_sms, cudaStream_t st);

// Count-once over a small alphabet (A <= 16 bytes): one CTA per long
// sequence, a shared-memory bitmap over the K * A candidates that can occur
// (DESIGN.md §3.2d).  Adds into table (p * 256 + byte layout).
size_t direct_smem(const RouteParams& rp, uint64_t nbits);
// Work item of the small-alphabet kernels: byte range `part` of `nparts`
// equal ranges of long sequence q.  A split sequence (nparts > 1) ORs each
// part's bitmap into global slot `slot`; the last part to finish counts the
// union once (so a corpus of a few long sequences still fills every SM).
struct DirectItem {
  uint32_t q, part, nparts, slot;
};
struct DirectWork {
  const DirectItem* items = nullptr;
  uint32_t nitems = 0;
  uint32_t nsplit = 0;       // split sequences (global bitmap slots)
  uint32_t* gbm = nullptr;   // [nsplit * nwords] bitmaps, zeroed per launch
  uint32_t* done = nullptr;  // [nsplit] finished parts, zeroed per launch
};
template <typename CT>
void count_once_direct(const DevCorpus& c, uint32_t L, const RouteParams& rp,
                       const DirectWork& w, const uint8_t* arank,
                       const uint8_t* alpha, uint32_t A, uint64_t K, uint32_t* compact, CT* table,
                       int num_sms, cudaStream_t st, const uint16_t* lut = nullptr,
                       uint32_t lut_n = 0, uint32_t bits = 0, bool expand = true);
// 256-bit mask of the bytes of a corpus (mask[0..7]); mask[8] = 1 when the
// scan stopped early at more than 16 distinct bytes (the mask is then partial).
void byte_presence(const uint8_t* data, uint64_t n, uint32_t* mask, int num_sms, cudaStream_t st);
// Dense small-alphabet counts (A^3, mixed radix) added into the permuted dense table.
template <typename CT>
void expand_dense(const uint32_t* compact, uint32_t A, const uint8_t* alpha, uint64_t mult,
                  uint64_t cmask, CT* table, cudaStream_t st);
// 256-bit mask of the bytes in the nonzero entries of a dense n0-gram table.
template <typename CT>
void alphabet_mask(const CT* table, uint64_t cap, uint64_t minv, uint64_t cmask, uint32_t n0,
                   uint32_t* mask, int num_sms, cudaStream_t st);

// --- selection (select_kernels.cu)
struct SelState {
  unsigned long long prefix;   // count digits chosen so far
  unsigned long long r;        // rank still to place among counts
  unsigned long long nonzero;  // nonzero entries (first pass)
  unsigned long long T;        // count threshold
  unsigned long long need;     // entries with count == T to take
  unsigned long long kprefix;  // key digits chosen so far (-> Kt)
  int take_all;
  int pad;
};

struct SelectCtx {
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  SelState* state = nullptr;          // device
  uint32_t* hist = nullptr;           // device [256]
  unsigned long long* scalar = nullptr;  // device
  DevBuf tmp_keys, tmp_counts, cub_tmp;
  uint64_t launches = 0;
  SelState* h_state = nullptr;            // pinned host mirrors (no pageable copies)
  unsigned long long* h_scalar = nullptr;  // mapped pinned: {max, sum}
  unsigned long long last_sum = 0;  // sum of the last selected table's counts
  SelectCtx() = default;
  SelectCtx(const SelectCtx&) = delete;
  SelectCtx& operator=(const SelectCtx&) = delete;
  ~SelectCtx() {
    if (h_state) cudaFreeHost(h_state);
    if (h_scalar) cudaFreeHost(h_scalar);
  }
};

// Canonical top-k of table[0..cap) (cap % 4 == 0).  Gram key = id, or
// (pkeys[id>>8] << 8) | (id & 255) when pkeys != nullptr.  Writes
// min(k, nonzero) entries to out_keys/out_counts (device) and returns that
// number.  key_bits = 8 * gram length.
// Table index -> gram key: id = (index * minv) & cmask (identity when
// minv == 0), then key = id, or (pkeys[id>>8] << 8) | (id & 255).
struct KeyMap {
  const uint64_t* pkeys = nullptr;
  uint64_t minv = 0, cmask = ~0ull;
};

template <typename CT>
uint64_t select_topk(SelectCtx& x, const CT* table, uint64_t cap, uint64_t k, KeyMap km,
                     int key_bits, uint64_t* out_keys, uint64_t* out_counts);

}  // namespace igb
