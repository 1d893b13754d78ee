// session.cu — the Intergrams driver and the C-ABI (include/intergrams_b200.h).
//
// Orchestration follows run_intergrams, proj/src/intergrams.cpp:68-166:
//   validate (:37-42) -> dense n0-gram pass, n0 = min(n,3) (:76-103) ->
//   n <= 3: top-k and return (:105-113) -> top-k' survivors + prefix set
//   (:115-132) -> for j = 4..n: extension pass (:135-141), then top-k'
//   (:143-157) or the final top-k (:158-163).
// PassResult rows, labels and diagnostics are the reference's own; seconds
// are CUDA-event times of each step on the session stream.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include "ig_internal.cuh"
#include "kernels.h"
#include "session.h"

namespace igb {

static constexpr uint64_t kUnitBytes = 4ull << 20;     // count-once work unit
static constexpr uint32_t kPrefixesPerOwner = 64;       // count-once ext: 64*256 ids/owner

// ---------------------------------------------------------------- helpers

void use_device(Session& s) { IGB_CUDA(cudaSetDevice(s.device)); }

void validate(const ig_params& p) {
  // IntergramConfig::validate, intergrams.cpp:37-42
  if (p.n < 1) throw Error(IG_ECONFIG, "gram length n must be >= 1");
  if (p.k < 1) throw Error(IG_ECONFIG, "k must be >= 1");
  if (!(p.z >= 1.0)) throw Error(IG_ECONFIG, "oversample factor z must be >= 1");
  if (p.flush_batch_size < 1) throw Error(IG_ECONFIG, "flush batch size must be >= 1");
  if (p.mode != IG_MODE_ONCE && p.mode != IG_MODE_ALL)
    throw Error(IG_ECONFIG, "count mode must be ONCE (0) or ALL (1)");
}

static uint64_t k_prime(const ig_params& p) {
  // k_prime(), intergrams.hpp:29-31: ceil(z * k)
  // (the reference's size_t cast; saturated where that cast is undefined)
  const double v = std::ceil(p.z * (double)p.k);
  if (v >= 18446744073709551615.0) return ~0ull;
  return (uint64_t)v;
}

// Allocates the padded corpus buffer for `total` bytes (zero pads) and
// returns the address of byte 0.
uint8_t* alloc_corpus(Session& s, uint64_t total) {
  const uint64_t ntiles = (total + kTileBytes - 1) / kTileBytes;
  const size_t alloc = kFrontPad + ntiles * kTileBytes + kBackPad;
  uint8_t* base = s.data.as<uint8_t>(alloc);
  IGB_CUDA(cudaMemsetAsync(base, 0, kFrontPad, s.stream));
  IGB_CUDA(cudaMemsetAsync(base + kFrontPad + total, 0, alloc - kFrontPad - total, s.stream));
  return base + kFrontPad;
}

// Everything derived from the host offsets once the bytes are (or are being)
// placed at s.data + kFrontPad: device offsets, tile descriptors, the
// longest-first order and the count-once work units.
void finish_corpus(Session& s, std::vector<uint64_t>& hoff) {
  const uint64_t m = hoff.size() - 1;
  const uint64_t total = hoff[m];
  const uint64_t ntiles = (total + kTileBytes - 1) / kTileBytes;
  uint8_t* base = static_cast<uint8_t*>(s.data.p);
  uint64_t* doff = s.off.as<uint64_t>(m + 1);
  s.pin.reset();  // the stream is idle between runs and loads
  h2d(s, doff, hoff.data(), (m + 1) * sizeof(uint64_t));
  uint32_t* dtile = s.tile.as<uint32_t>(ntiles + 1);
  launch_tile_seq(doff, m, ntiles, dtile, s.stream);
  s.launches++;
  // count-once schedule: longest sequences first
  std::vector<uint32_t> ord(m);
  for (uint64_t i = 0; i < m; ++i) ord[i] = (uint32_t)i;
  std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
    return hoff[a + 1] - hoff[a] > hoff[b + 1] - hoff[b];
  });
  uint32_t* dord = s.order.as<uint32_t>(m + 1);
  if (m)
    h2d(s, dord, ord.data(), m * sizeof(uint32_t));
  // count-once work units: <= kUnitBytes of gram ends of one long sequence;
  // short sequences are counted without routing (k_once_short), a warp or a
  // CTA per sequence
  uint32_t n_long = 0;
  for (uint64_t q = 0; q < m; ++q) n_long += hoff[q + 1] - hoff[q] > (uint64_t)kShortCtaLen;
  s.n_long = n_long;
  // small-alphabet work items: long sequences, the longest
  // cut into parts of ~1/(4 * SMs) of the long bytes (>= 1 MiB) so a corpus
  // of a few long sequences (a genome per chromosome) still fills every SM
  {
    uint64_t long_bytes = 0;
    for (uint32_t i = 0; i < n_long; ++i) long_bytes += hoff[ord[i] + 1] - hoff[ord[i]];
    const char* sb = getenv("IG_DIRECT_SPLIT_BYTES");  // tests: force splits
    const uint64_t target = sb ? std::max<uint64_t>(1024, strtoull(sb, nullptr, 10))
                               : std::max<uint64_t>(1ull << 20, long_bytes / (4ull * s.num_sms));
    std::vector<DirectItem> items;
    uint32_t nsplit = 0;
    for (uint32_t i = 0; i < n_long; ++i) {
      const uint64_t len = hoff[ord[i] + 1] - hoff[ord[i]];
      const uint32_t np = len > 2 * target
                              ? (uint32_t)std::min<uint64_t>((len + target - 1) / target, 1u << 16)
                              : 1u;
      const uint32_t slot = np > 1 ? nsplit++ : 0u;
      for (uint32_t p = 0; p < np; ++p) items.push_back(DirectItem{ord[i], p, np, slot});
    }
    std::stable_sort(items.begin(), items.end(), [&](const DirectItem& a, const DirectItem& b) {
      return (hoff[a.q + 1] - hoff[a.q]) / a.nparts > (hoff[b.q + 1] - hoff[b.q]) / b.nparts;
    });
    DirectItem* di = s.direct_items.as<DirectItem>(items.size() + 1);
    if (!items.empty()) h2d(s, di, items.data(), items.size() * sizeof(DirectItem));
    s.n_direct_items = (uint32_t)items.size();
    s.n_direct_split = nsplit;
  }
  s.corpus_alpha = -1;  // measured lazily by the first count-once run
  std::vector<RouteUnit> units;
  std::vector<uint32_t> ufirst(m + 1, 0);
  std::vector<uint32_t> sw, sc;
  for (uint64_t q = 0; q < m; ++q) {
    ufirst[q] = (uint32_t)units.size();
    const uint64_t len = hoff[q + 1] - hoff[q];
    if (len <= (uint64_t)kShortWarpLen) {
      if (len) sw.push_back((uint32_t)q);
      continue;
    }
    if (len <= (uint64_t)kShortCtaLen) {
      sc.push_back((uint32_t)q);
      continue;
    }
    for (uint64_t b = hoff[q]; b < hoff[q + 1]; b += kUnitBytes) {
      RouteUnit u{};
      u.q = (uint32_t)q;
      u.b0 = b;
      u.b1 = std::min<uint64_t>(b + kUnitBytes, hoff[q + 1]);
      units.push_back(u);
    }
  }
  RouteUnit* dun = s.units.as<RouteUnit>(units.size() + 1);
  if (!units.empty())
    h2d(s, dun, units.data(), units.size() * sizeof(RouteUnit));
  ufirst[m] = (uint32_t)units.size();
  uint32_t* duf = s.unit_first.as<uint32_t>(m + 1);
  h2d(s, duf, ufirst.data(), (m + 1) * sizeof(uint32_t));
  uint32_t* dsw = s.short_w.as<uint32_t>(sw.size() + 1);
  uint32_t* dsc = s.short_c.as<uint32_t>(sc.size() + 1);
  if (!sw.empty())
    h2d(s, dsw, sw.data(), sw.size() * 4);
  if (!sc.empty())
    h2d(s, dsc, sc.data(), sc.size() * 4);
  s.rc.units = dun;
  s.rc.unit_first = duf;
  s.rc.nunits = (uint32_t)units.size();
  s.rc.u0 = 0;
  s.rc.u1 = s.rc.nunits;
  s.rc.q0 = 0;
  s.rc.q1 = (uint32_t)m;
  IGB_CUDA(cudaStreamSynchronize(s.stream));
  s.hoff.swap(hoff);
  s.hufirst.swap(ufirst);
  s.h_short_w.swap(sw);
  s.h_short_c.swap(sc);
  s.batches.clear();
  s.dc.data = base + kFrontPad;
  s.dc.off = doff;
  s.dc.tile_seq = dtile;
  s.dc.order = dord;
  s.dc.m = m;
  s.dc.total = total;
  s.dc.ntiles = ntiles;
  s.loaded = true;
}

void check_offsets(const std::vector<uint64_t>& hoff) {
  const uint64_t m = hoff.size() - 1;
  if (hoff[0] != 0) throw Error(IG_ECONFIG, "corpus offsets must start at 0");
  for (uint64_t i = 0; i < m; ++i)
    if (hoff[i + 1] < hoff[i]) throw Error(IG_ECONFIG, "corpus offsets must be non-decreasing");
  if (m >= 0xffffffffull) throw Error(IG_ECONFIG, "too many sequences");
}

void load_corpus(Session& s, const ig_corpus& c, bool copy_data) {
  use_device(s);
  const uint64_t m = c.num_seqs;
  std::vector<uint64_t> hoff(m + 1);
  if (c.location == IG_DEVICE) {
    IGB_CUDA(cudaMemcpy(hoff.data(), c.offsets, (m + 1) * sizeof(uint64_t),
                        cudaMemcpyDeviceToHost));
  } else {
    memcpy(hoff.data(), c.offsets, (m + 1) * sizeof(uint64_t));
  }
  check_offsets(hoff);
  const uint64_t total = hoff[m];
  uint8_t* data = alloc_corpus(s, total);
  if (total && copy_data) {
    IGB_CUDA(cudaMemcpyAsync(data, c.data, total,
                             c.location == IG_DEVICE ? cudaMemcpyDeviceToDevice
                                                     : cudaMemcpyHostToDevice,
                             s.stream));
  }
  finish_corpus(s, hoff);
}

void init_select(Session& s) {
  s.sel.stream = s.stream;
  s.sel.num_sms = s.num_sms;
  s.sel.state = s.sel_state.as<SelState>(1);
  s.sel.hist = s.sel_hist.as<uint32_t>(256);
  s.sel.scalar = s.sel_scalar.as<unsigned long long>(2);  // max, sum
  if (!s.sel.h_state) {
    IGB_CUDA(cudaHostAlloc(&s.sel.h_state, sizeof(SelState), cudaHostAllocMapped));
    IGB_CUDA(cudaHostAlloc(&s.sel.h_scalar, 2 * sizeof(unsigned long long), cudaHostAllocMapped));
  }
}

// Builds the count-all prefix set for survivors keys[0..K) of length plen:
// one open-addressing slice (load <= 0.5), p = survivor rank.
static DevPrefixSet build_prefix_set(Session& s, const uint64_t* keys, uint64_t K, uint32_t plen,
                                     bool dense_rank = false) {
  DevPrefixSet ps;
  ps.K = (uint32_t)K;
  ps.plen = plen;
  if (dense_rank && plen == 3 && K > 4096 && !getenv("IG_NO_RANK_BITMAP")) {
    // 3-byte prefixes too many for the shared-memory set: a rank bitmap over
    // the whole 2^24 prefix space (4 MiB, L2-resident), p = rank in key order
    uint64_t* rb = s.rankbits.as<uint64_t>((size_t)2 << 18);
    uint64_t* pk = s.pkeys.as<uint64_t>(K + 1);
    uint32_t* rp = s.rank_of_p.as<uint32_t>(K + 1);
    launch_rank_prefix(keys, (uint32_t)K, rb, pk, rp, s.stream);
    s.launches += 3;
    ps.pkeys = pk;
    ps.rankbits = rb;
    return ps;
  }
  uint32_t* owner = s.owner.as<uint32_t>(K + 1);
  uint32_t* ocnt = s.owner_cnt.as<uint32_t>(16);
  uint32_t* ostart = s.owner_start.as<uint32_t>(17);
  uint32_t* cursor = s.cursor.as<uint32_t>(16);
  const uint32_t G = 1;
  std::vector<uint32_t> cnt(16, 0);
  uint32_t lgG = 0;
  while ((1u << lgG) < G) ++lgG;
  std::vector<uint32_t> gc(G, 0), gs(G + 1, 0);
  if (G == 1) {
    gc[0] = (uint32_t)K;
  } else {
    for (uint32_t q = 0; q < 16; ++q) gc[q & (G - 1)] += cnt[q];
  }
  uint32_t mx = 0;
  for (uint32_t o = 0; o < G; ++o) {
    gs[o + 1] = gs[o] + gc[o];
    mx = std::max(mx, gc[o]);
  }
  uint32_t lgS = 2;  // >= one 4-slot bucket (hash_slot)
  while ((1ull << lgS) < 2ull * std::max<uint32_t>(mx, 1)) ++lgS;
  const uint32_t S = 1u << lgS;
  // recompute owners at width G (owner16 & (G-1) == owner_G)
  launch_prefix_owner(keys, (uint32_t)K, plen, G, owner, ocnt /*scratch*/, s.stream);
  s.launches++;
  h2d(s, ostart, gs.data(), (G + 1) * sizeof(uint32_t));
  IGB_CUDA(cudaMemsetAsync(cursor, 0, 16 * sizeof(uint32_t), s.stream));
  uint64_t* hk = s.hkeys.as<uint64_t>((size_t)G * S);
  uint32_t* hi = s.hidx.as<uint32_t>((size_t)G * S);
  uint64_t* pk = s.pkeys.as<uint64_t>(K + 1);
  uint32_t* rp = s.rank_of_p.as<uint32_t>(K + 1);
  IGB_CUDA(cudaMemsetAsync(hk, 0xff, (size_t)G * S * sizeof(uint64_t), s.stream));
  // a set that will be read as {key, p} 16-byte slots (key and index do not
  // pack into 64 bits) gets 2-aligned homes: a 32-byte probe holds 2 slots
  {
    uint32_t ibw = 1;
    while ((1ull << ibw) <= mx) ++ibw;
    ps.hmask = (8 * plen + ibw > 64 && G == 1) ? ~1u : ~3u;
  }
  // p = rank in key order (deterministic on every GPU; hot-gram slices of
  // the pass table are then contiguous p ranges)
  uint64_t* sk = s.sort_keys.as<uint64_t>(K + 1);
  uint32_t* sr = s.sort_vals.as<uint32_t>(2 * K + 2);
  sort_keys_by_value(keys, (uint32_t)K, 8 * plen, sk, sr, sr + K + 1, s.sort_tmp, s.stream);
  s.launches += 2;
  launch_prefix_insert(sk, (uint32_t)K, owner, G == 1 ? nullptr : ostart, cursor, S, lgS, hk, hi,
                       pk, rp, s.stream, sr, ps.hmask);
  s.launches++;
  ps.pkeys = pk;
  ps.hkeys = hk;
  ps.hidx = hi;
  ps.owner_start = ostart;
  ps.G = G;
  ps.lgG = lgG;
  ps.S = S;
  ps.lgS = lgS;
  ps.max_owner = mx;
  // packed copy for shared-memory staging when key and local index fit in 64 bits
  uint32_t ib = 1;
  while ((1ull << ib) <= mx) ++ib;
  if (8 * plen + ib <= 64) {
    ps.ib = ib;
    uint64_t* pk2 = s.hpacked.as<uint64_t>((size_t)G * S);
    ps.packed = pk2;
    launch_pack_prefix(ps, pk2, s.stream);
    s.launches++;
  } else if (G == 1) {
    uint64_t* w = s.hpacked.as<uint64_t>((size_t)2 * S);
    ps.wide = w;
    launch_pack_wide(ps, w, s.stream);
    s.launches++;
  }
  return ps;
}

// A collective at world 1 is skipped, except under IG_COLLECTIVE_AT_WORLD1
// (tests: the whole collective plumbing on a one-GPU box).
static bool coll_active(const Session& s) {
  static const bool at1 = getenv("IG_COLLECTIVE_AT_WORLD1") != nullptr;
  return s.has_coll && (s.coll.world > 1 || at1);
}

static void allreduce(Session& s, void* buf, uint64_t count, int dtype) {
  if (!coll_active(s)) return;
  if (!s.coll.allreduce) throw Error(IG_EINTERNAL, "collective has no allreduce");
  const int rc = s.coll.allreduce(buf, count, dtype, (void*)s.stream, s.coll.user);
  if (rc != 0) throw Error(IG_EINTERNAL, "allreduce callback failed");
}

// A pass table summed over the ranks.  A u64 table goes through the
// collective as u32 when that is provably exact: the sum of the per-rank
// maxima (itself all-reduced, one u64) bounds every summed entry, so below
// 2^32 no entry can overflow.  Halves the bytes of count-all tables whose
// totals only might reach 2^32 (c5: 3 GB per pass -> 1.5 GB).
template <typename CT>
static void allreduce_table(Session& s, CT* t, uint64_t n) {
  if (!coll_active(s)) return;
  if constexpr (sizeof(CT) == 8) {
    static const bool no_narrow = getenv("IG_NO_NARROW_ALLREDUCE") != nullptr;
    if (!no_narrow && n && n % 4 == 0) {
      unsigned long long* mx = reinterpret_cast<unsigned long long*>(s.work.as<uint32_t>(64));
      launch_max_u64(t, n, mx, s.num_sms, s.stream);
      s.launches++;
      allreduce(s, mx, 1, 1);
      unsigned long long bound = 0;
      d2h(s, &bound, mx, sizeof(bound));
      if (bound < (1ull << 32)) {
        uint32_t* nar = s.scratch32.as<uint32_t>(n);
        launch_narrow_u64(t, nar, n, s.num_sms, s.stream);
        allreduce(s, nar, n, 0);
        launch_widen_set(nar, t, n, s.num_sms, s.stream);
        s.launches += 2;
        return;
      }
    }
  }
  allreduce(s, t, n, sizeof(CT) == 4 ? 0 : 1);
}

// Owner-hash width the count-once extension passes use for k' survivors: ~40
// prefixes per owner on average (at most kPrefixesPerOwner after the check in
// prepare_prefix).  Known before the survivors are, so the previous pass's
// scatter can histogram the next pass's owners (fused count).
static uint32_t predicted_lgno(uint64_t kp) {
  uint32_t lg = 0;
  while (lg < 63 && (kp >> lg) + ((kp & ((1ull << lg) - 1)) != 0) > 40) ++lg;
  return lg;
}

// Survivor prefix structure for the next extension pass: the bucketed (CSR)
// set for count-once routing, the open-addressing set for count-all.
struct Prefix {
  DevPrefixSet ps;
  RouteParams rp;
  bool csr = false;  // perfect-hash prefix set (count-once)
  bool exact_once = false;  // count-once by sorting (survivor set too large to route)
  uint64_t K = 0;
  std::vector<uint32_t> rank_of_p;  // count-once: p -> survivor rank
  const uint64_t* pkeys = nullptr;   // count-once: keys by p
  std::vector<uint64_t> pk;          // count-once: host keys by p
  std::vector<uint32_t> ostart;      // count-once: host owner ranges
  uint32_t plen = 0;
  bool table_built = false;  // count-once: build_prefix_table already ran
};

static Prefix prepare_prefix(Session& s, const uint64_t* keys, uint64_t K, uint32_t plen,
                             int mode, uint32_t lgno_start = 0) {
  Prefix P;
  P.K = K;
  if (!K) return P;
  // count-once with a survivor set too large for 16-bit owners (or forced by
  // IG_ONCE_EXACT_MIN_K for tests): the open-addressing set + the sort path
  static const char* force = getenv("IG_ONCE_EXACT_MIN_K");
  const uint64_t exact_min = force ? strtoull(force, nullptr, 10) : (uint64_t)kPrefixesPerOwner << 15;
  if (mode == IG_MODE_ONCE && K >= exact_min) {
    P.ps = build_prefix_set(s, keys, K, plen);
    P.exact_once = true;
    P.plen = plen;
    return P;
  }
  if (mode == IG_MODE_ONCE) {
    // count-once routing: owners = hash(prefix) with <= 64 prefixes each,
    // prefixes numbered owner by owner (stable by rank), CHD perfect-hash set
    std::vector<uint64_t> hk(K);
    d2h(s, hk.data(), keys, K * 8);
    auto owner_of = [plen](uint64_t key, uint32_t lgno) -> uint32_t {
      return owner_hash(key, plen, lgno);
    };
    uint32_t lgno = lgno_start;
    std::vector<uint32_t> cnt;
    for (;; ++lgno) {
      cnt.assign((size_t)1 << lgno, 0);
      uint32_t mx = 0;
      for (uint64_t i = 0; i < K; ++i) mx = std::max(mx, ++cnt[owner_of(hk[i], lgno)]);
      if (mx <= kPrefixesPerOwner) break;
      // routed entries carry the owner in 16 bits (route_kernels.cu)
      if (lgno >= 16) {
        P.ps = build_prefix_set(s, keys, K, plen);
        P.exact_once = true;
        P.plen = plen;
        return P;
      }
    }
    const uint32_t NO = 1u << lgno;
    std::vector<uint32_t> ostart(NO + 1, 0);
    for (uint32_t o = 0; o < NO; ++o) ostart[o + 1] = ostart[o] + cnt[o];
    std::vector<uint32_t> cur(ostart.begin(), ostart.end() - 1);
    std::vector<uint64_t> pk(K);
    P.rank_of_p.assign(K, 0);
    for (uint64_t i = 0; i < K; ++i) {
      const uint32_t pp = cur[owner_of(hk[i], lgno)]++;
      pk[pp] = hk[i];
      P.rank_of_p[pp] = (uint32_t)i;
    }
    uint64_t* dpk = s.pkeys.as<uint64_t>(K + 1);
    uint32_t* dos = s.owner_start.as<uint32_t>(NO + 1);
    h2d(s, dpk, pk.data(), K * 8);
    h2d(s, dos, ostart.data(), (NO + 1) * 4);
    P.pk = std::move(pk);
    P.ostart = std::move(ostart);
    P.plen = plen;
    RouteParams& rp = P.rp;
    rp.ext = true;
    rp.lgno = lgno;
    rp.NO = NO;
    rp.lgl = 14;  // kPrefixesPerOwner * 256 ids per owner
    rp.ostart = dos;
    rp.minv = 0;  // table index = p * 256 + last byte
    P.pkeys = dpk;
    P.csr = true;
  } else {
    P.ps = build_prefix_set(s, keys, K, plen, /*dense_rank=*/true);
  }
  return P;
}

// The perfect-hash table of a count-once prefix set (host build + upload).  Run
// while the pass's count kernel (which needs only the owner function) is in
// flight.
static void build_prefix_table(Session& s, Prefix& P) {
  static const bool trace = getenv("IG_TRACE_BUILD") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  struct Tr {
    bool on;
    std::chrono::steady_clock::time_point t0;
    uint64_t K;
    ~Tr() {
      if (on)
        fprintf(stderr, "[ig] prefix table build: K=%llu %.3f ms\n", (unsigned long long)K,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
  } tr{trace, t0, P.K};
  const uint64_t K = P.K;
  const uint32_t lgno = P.rp.lgno;
  const uint32_t plen = P.plen;
  auto owner_of = [plen](uint64_t key, uint32_t lg) -> uint32_t { return owner_hash(key, plen, lg); };
  const std::vector<uint64_t>& pk = P.pk;
  const std::vector<uint32_t>& ostart = P.ostart;
  // perfect-hash slots; slot value: owner << 6 | index of the prefix in its owner
  std::vector<uint32_t> slot_of_key;
  std::vector<uint16_t> disp;
  uint32_t nb = 0, nslots = 0;
  const bool narrow = P.plen <= 4;
  build_prefix_mphf(pk, narrow, slot_of_key, disp, nb, nslots);
  std::vector<uint64_t> slots(nslots, kEmptyKey);
  std::vector<uint32_t> slot_v(nslots, 0xffffffu);
  for (uint64_t pp = 0; pp < K; ++pp) {
    const uint32_t o = owner_of(pk[pp], lgno);
    slots[slot_of_key[pp]] = pk[pp];
    slot_v[slot_of_key[pp]] = (o << 6) | (uint32_t)(pp - ostart[o]);
  }
  // slot layout by prefix length (route_kernels.cu: prefix_lookup_v)
  for (size_t i = 0; i < slots.size(); ++i) {
    if (slots[i] == kEmptyKey) continue;
    if (P.plen <= 4)
      slots[i] = (slots[i] << 32) | ((slot_v[i] >> 6) << 16) | ((slot_v[i] & 63u) << 8);
    else if (P.plen == 5) slots[i] = (slots[i] << 24) | slot_v[i];
    else slots[i] = (slots[i] << 8) | (slot_v[i] & 63u);
  }
  uint64_t* ds = s.hkeys.as<uint64_t>(slots.size() + 2);
  uint16_t* ddisp = s.hpacked.as<uint16_t>(disp.size() + 8);
  h2d(s, ds, slots.data(), slots.size() * 8);
  h2d(s, ddisp, disp.data(), disp.size() * 2);
  IGB_CUDA(cudaStreamSynchronize(s.stream));  // host vectors die here
  P.rp.nb = nb;
  P.rp.nslots = nslots;
  P.rp.slots = ds;
  P.rp.disp = ddisp;
}

// Count-once short sequences of [q0, q1) (both classes) into the pass table.
template <typename CT>
static void short_pass(Session& s, int kind, uint32_t L, const RouteParams& rp, CT* t, uint32_t q0,
                       uint32_t q1) {
  auto range = [&](const std::vector<uint32_t>& v) {
    const size_t a = std::lower_bound(v.begin(), v.end(), q0) - v.begin();
    const size_t b = std::lower_bound(v.begin(), v.end(), q1) - v.begin();
    return std::make_pair(a, b);
  };
  const auto w = range(s.h_short_w), c = range(s.h_short_c);
  if (w.first == w.second && c.first == c.second) return;
  const size_t ev = s.kt.begin(IG_KF_ONCE_SHORT, s.stream);
  count_once_short<CT>(kind, L, s.dc, rp, static_cast<const uint32_t*>(s.short_w.p) + w.first,
                       (uint32_t)(w.second - w.first),
                       static_cast<const uint32_t*>(s.short_c.p) + c.first,
                       (uint32_t)(c.second - c.first), t, s.num_sms, s.stream);
  s.kt.end(ev, s.stream);
  s.launches += (w.first != w.second) + (c.first != c.second);
}

// ---- count-all with sampled hot-gram tables
static constexpr uint64_t kHotMinTiles = 1ull << 19;  // 256 MiB: below, the plain kernel

static uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* v = getenv(name);
  return v ? strtoull(v, nullptr, 10) : dflt;
}

// Tiles per count-all segment of a u64 table (< 2^32 positions each, so the
// u32 scratch cannot wrap).  IG_SEG_TILES shrinks it for tests.
static uint64_t seg_tiles() {
  return std::max<uint64_t>(1, env_u64("IG_SEG_TILES", 0xF0000000ull / kTileBytes));
}

static bool hot_path_ok(Session& s, bool dense, const Prefix* P) {
  if (getenv("IG_NO_HOT") || s.dc.ntiles < env_u64("IG_HOT_MIN_TILES", kHotMinTiles)) return false;
  if (dense) return true;
  const DevPrefixSet& ps = P->ps;
  if (ps.packed && (size_t)ps.S * 8 <= 64 * 1024) return false;  // smem-staged: plain kernel
  return ps.rankbits || ps.packed || ps.wide;
}


template <typename CT>
static void count_all_hot(Session& s, bool dense, uint32_t L, const Prefix* P, CT* t,
                          uint64_t tcap) {
  // slices: the cold REDs of one sweep touch <= IG_HOT_SLICE_MB of table
  const uint64_t slice_mb = env_u64("IG_HOT_SLICE_MB", 4096);
  const uint32_t lgnb = (uint32_t)std::max<uint64_t>(6, std::min<uint64_t>(13, env_u64("IG_HOT_LGNB", 13)));
  const uint64_t cold_bytes = tcap * 4;
  uint32_t S = 1;
  while (S < (uint32_t)kMaxHotSlices && cold_bytes > (uint64_t)S * slice_mb * (1ull << 20)) S *= 2;
  if (getenv("IG_HOT_SLICES"))
    S = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(kMaxHotSlices, env_u64("IG_HOT_SLICES", 1)));
  const uint64_t K = dense ? 0 : P->K;
  if (!dense && S > K) S = 1;
  HotSliceIds sl;
  sl.S = S;
  uint64_t* bounds = s.hot_bounds.as<uint64_t>(kMaxHotSlices + 2);
  if (dense) {
    std::vector<uint64_t> b(S + 1);
    for (uint32_t i = 0; i < S; ++i) b[i] = sl.lo[i] = tcap * i / S;
    b[S] = ~0ull;
    h2d(s, bounds, b.data(), (S + 1) * 8);
  } else {
    for (uint32_t i = 0; i < S; ++i) sl.lo[i] = 256 * (K * i / S);
    launch_slice_bounds(P->ps.pkeys, (uint32_t)K, S, bounds, s.stream);
    s.launches++;
  }
  // 1. sample: every stride-th tile, plain kernel, into a u32 scratch (< 2^32
  // positions: at most 1/16 of the corpus); the sweeps below count every tile
  uint32_t* sample = s.scratch32.as<uint32_t>(tcap);
  IGB_CUDA(cudaMemsetAsync(sample, 0, tcap * 4, s.stream));
  uint32_t sample_stride = kHotSampleStrideMin;
  {
    DevCorpus dc = s.dc;
    dc.tile0 = 0;
    // ~2^17 sample tiles (64 MiB): every 16th tile of a 1 GiB corpus, every
    // 256th from 16 GiB up (c3: 64 -> 256 saved 6 ms per run, same hot sets)
    const uint64_t want = std::max<uint64_t>(kHotSampleStrideMin,
                                             std::min<uint64_t>(kHotSampleStrideMax, s.dc.ntiles >> 17));
    sample_stride = (uint32_t)env_u64("IG_HOT_SAMPLE_STRIDE", want);
    dc.tstride = sample_stride;
    DevPrefixSet sps = dense ? DevPrefixSet{} : P->ps;
    sps.hit_out = nullptr;  // the sweeps write this pass's hit masks
    const size_t ev = s.kt.begin(IG_KF_COUNT_ALL, s.stream);
    uint32_t* work = s.work.as<uint32_t>(64);
    if (dense) launch_count_dense<uint32_t>(dc, L, IG_MODE_ALL, sample, work, s.num_sms, s.stream);
    else launch_count_extend<uint32_t>(dc, sps, L, IG_MODE_ALL, sample, work, s.num_sms, s.stream);
    s.kt.end(ev, s.stream);
    s.launches++;
  }
  // 2-3. hot sets of every slice from the sample counts
  HotSet hs;
  const size_t slots = (size_t)S * (2u << lgnb);
  hs.keys = s.hot_keys.as<uint64_t>(slots);
  hs.ids = s.hot_ids.as<uint32_t>(slots);
  bool direct = hot_sweep_queued(dense ? DevPrefixSet{} : P->ps, dense, L, S > 1);
  // a gram above ~1/1024 of the positions must not be left to same-address L2
  // REDs: when a direct table (one slot per key) loses one to a hotter key,
  // the table is rebuilt two-way and the pass takes the two-way kernels
  const uint64_t sample_pos = (s.dc.ntiles / sample_stride + 1) * kTileBytes;
  const uint64_t important = env_u64("IG_HOT_IMPORTANT", sample_pos >> 10);
  // up to 4 multipliers per table kind: a rebuild with another multiplier
  // moves apart the keys that shared a slot; then (direct tables only) the
  // two-way build, whose pass takes the two-way kernels
  static const uint32_t kMuls[4] = {0x9E3779B1u, 0xC2B2AE3Du, 0x27D4EB2Fu, 0x165667B1u};
  for (int attempt = 0;; ++attempt) {
    build_hot_set<uint32_t>(sample, tcap, sl, dense ? nullptr : P->ps.pkeys, lgnb, hs,
                            s.hot_work, s.num_sms, s.stream, direct, important, kMuls[attempt & 3]);
    s.launches += 6 + (direct ? 0 : 1);
    uint32_t lost = 0;
    d2h(s, &lost, hs.lost, sizeof(lost));
    if (!lost) break;
    if ((attempt & 3) == 3) {
      if (!direct) break;  // every multiplier lost one: keep the last table
      direct = false;
    }
  }
  // 4. sweeps: per < 2^32-position segment when the table is u64 (cold REDs
  // into a u32 scratch, widened after the segment), once per slice
  const DevPrefixSet& ps = dense ? DevPrefixSet{} : P->ps;
  auto sweep = [&](const DevCorpus& dc, auto* cold) {
    for (uint32_t i = 0; i < S; ++i) {
      HotSweep hw;
      hw.keys = hs.keys + (size_t)i * (2u << lgnb);
      hw.ids = hs.ids + (size_t)i * (2u << lgnb);
      hw.lgnb = lgnb;
      hw.bounds = bounds + i;
      hw.first = i == 0;
      hw.sliced = S > 1;
      hw.direct = hs.direct;
      hw.mul = hs.mul;
      hw.sparse_iters = (uint32_t)env_u64("IG_SPARSE_ITERS", 10);
      const size_t ev = s.kt.begin(IG_KF_COUNT_ALL, s.stream);
      launch_count_hot(dc, ps, dense, L, hw, t, cold, s.num_sms, s.stream);
      s.kt.end(ev, s.stream);
      s.launches++;
    }
  };
  if constexpr (sizeof(CT) == 8) {
    uint32_t* scratch = s.scratch32.as<uint32_t>(tcap);
    const uint64_t seg = seg_tiles();
    for (uint64_t t0 = 0; t0 < s.dc.ntiles; t0 += seg) {
      DevCorpus dc = s.dc;
      dc.tile0 = t0;
      dc.ntiles = std::min<uint64_t>(s.dc.ntiles, t0 + seg);
      IGB_CUDA(cudaMemsetAsync(scratch, 0, tcap * 4, s.stream));
      sweep(dc, scratch);
      launch_widen_add(scratch, t, tcap, s.num_sms, s.stream);
      s.launches++;
    }
  } else {
    sweep(s.dc, t);
  }
}

// The small-alphabet kernels' work for a candidate space of nbits bits.
static DirectWork direct_work(Session& s, uint64_t nbits) {
  DirectWork w;
  w.items = static_cast<const DirectItem*>(s.direct_items.p);
  w.nitems = s.n_direct_items;
  w.nsplit = s.n_direct_split;
  if (w.nsplit) {
    const size_t nwords = (nbits + 31) / 32;
    w.gbm = s.direct_gbm.as<uint32_t>((size_t)w.nsplit * (nwords + 1));
    w.done = w.gbm + (size_t)w.nsplit * nwords;
  }
  return w;
}

// One counting pass.  Returns the device table (tcap entries) and how table
// indices map to gram keys.
template <typename CT>
static CT* count_pass(Session& s, bool dense, uint32_t L, int mode, const Prefix* P,
                      uint64_t& tcap, KeyMap& km, int32_t next_lgno = -1) {
  if (mode == IG_MODE_ONCE && !dense && P->exact_once) {
    tcap = 256 * P->K;
    CT* t = s.table.as<CT>(tcap);
    IGB_CUDA(cudaMemsetAsync(t, 0, tcap * sizeof(CT), s.stream));
    const size_t ev = s.kt.begin(IG_KF_ONCE_SHORT, s.stream);
    count_once_exact<CT>(s, L, P->ps, tcap, t);
    s.kt.end(ev, s.stream);
    km = KeyMap{};
    km.pkeys = P->ps.pkeys;
    return t;
  }
  if (mode == IG_MODE_ONCE && !dense && s.alpha_n <= 16 && !getenv("IG_NO_DIRECT")) {
    // small alphabet: K' * A candidates in a shared-memory bitmap per sequence
    const uint64_t nbits = P->K * s.alpha_n;
    const size_t est = (nbits + 31) / 32 * 4 + (size_t)P->rp.NO * 4 + 256 + 12 * P->K + 1024;
    // prefixes as rank-packed indices into a direct table when they fit 16 bits
    uint32_t bits = 1;
    while ((1u << bits) < s.alpha_n) ++bits;
    const uint32_t plen = L - 1;
    const uint64_t lut_n = bits * plen <= 16 ? (1ull << (bits * plen)) : 0;
    const bool lut_ok = lut_n && P->K < 0xffff && L >= 4 && !getenv("IG_NO_DIRECT_LUT") &&
                        (nbits + 31) / 32 * 4 + 256 + lut_n * 2 + 1024 <= kMaxOnceSmem;
    if (nbits <= (1ull << 20) && lut_ok) {
      std::vector<uint16_t> lut(lut_n, 0xffff);
      for (uint64_t pp = 0; pp < P->K; ++pp) {
        uint32_t ci = 0;
        for (uint32_t i = 0; i < plen; ++i)
          ci = (ci << bits) | s.h_arank[(P->pk[pp] >> (8 * (plen - 1 - i))) & 0xffu];
        lut[ci] = (uint16_t)pp;
      }
      uint16_t* dl = s.lut.as<uint16_t>(lut_n);
      h2d(s, dl, lut.data(), lut_n * 2);
      tcap = 256 * P->K;
      CT* t = s.table.as<CT>(tcap);
      IGB_CUDA(cudaMemsetAsync(t, 0, tcap * sizeof(CT), s.stream));
      s.rc.have_next = false;
      if (!s.h_short_w.empty() || !s.h_short_c.empty()) {  // short sequences: route table
        build_prefix_table(s, *const_cast<Prefix*>(P));
        short_pass<CT>(s, 1, L, P->rp, t, 0, (uint32_t)s.dc.m);
      }
      const uint8_t* ab = static_cast<const uint8_t*>(s.alpha_dev.p) + 32;
      const size_t ev = s.kt.begin(IG_KF_ONCE_DIRECT, s.stream);
      count_once_direct<CT>(s.dc, L, P->rp, direct_work(s, nbits), ab, ab + 256, s.alpha_n,
                            P->K, s.compact.as<uint32_t>(nbits + 1), t, s.num_sms, s.stream, dl,
                            (uint32_t)lut_n, bits);
      s.kt.end(ev, s.stream);
      s.launches += (s.n_long ? 1 : 0) + 1;
      km = KeyMap{};
      km.pkeys = P->pkeys;
      return t;
    }
    if (nbits <= (1ull << 20) && est <= kMaxOnceSmem) {
      build_prefix_table(s, *const_cast<Prefix*>(P));
      if (direct_smem(P->rp, nbits) <= kMaxOnceSmem) {
        tcap = 256 * P->K;
        CT* t = s.table.as<CT>(tcap);
        IGB_CUDA(cudaMemsetAsync(t, 0, tcap * sizeof(CT), s.stream));
        s.rc.have_next = false;  // no fused histogram for the pass after this one
        short_pass<CT>(s, 1, L, P->rp, t, 0, (uint32_t)s.dc.m);
        const uint8_t* ab = static_cast<const uint8_t*>(s.alpha_dev.p) + 32;
        const size_t ev = s.kt.begin(IG_KF_ONCE_DIRECT, s.stream);
        count_once_direct<CT>(s.dc, L, P->rp, direct_work(s, nbits), ab, ab + 256,
                              s.alpha_n, P->K, s.compact.as<uint32_t>(nbits + 1), t, s.num_sms,
                              s.stream);
        s.kt.end(ev, s.stream);
        s.launches += (s.n_long ? 1 : 0) + 1;
        km = KeyMap{};
        km.pkeys = P->pkeys;
        return t;
      }
      // did not fit after all: the route path (its table build is done)
      const_cast<Prefix*>(P)->table_built = true;
    }
  }
  if (mode == IG_MODE_ONCE && dense && L == 3 && s.batches.empty() && !getenv("IG_NO_DIRECT")) {
    // resident corpus over <= 16 distinct bytes: the dense pass counts the
    // A^3 possible 3-grams in a per-sequence bitmap too
    if (s.corpus_alpha < 0) {
      uint8_t* ad = s.calpha_dev.as<uint8_t>(48 + 512);  // mask[9] | pad | arank | alpha
      byte_presence(s.dc.data, s.dc.total, reinterpret_cast<uint32_t*>(ad), s.num_sms, s.stream);
      s.launches++;
      uint32_t mask[9];
      d2h(s, mask, ad, sizeof(mask));
      uint8_t tab[512];
      memset(tab, 0, sizeof(tab));
      uint32_t A = 0;
      for (uint32_t b = 0; b < 256; ++b)
        if (mask[b >> 5] >> (b & 31) & 1u) {
          tab[b] = (uint8_t)std::min<uint32_t>(A, 255);
          if (A < 256) tab[256 + A] = (uint8_t)b;
          ++A;
        }
      s.corpus_alpha = mask[8] ? 257 : (int32_t)A;
      if (!mask[8] && A >= 1 && A <= 16) h2d(s, ad + 48, tab, sizeof(tab));
    }
    const uint32_t A = (uint32_t)s.corpus_alpha;
    if (A >= 1 && A <= 16) {
      RouteParams rp;
      make_route_params(1ull << 24, rp);
      uint32_t bits = 1;
      while ((1u << bits) < A) ++bits;
      const uint32_t lut_n = 1u << (2 * bits);
      std::vector<uint16_t> lut(lut_n, 0xffff);
      for (uint32_t r0 = 0; r0 < A; ++r0)
        for (uint32_t r1 = 0; r1 < A; ++r1) lut[(r0 << bits) | r1] = (uint16_t)(r0 * A + r1);
      uint16_t* dl = s.lut.as<uint16_t>(lut_n);
      h2d(s, dl, lut.data(), (size_t)lut_n * 2);
      tcap = 1ull << rp.lgc;
      CT* t = s.table.as<CT>(tcap);
      IGB_CUDA(cudaMemsetAsync(t, 0, tcap * sizeof(CT), s.stream));
      s.rc.have_next = false;
      short_pass<CT>(s, 0, L, rp, t, 0, (uint32_t)s.dc.m);
      const uint8_t* ab = static_cast<const uint8_t*>(s.calpha_dev.p) + 48;
      uint32_t* cmp = s.compact.as<uint32_t>((size_t)A * A * A + 1);
      const size_t ev = s.kt.begin(IG_KF_ONCE_DIRECT, s.stream);
      count_once_direct<CT>(s.dc, 3, rp, direct_work(s, (uint64_t)A * A * A), ab,
                            ab + 256, A, (uint64_t)A * A, cmp, t, s.num_sms, s.stream, dl, lut_n,
                            bits, /*expand=*/false);
      expand_dense<CT>(cmp, A, ab + 256, rp.mult, rp.cmask, t, s.stream);
      s.kt.end(ev, s.stream);
      s.launches += (s.n_long ? 1 : 0) + 1;
      km = KeyMap{};
      km.minv = rp.minv;
      km.cmask = rp.cmask;
      return t;
    }
  }
  if (mode == IG_MODE_ONCE) {
    RouteParams rp;
    if (dense) make_route_params(1ull << (8 * L), rp);
    else rp = P->rp;
    static const char* nd = getenv("IG_NO_DEDUP");  // experiment switch: 1 dense, 2 all
    if (nd && (nd[0] == '2' || dense)) rp.dedup = false;
    tcap = dense ? (1ull << rp.lgc) : 256 * P->K;
    CT* t = s.table.as<CT>(tcap);
    IGB_CUDA(cudaMemsetAsync(t, 0, tcap * sizeof(CT), s.stream));
    const uint64_t l0 = s.rc.launches;
    if (dense && !s.batches.empty()) {
      // pipelined load: route each batch as soon as its bytes have landed
      rp.next_lgno = next_lgno;
      for (size_t bi = 0; bi < s.batches.size(); ++bi) {
        const auto& b = s.batches[bi];
        if (s.batch_gate) s.batch_gate(bi);
        if (b.ready) IGB_CUDA(cudaStreamWaitEvent(s.stream, b.ready, 0));
        s.rc.u0 = b.u0;
        s.rc.u1 = b.u1;
        s.rc.q0 = b.q0;
        s.rc.q1 = b.q1;
        route_count_once<CT>(1, s.rc, s.dc, 0, L, rp, t, s.num_sms, s.stream);
        route_count_once<CT>(2, s.rc, s.dc, 0, L, rp, t, s.num_sms, s.stream);
        short_pass<CT>(s, 0, L, rp, t, b.q0, b.q1);
      }
      s.rc.u0 = 0;
      s.rc.u1 = s.rc.nunits;
      s.rc.q0 = 0;
      s.rc.q1 = (uint32_t)s.dc.m;
    } else {
      route_count_once<CT>(1, s.rc, s.dc, dense ? 0 : 1, L, rp, t, s.num_sms, s.stream);
      if (!dense) {  // the host table build overlaps the count kernel
        if (!P->table_built) build_prefix_table(s, *const_cast<Prefix*>(P));
        const bool dd = rp.dedup;
        rp = P->rp;
        rp.dedup = dd;
      }
      rp.next_lgno = next_lgno;
      route_count_once<CT>(2, s.rc, s.dc, dense ? 0 : 1, L, rp, t, s.num_sms, s.stream);
      short_pass<CT>(s, dense ? 0 : 1, L, rp, t, 0, (uint32_t)s.dc.m);
    }
    s.launches += s.rc.launches - l0;
    km = KeyMap{};
    if (dense) {
      km.minv = rp.minv;
      km.cmask = rp.cmask;
    } else {
      km.pkeys = P->pkeys;
    }
    return t;
  }
  uint32_t* work = s.work.as<uint32_t>(64);
  tcap = dense ? (1ull << (8 * L)) : 256 * P->K;
  CT* t = s.table.as<CT>(tcap);
  IGB_CUDA(cudaMemsetAsync(t, 0, tcap * sizeof(CT), s.stream));
  if (!(dense && !s.batches.empty()) && hot_path_ok(s, dense, P)) {
    count_all_hot<CT>(s, dense, L, P, t, tcap);
    km = KeyMap{};
    if (!dense) km.pkeys = P->ps.pkeys;
    return t;
  }
  auto launch = [&](const DevCorpus& dc, auto* tab) {
    using T = std::remove_pointer_t<decltype(tab)>;
    const size_t ev = s.kt.begin(IG_KF_COUNT_ALL, s.stream);
    if (dense) launch_count_dense<T>(dc, L, mode, tab, work, s.num_sms, s.stream);
    else launch_count_extend<T>(dc, P->ps, L, mode, tab, work, s.num_sms, s.stream);
    s.kt.end(ev, s.stream);
    s.launches++;
  };
  // tile ranges: the pipelined load's batches (dense pass only), else all
  std::vector<std::pair<uint64_t, uint64_t>> ranges;
  std::vector<cudaEvent_t> waits;
  if (dense && !s.batches.empty()) {
    for (const auto& b : s.batches) {
      ranges.emplace_back(b.t0, b.t1);
      waits.push_back(b.ready);
    }
  } else {
    ranges.emplace_back(0, s.dc.ntiles);
    waits.push_back(nullptr);
  }
  for (size_t r = 0; r < ranges.size(); ++r) {
    if (s.batch_gate && dense && !s.batches.empty()) s.batch_gate(r);
    if (waits[r]) IGB_CUDA(cudaStreamWaitEvent(s.stream, waits[r], 0));
    if constexpr (sizeof(CT) == 8) {
      // 64-bit totals: count each < 2^32-byte corpus segment into an
      // L2-friendly u32 scratch table, then widen-accumulate into the u64 table
      uint32_t* scratch = s.scratch32.as<uint32_t>(tcap);
      const uint64_t seg = seg_tiles();
      for (uint64_t t0 = ranges[r].first; t0 < ranges[r].second; t0 += seg) {
        DevCorpus dc = s.dc;
        dc.tile0 = t0;
        dc.ntiles = std::min<uint64_t>(ranges[r].second, t0 + seg);
        IGB_CUDA(cudaMemsetAsync(scratch, 0, tcap * 4, s.stream));
        launch(dc, scratch);
        launch_widen_add(scratch, t, tcap, s.num_sms, s.stream);
        s.launches++;
      }
    } else {
      DevCorpus dc = s.dc;
      dc.tile0 = ranges[r].first;
      dc.ntiles = ranges[r].second;
      launch(dc, t);
    }
  }
  km = KeyMap{};
  if (!dense) km.pkeys = P->ps.pkeys;
  return t;
}

template <typename CT>
static uint64_t timed_select(Session& s, const CT* table, uint64_t cap, uint64_t k, KeyMap km,
                             int key_bits, uint64_t* ok, uint64_t* oc) {
  const size_t ev = s.kt.begin(IG_KF_SELECT, s.stream);
  const uint64_t n = select_topk<CT>(s.sel, table, cap, k, km, key_bits, ok, oc);
  s.kt.end(ev, s.stream);
  return n;
}

// Count-table dtype: u32 whenever no count can reach 2^32 (count-once counts
// are <= m; count-all counts are <= the corpus bytes), else u64.
static bool use_u32(Session& s, int mode) {
  if (getenv("IG_FORCE_U64")) return false;  // tests: the u64 / segment paths on small corpora
  const uint64_t bytes = s.has_coll ? s.coll.bytes_total : s.dc.total;
  const uint64_t seqs = s.has_coll ? s.coll.seqs_total : s.dc.m;
  return mode == IG_MODE_ONCE ? seqs < 0xffffffffull : bytes < 0xffffffffull;
}

template <typename CT>
static void run_t(Session& s, const ig_params& p, ig_result* out) {
  init_select(s);
  s.rc.kt = &s.kt;
  s.rc.have_next = false;  // fused next-pass counts never outlive a run
  IGB_CUDA(cudaStreamSynchronize(s.stream));
  s.pin.reset();
  const uint64_t kp = k_prime(p);
  const uint32_t n = p.n;
  const uint32_t n0 = std::min<uint32_t>(n, 3);
  const uint64_t total_bytes = s.has_coll ? s.coll.bytes_total : s.dc.total;
  StepTimer tm(s);
  std::vector<Row> rows;
  std::string diag;
  const uint64_t sel_before = s.sel.launches;

  // ---- dense pass (intergrams.cpp:76-103)
  const uint64_t dcap = 1ull << (8 * n0);
  size_t ev = tm.begin();
  uint64_t tcap = 0;
  KeyMap km;
  // the next pass's owner histogram lives in the scatter's shared memory:
  // fused only up to 2^13 owners (32 KB)
  constexpr uint32_t kMaxFusedLg = 13;
  const int32_t fuse_lg = (p.mode == IG_MODE_ONCE && n > 3 && !getenv("IG_NO_FUSED_COUNT") &&
                           predicted_lgno(kp) <= kMaxFusedLg)
                              ? (int32_t)predicted_lgno(kp) : -1;
  CT* table = count_pass<CT>(s, true, n0, p.mode, nullptr, tcap, km, fuse_lg);
  int32_t next_lg = fuse_lg;
  // owner bits of a count-once prefix set of K survivors: the width the fused
  // histogram was built for, unless K came out far shorter (then recount:
  // thousands of near-empty owners cost more than one count kernel)
  auto owner_bits = [](int32_t fused, uint64_t K) -> uint32_t {
    const uint32_t want = predicted_lgno(K);
    if (fused <= 0) return 0u;
    return want + 1 < (uint32_t)fused ? want : (uint32_t)fused;
  };
  IGB_CUDA(cudaGetLastError());
  allreduce_table<CT>(s, table, tcap);
  s.alpha_n = 256;
  if (p.mode == IG_MODE_ONCE && n > 3) {
    // the byte alphabet, from the (global) dense table: a small one lets the
    // extension passes count candidates in a per-sequence bitmap
    uint8_t* ad = s.alpha_dev.as<uint8_t>(32 + 512);
    alphabet_mask<CT>(table, tcap, km.minv, km.cmask, n0, reinterpret_cast<uint32_t*>(ad),
                      s.num_sms, s.stream);
    s.launches++;
    uint32_t mask[8];
    d2h(s, mask, ad, sizeof(mask));
    uint8_t tab[512];
    memset(tab, 0, sizeof(tab));
    uint32_t A = 0;
    for (uint32_t b = 0; b < 256; ++b)
      if (mask[b >> 5] >> (b & 31) & 1u) {
        tab[b] = (uint8_t)std::min<uint32_t>(A, 255);  // arank
        if (A < 256) tab[256 + A] = (uint8_t)b;       // alpha
        ++A;
      }
    s.alpha_n = std::max<uint32_t>(A, 1);
    if (s.alpha_n <= 16) h2d(s, ad + 32, tab, sizeof(tab));
    s.h_arank.assign(tab, tab + 256);
  }
  tm.end(ev);
  rows.push_back(make_row(std::to_string(n0) + "-gram pass", n0, total_bytes, dcap, 0, false, ev));

  uint64_t* out_keys_d = nullptr;
  uint64_t* out_counts_d = nullptr;
  uint64_t out_len = 0;
  // grams longer than 8 bytes (passes j >= 9): the 8-byte survivors (p =
  // rank in key order) and per later level the survivor ids in id order
  // plus an id -> rank table; a j-gram's prefix rank is walked up from its
  // first 8 bytes, and since every rank follows byte order, ids (p * 256 +
  // last byte) order the grams as their bytes do (intergrams.cpp:56-59)
  DevPrefixSet ps8{};
  uint64_t ns8 = 0;
  std::vector<const uint32_t*> remap_ptrs;
  std::vector<uint64_t> level_len;  // survivors of levels 9 .. j-1

  if (n <= 3) {  // intergrams.cpp:105-113
    ev = tm.begin();
    out_keys_d = s.next_keys.as<uint64_t>(std::min<uint64_t>(p.k, dcap) + 1);
    out_counts_d = s.next_counts.as<uint64_t>(std::min<uint64_t>(p.k, dcap) + 1);
    out_len = timed_select<CT>(s, table, tcap, p.k, km, 8 * n0, out_keys_d, out_counts_d);
    tm.end(ev);
    rows.push_back(make_row("top-k " + std::to_string(n) + "-grams", n, 0, 0, out_len, false, ev));
  } else {
    // ---- survivors of the 3-gram pass (intergrams.cpp:115-132)
    ev = tm.begin();
    uint64_t scap = std::min<uint64_t>(kp, dcap);
    uint64_t* sk = s.surv_keys.as<uint64_t>(scap + 1);
    uint64_t* sc = s.surv_counts.as<uint64_t>(scap + 1);
    uint64_t ns = timed_select<CT>(s, table, tcap, kp, km, 24, sk, sc);
    bool shrt = ns < kp;
    if (shrt)
      diag += "pass 3 retained " + std::to_string(ns) + " candidates (requested " +
              std::to_string(kp) + ")\n";
    Prefix P = prepare_prefix(s, sk, ns, 3, p.mode, owner_bits(fuse_lg, ns));
    tm.end(ev);
    rows.push_back(make_row("top-zk 3-grams/trie building", 3, 0, 0, ns, shrt, ev));

    // count-all hit chaining: a j-gram can be a candidate
    // only where its (j-1)-byte prefix was counted by pass j-1 one byte
    // earlier, so each pass records its hits and the next probes only those
    uint16_t* hmask[2] = {nullptr, nullptr};
    if (p.mode == IG_MODE_ALL && n >= 5 && !getenv("IG_NO_HIT_CHAIN")) {
      const size_t words = (size_t)s.dc.ntiles * 32 + 32;
      size_t fr = 0, tot = 0;
      IGB_CUDA(cudaMemGetInfo(&fr, &tot));
      const size_t have = s.hitmask[0].bytes + s.hitmask[1].bytes;
      if (have >= 4 * words || fr + have > 4 * words + (1ull << 30)) {
        for (int b = 0; b < 2; ++b) {
          uint16_t* w = s.hitmask[b].as<uint16_t>(words);
          IGB_CUDA(cudaMemsetAsync(w, 0, 32 * sizeof(uint16_t), s.stream));
          hmask[b] = w + 32;
        }
      }
    }

    for (uint32_t j = 4; j <= n; ++j) {
      // an empty survivor list is a depth-0 trie (trie.cpp:23) and the
      // extension pass rejects it (intergrams.cpp:46-48)
      if (ns == 0) throw Error(IG_ECONFIG, "extension pass needs a trie of depth j-1");
      const bool chain = j >= 9;
      if (hmask[0] && !chain) {
        P.ps.hit_in = j >= 5 ? hmask[(j - 1) & 1] : nullptr;
        P.ps.hit_out = j < n ? hmask[j & 1] : nullptr;
        // sparse switch of the hot sweeps: on when pass j-1
        // counted fewer than half of the positions (the sum of its table,
        // which its selection read anyway; global on every rank).
        // IG_SPARSE=0/1 forces it.
        P.ps.sparse = P.ps.hit_in && 2 * s.sel.last_sum < total_bytes;
        if (const char* f = getenv("IG_SPARSE")) P.ps.sparse = P.ps.hit_in && f[0] != '0';
      }
      // count-all: a j-gram occurs at most as often as its (j-1)-byte prefix
      // (each occurrence ends one byte after one of the prefix's), so when
      // pass j-1's largest global count (its first survivor) is below 2^32,
      // pass j counts into a u32 table over the whole corpus: no < 4 GiB
      // segments, no scratch widening, half the selection bytes.  Every
      // rank sees the same global bound, so table layouts still agree.
      bool narrow = false;
      if constexpr (sizeof(CT) == 8) {
        if (p.mode == IG_MODE_ALL && !getenv("IG_FORCE_U64")) {
          uint64_t top = 0;
          d2h(s, &top, sc, sizeof(top));
          narrow = top < 0xffffffffull;
        }
      }
      ev = tm.begin();
      const uint64_t cap = 256 * ns;
      // fused histogram of the next pass's owners, sized for its largest
      // possible prefix count min(k', 256 * this pass's survivors)
      next_lg = fuse_lg >= 0 && j < n && j < 8
                    ? (int32_t)predicted_lgno(std::min<uint64_t>(kp, 256 * ns))
                    : -1;  // (passes j >= 9 do not route)
      if (next_lg > (int32_t)kMaxFusedLg) next_lg = -1;
      void* ct = nullptr;
      if (chain) {
        tcap = cap;
        km = KeyMap{};  // table index = id = key (byte order)
        auto go = [&](auto* tag) -> void* {
          using T = std::remove_pointer_t<decltype(tag)>;
          T* t = s.table.as<T>(tcap);
          IGB_CUDA(cudaMemsetAsync(t, 0, tcap * sizeof(T), s.stream));
          count_chain_exact<T>(s, j, ps8, static_cast<const uint32_t* const*>(s.chain_ptrs.p),
                               p.mode, tcap, t);
          IGB_CUDA(cudaGetLastError());
          allreduce_table<T>(s, t, tcap);
          return t;
        };
        ct = narrow ? go((uint32_t*)nullptr) : go((CT*)nullptr);
      } else if (narrow) {
        ct = count_pass<uint32_t>(s, false, j, p.mode, &P, tcap, km, next_lg);
        IGB_CUDA(cudaGetLastError());
        allreduce_table<uint32_t>(s, static_cast<uint32_t*>(ct), tcap);
      } else {
        ct = count_pass<CT>(s, false, j, p.mode, &P, tcap, km, next_lg);
        IGB_CUDA(cudaGetLastError());
        allreduce_table<CT>(s, static_cast<CT*>(ct), tcap);
      }
      int kbits = 8 * (int)j;
      if (chain) {
        kbits = 1;
        while (kbits < 64 && ((tcap - 1) >> kbits) != 0) ++kbits;
      }
      auto select = [&](uint64_t kk, uint64_t* ok, uint64_t* oc) {
        return narrow ? timed_select<uint32_t>(s, static_cast<uint32_t*>(ct), tcap, kk, km,
                                               kbits, ok, oc)
                      : timed_select<CT>(s, static_cast<CT*>(ct), tcap, kk, km, kbits, ok, oc);
      };
      tm.end(ev);
      rows.push_back(
          make_row(std::to_string(j) + "-gram pass", j, total_bytes, cap, 0, false, ev));

      ev = tm.begin();
      if (j < n) {
        uint64_t ncap = std::min<uint64_t>(kp, cap);
        uint64_t* nk = s.next_keys.as<uint64_t>(ncap + 1);
        uint64_t* nc = s.next_counts.as<uint64_t>(ncap + 1);
        uint64_t nn = select(kp, nk, nc);
        shrt = nn < kp;
        if (shrt)
          diag += "pass " + std::to_string(j) + " retained " + std::to_string(nn) +
                  " candidates (requested " + std::to_string(kp) + ")\n";
        s.surv_keys.swap(s.next_keys);
        s.surv_counts.swap(s.next_counts);
        sk = nk;
        sc = nc;
        ns = nn;
        if (j == 8) {  // the next pass walks ranks from these 8-byte survivors
          ps8 = build_prefix_set(s, sk, ns, 8);
          ns8 = ns;
        } else if (j > 8) {  // level j: survivor ids in id order, id -> rank
          if (s.chain_ids.size() <= j) {
            s.chain_ids.resize(j + 1);
            s.chain_remap.resize(j + 1);
          }
          if (!s.chain_ids[j]) s.chain_ids[j].reset(new DevBuf());
          if (!s.chain_remap[j]) s.chain_remap[j].reset(new DevBuf());
          uint64_t* sid = s.chain_ids[j]->as<uint64_t>(ns + 1);
          uint32_t* rk = s.chain_ranks.as<uint32_t>(2 * ns + 2);
          sort_keys_by_value(sk, (uint32_t)ns, kbits, sid, rk, rk + ns + 1, s.chain_sort_tmp,
                             s.stream);
          uint32_t* rm = s.chain_remap[j]->as<uint32_t>(tcap);
          IGB_CUDA(cudaMemsetAsync(rm, 0xff, tcap * sizeof(uint32_t), s.stream));
          launch_scatter_rank(sid, ns, rm, s.stream);
          s.launches += 3;
          remap_ptrs.push_back(rm);
          level_len.push_back(ns);
          const uint32_t** dp = s.chain_ptrs.as<const uint32_t*>(remap_ptrs.size());
          h2d(s, dp, remap_ptrs.data(), remap_ptrs.size() * sizeof(void*));
        } else {
          P = prepare_prefix(s, sk, ns, j, p.mode, owner_bits(next_lg, ns));
        }
        tm.end(ev);
        rows.push_back(make_row("top-zk " + std::to_string(j) + "-grams/trie building", j, 0, 0,
                                ns, shrt, ev));
      } else {
        uint64_t ocap = std::min<uint64_t>(p.k, cap);
        out_keys_d = s.next_keys.as<uint64_t>(ocap + 1);
        out_counts_d = s.next_counts.as<uint64_t>(ocap + 1);
        out_len = select(p.k, out_keys_d, out_counts_d);
        tm.end(ev);
        rows.push_back(
            make_row("top-k " + std::to_string(j) + "-grams", j, 0, 0, out_len, false, ev));
      }
    }
  }

  // ---- results to host
  out->len = out_len;
  out->gram_len = n;
  out->keys = (uint64_t*)malloc((out_len + 1) * sizeof(uint64_t));
  out->counts = (uint64_t*)malloc((out_len + 1) * sizeof(uint64_t));
  out->grams = (uint8_t*)malloc(out_len * n + 1);
  out->passes = (ig_pass_stat*)malloc(rows.size() * sizeof(ig_pass_stat));
  out->diagnostics = (char*)malloc(diag.size() + 1);
  if (!out->keys || !out->counts || !out->grams || !out->passes || !out->diagnostics)
    throw Error(IG_EINTERNAL, "host allocation failed");
  if (out_len) {
    d2h(s, out->keys, out_keys_d, out_len * sizeof(uint64_t));
    d2h(s, out->counts, out_counts_d, out_len * sizeof(uint64_t));
  }
  IGB_CUDA(cudaStreamSynchronize(s.stream));
  if (n <= 8) {
    for (uint64_t i = 0; i < out_len; ++i)
      for (uint32_t b = 0; b < n; ++b)
        out->grams[i * n + b] = (uint8_t)(out->keys[i] >> (8 * (n - 1 - b)));
  } else {
    // keys are ids p * 256 + last byte: walk each down the levels to its
    // first 8 bytes (the trie path, trie.cpp:139-160)
    std::vector<uint64_t> k8(ns8);
    if (ns8) d2h(s, k8.data(), ps8.pkeys, ns8 * sizeof(uint64_t));
    std::vector<std::vector<uint64_t>> lv(level_len.size());
    for (size_t L = 0; L < level_len.size(); ++L) {
      lv[L].resize(level_len[L]);
      if (level_len[L])
        d2h(s, lv[L].data(), s.chain_ids[9 + L]->p, level_len[L] * sizeof(uint64_t));
    }
    for (uint64_t i = 0; i < out_len; ++i) {
      uint8_t* g = out->grams + i * n;
      uint64_t id = out->keys[i];
      for (uint32_t L = n; L > 8; --L) {
        g[L - 1] = (uint8_t)(id & 255);
        const uint64_t r = id >> 8;  // rank at level L - 1
        id = L - 1 > 8 ? lv[L - 1 - 9][r] : k8[r];
      }
      for (uint32_t b = 0; b < 8; ++b) g[b] = (uint8_t)(id >> (8 * (7 - b)));
    }
    free(out->keys);
    out->keys = nullptr;  // n > 8: the grams do not fit packed u64 keys
  }
  for (size_t i = 0; i < rows.size(); ++i) {
    rows[i].st.seconds = tm.seconds(rows[i].ev);
    out->passes[i] = rows[i].st;
  }
  out->num_passes = (uint32_t)rows.size();
  s.kt.collect();
  memcpy(out->diagnostics, diag.c_str(), diag.size() + 1);
  s.launches += s.sel.launches - sel_before;
}

void run(Session& s, const ig_params& p, ig_result* out) {
  validate(p);
  if (!s.loaded) throw Error(IG_ECONFIG, "no corpus loaded");
  use_device(s);
  memset(out, 0, sizeof(*out));
  try {
    if (use_u32(s, p.mode)) run_t<uint32_t>(s, p, out);
    else run_t<unsigned long long>(s, p, out);
  } catch (...) {
    ig_result_free(out);
    throw;
  }
}

}  // namespace igb

using namespace igb;


namespace igb {
// Host corpus: offsets/units/tiles first, then the bytes in sequence-aligned
// batches on a copy stream (one event per batch); the dense pass consumes the
// batches as they land, so most of the H2D hides behind counting.
// Sequence-aligned batches of the loaded corpus (>= 256 MiB or 1/8 of it)
// for a dense pass that consumes the corpus as it lands: fills s.batches
// (one event each, not yet recorded) and returns each batch's byte end.
std::vector<uint64_t> plan_batches(Session& s) {
  const uint64_t m = s.dc.m, total = s.dc.total;
  // small batches shorten the dense-pass tail after the last byte lands
  // (measured on c2: 1/8 -> 1/32 of the corpus took 1.7 % off e2e)
  static const char* bb = getenv("IG_LOAD_BATCH_DIV");
  const uint64_t div = bb ? std::max<uint64_t>(1, strtoull(bb, nullptr, 10)) : 32;
  const uint64_t want = std::max<uint64_t>(16ull << 20, (total + div - 1) / div);
  s.batches.clear();
  std::vector<uint64_t> ends;
  uint64_t q = 0, prev_t1 = 0;
  size_t nb = 0;
  while (q < m || (m == 0 && nb == 0)) {
    const uint64_t q0 = q;
    const uint64_t b0 = s.hoff[q0];
    while (q < m && s.hoff[q + 1] - b0 < want) ++q;
    if (q == q0 && q < m) ++q;  // one long sequence
    const uint64_t b1 = s.hoff[q];
    if (nb >= s.batch_events.size()) {
      cudaEvent_t e;
      IGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s.batch_events.push_back(e);
    }
    Session::Batch b{};
    b.q0 = (uint32_t)q0;
    b.q1 = (uint32_t)q;
    b.u0 = s.hufirst[q0];
    b.u1 = s.hufirst[q];
    b.t0 = prev_t1;
    b.t1 = q >= m ? s.dc.ntiles : std::min<uint64_t>(s.dc.ntiles, b1 / kTileBytes);
    if (b.t1 < b.t0) b.t1 = b.t0;
    prev_t1 = b.t1;
    b.ready = s.batch_events[nb];
    s.batches.push_back(b);
    ends.push_back(b1);
    ++nb;
    if (m == 0) break;
  }
  return ends;
}

// Host corpus: offsets/units/tiles first, then the bytes in sequence-aligned
// batches on a copy stream (one event per batch); the dense pass consumes the
// batches as they land, so most of the H2D hides behind counting.
static bool page_locked(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static void load_and_run(Session& s, const ig_corpus& c, const ig_params& p, ig_result* out) {
  validate(p);
  if (c.location == IG_DEVICE) {
    load_corpus(s, c, true);
    run(s, p, out);
    return;
  }
  if (c.num_seqs && c.offsets[c.num_seqs] && !page_locked(c.data)) {
    // pageable: a DMA from it would stage synchronously before the run
    // starts; host threads stream it through pinned slabs instead
    std::vector<uint64_t> hoff(c.offsets, c.offsets + c.num_seqs + 1);
    run_host_streamed(s, c.data, nullptr, hoff, p, out);
    return;
  }
  load_corpus(s, c, false);
  if (!s.copy_stream) IGB_CUDA(cudaStreamCreateWithFlags(&s.copy_stream, cudaStreamNonBlocking));
  const std::vector<uint64_t> ends = plan_batches(s);
  uint64_t b0 = 0;
  for (size_t i = 0; i < ends.size(); ++i) {
    if (ends[i] > b0)
      IGB_CUDA(cudaMemcpyAsync(const_cast<uint8_t*>(s.dc.data) + b0, c.data + b0, ends[i] - b0,
                               cudaMemcpyHostToDevice, s.copy_stream));
    IGB_CUDA(cudaEventRecord(s.batches[i].ready, s.copy_stream));
    b0 = ends[i];
  }
  try {
    run(s, p, out);
  } catch (...) {
    s.batches.clear();
    throw;
  }
  s.batches.clear();
}

ig_session* create(int32_t device, void* stream, const ig_collective* coll) {
  ig_session* s = new ig_session();
  try {
    if (device < 0) IGB_CUDA(cudaGetDevice(&device));
    s->device = device;
    IGB_CUDA(cudaSetDevice(device));
    IGB_CUDA(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (stream) {
      s->stream = (cudaStream_t)stream;
    } else {
      IGB_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
      s->own_stream = true;
    }
    if (coll) {
      s->coll = *coll;
      s->has_coll = true;
    }
  } catch (...) {
    delete s;
    throw;
  }
  return s;
}

}  // namespace igb

extern "C" {

const char* ig_version(void) { return "intergrams-b200 0.1 (sm_100a)"; }

void ig_result_free(ig_result* r) {
  if (!r) return;
  free(r->keys);
  free(r->counts);
  free(r->grams);
  free(r->passes);
  free(r->diagnostics);
  r->keys = nullptr;
  r->counts = nullptr;
  r->passes = nullptr;
  r->diagnostics = nullptr;
  r->len = 0;
  r->num_passes = 0;
}

int ig_session_create(int32_t device, void* cuda_stream, const ig_collective* coll,
                      ig_session** out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!out) throw Error(IG_ECONFIG, "null session out-pointer");
    *out = create(device, cuda_stream, coll);
  });
}

int ig_session_load(ig_session* s, const ig_corpus* corpus, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!s || !corpus) throw Error(IG_ECONFIG, "null session or corpus");
    load_corpus(*s, *corpus);
  });
}

int ig_session_run_host(ig_session* s, const ig_corpus* corpus, const ig_params* params,
                        ig_result* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!s || !corpus || !params || !out) throw Error(IG_ECONFIG, "null argument");
    load_and_run(*s, *corpus, *params, out);
  });
}

int ig_session_run(ig_session* s, const ig_params* params, ig_result* out, char* err,
                   size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!s || !params || !out) throw Error(IG_ECONFIG, "null argument");
    run(*s, *params, out);
  });
}

uint64_t ig_session_launches(const ig_session* s) { return s ? s->launches : 0; }

void ig_session_set_profiling(ig_session* s, int32_t on) {
  if (s) s->kt.on = on != 0;
}

int ig_session_kernel_stats(ig_session* s, double* ms, uint64_t* launches, int32_t n, int32_t reset) {
  if (!s) return IG_ECONFIG;
  for (int i = 0; i < n && i < 8; ++i) {
    if (ms) ms[i] = s->kt.ms[i];
    if (launches) launches[i] = s->kt.n[i];
  }
  if (reset) s->kt.reset();
  return IG_OK;
}

void ig_session_destroy(ig_session* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  delete s;
}

}  // extern "C"

// One-shot entry points (ig_topk_ngrams*, the C++ run_intergrams) reuse an
// idle session per device instead of creating one per call: creating and
// destroying a session (stream, events, mapped pinned arena, every device
// buffer) costs ~0.1 s, which dominated a call on a small corpus.  A session
// that held a corpus above 1 GiB is destroyed instead of kept, so a finished
// large run does not pin its HBM; one that threw is never reused.
namespace igb {
namespace {
struct OneShotPool {
  std::mutex mu;
  std::map<int, ig_session*> idle;
  static OneShotPool& get() {
    static OneShotPool* p = new OneShotPool();
    return *p;
  }
};
}  // namespace

ig_session* acquire_oneshot(int32_t device) {
  if (device < 0) IGB_CUDA(cudaGetDevice(&device));
  {
    OneShotPool& p = OneShotPool::get();
    std::lock_guard<std::mutex> lk(p.mu);
    auto it = p.idle.find(device);
    if (it != p.idle.end() && it->second) {
      ig_session* s = it->second;
      it->second = nullptr;
      return s;
    }
  }
  return create(device, nullptr, nullptr);
}

void release_oneshot(ig_session* s) {
  if (!s) return;
  if (s->dc.total <= (1ull << 30) && !getenv("IG_NO_SESSION_POOL")) {
    OneShotPool& p = OneShotPool::get();
    std::lock_guard<std::mutex> lk(p.mu);
    ig_session*& slot = p.idle[s->device];
    if (!slot) {
      slot = s;
      return;
    }
  }
  ig_session_destroy(s);
}
}  // namespace igb

extern "C" {

int ig_topk_ngrams(const ig_corpus* corpus, const ig_params* params, ig_result* out, char* err,
                   size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!corpus || !params || !out) throw Error(IG_ECONFIG, "null argument");
    validate(*params);
    ig_session* s = acquire_oneshot(params->device);
    try {
      load_and_run(*s, *corpus, *params, out);
    } catch (...) {
      delete s;
      throw;
    }
    release_oneshot(s);
  });
}

int ig_topk_ngrams_seqs(const uint8_t* const* seqs, const uint64_t* lens, uint64_t num_seqs,
                        const ig_params* params, ig_result* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if ((num_seqs && (!seqs || !lens)) || !params || !out) throw Error(IG_ECONFIG, "null argument");
    validate(*params);
    std::vector<uint64_t> hoff(num_seqs + 1, 0);
    for (uint64_t q = 0; q < num_seqs; ++q) {
      if (lens[q] && !seqs[q]) throw Error(IG_ECONFIG, "null sequence pointer");
      hoff[q + 1] = hoff[q] + lens[q];
    }
    ig_session* s = acquire_oneshot(params->device);
    try {
      if (hoff[num_seqs]) {
        run_host_streamed(*s, nullptr, seqs, hoff, *params, out);
      } else {  // no bytes: the ordinary path (empty-corpus semantics)
        static const uint8_t none = 0;
        ig_corpus c{&none, hoff.data(), num_seqs, IG_HOST};
        load_and_run(*s, c, *params, out);
      }
    } catch (...) {
      delete s;
      throw;
    }
    release_oneshot(s);
  });
}

int ig_count_dense(const ig_corpus* corpus, uint32_t n, int32_t mode, int32_t device,
                   uint64_t* table_out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    // dense_capacity, dense_pass.cpp:5-10
    if (n < 1 || n > 3) throw Error(IG_ECONFIG, "dense pass supports gram lengths 1..3");
    if (mode != IG_MODE_ONCE && mode != IG_MODE_ALL) throw Error(IG_ECONFIG, "bad count mode");
    ig_session* s = create(device, nullptr, nullptr);
    try {
      load_corpus(*s, *corpus);
      const uint64_t cap = 1ull << (8 * n);
      uint64_t tcap = 0;
      KeyMap km;
      unsigned long long* t = count_pass<unsigned long long>(*s, true, n, mode, nullptr, tcap, km);
      IGB_CUDA(cudaGetLastError());
      std::vector<uint64_t> tab(tcap);
      IGB_CUDA(cudaMemcpyAsync(tab.data(), t, tcap * 8, cudaMemcpyDeviceToHost, s->stream));
      IGB_CUDA(cudaStreamSynchronize(s->stream));
      // back to the reference layout: table index = dense id (dense_pass.cpp:12-19)
      if (km.minv) {
        // index = (id * mult) & cmask; recover mult from minv
        uint64_t mult = km.minv;
        for (int it = 0; it < 6; ++it) mult *= 2ull - km.minv * mult;
        mult &= km.cmask;
        for (uint64_t id = 0; id < cap; ++id) table_out[id] = tab[(id * mult) & km.cmask];
      } else {
        memcpy(table_out, tab.data(), cap * 8);
      }
    } catch (...) {
      delete s;
      throw;
    }
    delete s;
  });
}

int ig_extend_pass(const ig_corpus* corpus, const uint64_t* prefix_keys, uint64_t nprefix,
                   uint32_t prefix_len, uint32_t j, int32_t mode, int32_t device,
                   uint64_t* table_out, uint64_t* bytes_processed, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const uint32_t depth = nprefix ? prefix_len : 0;  // trie.cpp:23
    if (j < 2 || depth != j - 1)  // intergrams.cpp:46-48
      throw Error(IG_ECONFIG, "extension pass needs a trie of depth j-1");
    if (j > IG_MAX_N) throw Error(IG_ECONFIG, "gram length above 8 is not supported");
    if (mode != IG_MODE_ONCE && mode != IG_MODE_ALL) throw Error(IG_ECONFIG, "bad count mode");
    {  // PrefixTrie::build rejects duplicates (trie.cpp:45-46)
      std::vector<uint64_t> v(prefix_keys, prefix_keys + nprefix);
      std::sort(v.begin(), v.end());
      if (std::adjacent_find(v.begin(), v.end()) != v.end())
        throw Error(IG_EINVALID, "duplicate prefix in trie input");
    }
    ig_session* s = create(device, nullptr, nullptr);
    try {
      load_corpus(*s, *corpus);
      uint64_t* dk = s->surv_keys.as<uint64_t>(nprefix + 1);
      IGB_CUDA(cudaMemcpyAsync(dk, prefix_keys, nprefix * 8, cudaMemcpyHostToDevice, s->stream));
      Prefix P = prepare_prefix(*s, dk, nprefix, prefix_len, mode);
      uint64_t tcap = 0;
      KeyMap km;
      unsigned long long* t = count_pass<unsigned long long>(*s, false, j, mode, &P, tcap, km);
      IGB_CUDA(cudaGetLastError());
      std::vector<uint64_t> tab(tcap);
      IGB_CUDA(cudaMemcpyAsync(tab.data(), t, tcap * 8, cudaMemcpyDeviceToHost, s->stream));
      std::vector<uint32_t> rank;  // p -> survivor rank
      if (P.csr) {
        rank = P.rank_of_p;
      } else {
        rank.resize(nprefix);
        IGB_CUDA(cudaMemcpyAsync(rank.data(), s->rank_of_p.p, nprefix * 4,
                                 cudaMemcpyDeviceToHost, s->stream));
      }
      IGB_CUDA(cudaStreamSynchronize(s->stream));
      uint64_t mult = 1;
      if (km.minv) {
        mult = km.minv;
        for (int it = 0; it < 6; ++it) mult *= 2ull - km.minv * mult;
        mult &= km.cmask;
      }
      // back to the reference layout: ordinal (rank) * 256 + last byte (candidate_id)
      memset(table_out, 0, nprefix * 256 * 8);
      for (uint64_t p = 0; p < rank.size(); ++p) {
        if (rank[p] == 0xffffffffu) continue;  // no prefix at this p
        for (uint64_t b = 0; b < 256; ++b) {
          const uint64_t id = p * 256 + b;
          table_out[(uint64_t)rank[p] * 256 + b] = tab[km.minv ? ((id * mult) & km.cmask) : id];
        }
      }
      if (bytes_processed) *bytes_processed = s->dc.total;
    } catch (...) {
      delete s;
      throw;
    }
    delete s;
  });
}

int ig_top_k(const uint64_t* table, uint64_t cap, uint64_t k, const uint64_t* prefix_keys,
             int32_t device, uint64_t* keys_out, uint64_t* counts_out, uint64_t* len_out,
             char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (k < 1) throw Error(IG_ECONFIG, "top_k requires k >= 1");  // counting.cpp:54
    ig_session* s = create(device, nullptr, nullptr);
    try {
      init_select(*s);
      const uint64_t cap4 = (cap + 255) / 256 * 256;
      unsigned long long* t = s->table.as<unsigned long long>(cap4);
      IGB_CUDA(cudaMemsetAsync(t, 0, cap4 * 8, s->stream));
      IGB_CUDA(cudaMemcpyAsync(t, table, cap * 8, cudaMemcpyHostToDevice, s->stream));
      uint64_t* pk = nullptr;
      int key_bits = 64;
      if (prefix_keys) {
        const uint64_t np = cap4 / 256;
        pk = s->pkeys.as<uint64_t>(np);
        IGB_CUDA(cudaMemsetAsync(pk, 0, np * 8, s->stream));
        IGB_CUDA(cudaMemcpyAsync(pk, prefix_keys, (cap + 255) / 256 * 8, cudaMemcpyHostToDevice,
                                 s->stream));
      } else {
        key_bits = 0;
        while (key_bits < 64 && (1ull << key_bits) < cap4) ++key_bits;
      }
      const uint64_t kk = std::min<uint64_t>(k, cap4);
      uint64_t* ok = s->next_keys.as<uint64_t>(kk + 1);
      uint64_t* oc = s->next_counts.as<uint64_t>(kk + 1);
      KeyMap km;
      km.pkeys = pk;
      const uint64_t n = select_topk<unsigned long long>(s->sel, t, cap4, kk, km, key_bits, ok, oc);
      if (n) {
        IGB_CUDA(cudaMemcpyAsync(keys_out, ok, n * 8, cudaMemcpyDeviceToHost, s->stream));
        IGB_CUDA(cudaMemcpyAsync(counts_out, oc, n * 8, cudaMemcpyDeviceToHost, s->stream));
      }
      IGB_CUDA(cudaStreamSynchronize(s->stream));
      *len_out = n;
    } catch (...) {
      delete s;
      throw;
    }
    delete s;
  });
}

void ig_shard_range(const uint64_t* offsets, uint64_t num_seqs, int32_t rank, int32_t world,
                    uint64_t* first, uint64_t* last) {
  // cut r: the sequence boundary nearest r*total/world (ties to the lower)
  auto cut = [&](int32_t r) -> uint64_t {
    if (r <= 0) return 0;
    if (r >= world) return num_seqs;
    const uint64_t total = offsets[num_seqs];
    const unsigned __int128 target128 = (unsigned __int128)total * (uint64_t)r / (uint64_t)world;
    const uint64_t target = (uint64_t)target128;
    const uint64_t* it = std::lower_bound(offsets, offsets + num_seqs + 1, target);
    uint64_t i = (uint64_t)(it - offsets);
    if (i > num_seqs) i = num_seqs;
    if (i > 0 && (offsets[i] - target) > (target - offsets[i - 1])) --i;
    return i;
  };
  if (world < 1) world = 1;
  uint64_t a = cut(rank), b = cut(rank + 1);
  if (b < a) b = a;
  *first = a;
  *last = b;
}

}  // extern "C"

// ---- IG_GUARD self-test: a kernel writes byte `at` of a 100-byte buffer
// (at >= 100: past its end, at < 0: before it); the guard check must report
// exactly the out-of-bounds writes.
namespace igb {
__global__ void k_poke(uint8_t* p, int64_t at) { p[at] = 0x5A; }
}  // namespace igb

extern "C" int ig_guard_selftest(int32_t device, int64_t at, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!guard_mode()) throw Error(IG_ECONFIG, "IG_GUARD is not set");
    IGB_CUDA(cudaSetDevice(device));
    DevBuf b;
    uint8_t* p = b.as<uint8_t>(100);
    k_poke<<<1, 1>>>(p, at);
    IGB_CUDA(cudaGetLastError());
    check_guards("self-test");
  });
}
