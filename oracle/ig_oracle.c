/* ig_oracle.c — TEST INFRASTRUCTURE ONLY (see ig_oracle.h).
 *
 * Single-threaded C restatement of the reference hot path.  Every function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Worker counts, merge strategies and the trie node
 * layout are performance details of the reference that never change results
 * (tests/test_dense_pass.cpp:141-161, tests/test_trie.cpp:134-150), so the
 * restatement uses the simplest sequential equivalents: a per-sequence epoch
 * stamp for count-once dedup (SeenBitset + flush_batch, counting.hpp:48-74,
 * counting.cpp:27-50) and a sorted (key, rank) array for the prefix trie
 * (trie.cpp:20-151).
 */
#include "ig_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- mt19937_64
 * The standard 64-bit Mersenne Twister (std::mt19937_64), used by the
 * reference tests' random corpora (tests/helpers.hpp:46-65). */
void igo_mt64_seed(igo_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  }
  r->idx = 312;
}

uint64_t igo_mt64_next(igo_mt64* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static void set_err(char* err, size_t len, const char* msg) {
  if (err && len) {
    strncpy(err, msg, len - 1);
    err[len - 1] = 0;
  }
}

/* ------------------------------------------------------------ count sinks
 * ALL: table[id] += 1 per occurrence (pipeline.hpp:106-113,
 * counting.hpp:89-92).  ONCE: a gram adds 1 per sequence containing it
 * (counting.hpp:48-74 mark, counting.cpp:27-50 flush): stamp[id] records the
 * last sequence (1-based) that counted id. */
typedef struct {
  int mode;
  uint64_t* table;
  uint32_t* stamp;
  uint32_t epoch;
} sink_t;

static inline void sink_emit(sink_t* s, uint64_t id) {
  if (s->mode == IGO_ALL) {
    s->table[id] += 1;
  } else if (s->stamp[id] != s->epoch) {
    s->stamp[id] = s->epoch;
    s->table[id] += 1;
  }
}

static int sink_init(sink_t* s, int mode, uint64_t* table, uint64_t cap) {
  s->mode = mode;
  s->table = table;
  s->stamp = NULL;
  s->epoch = 0;
  memset(table, 0, cap * sizeof(uint64_t));
  if (mode == IGO_ONCE && cap) {
    s->stamp = (uint32_t*)calloc(cap, sizeof(uint32_t));
    if (!s->stamp) return IGO_INTERNAL;
  }
  return IGO_OK;
}

/* ------------------------------------------------------------ dense pass
 * dense_pass.cpp:21-39 / intergrams.cpp:84-98: rolling big-endian id over
 * n bytes, masked to 256^n - 1, one emit per position i >= n-1. */
int igo_count_dense(const uint8_t* data, const uint64_t* off, uint64_t m,
                    uint32_t n, int mode, uint64_t* table) {
  if (n < 1 || n > 3) return IGO_CONFIG; /* dense_pass.cpp:5-10 */
  const uint64_t cap = 1ULL << (8 * n), mask = cap - 1;
  sink_t s;
  if (sink_init(&s, mode, table, cap)) return IGO_INTERNAL;
  for (uint64_t q = 0; q < m; ++q) {
    const uint8_t* b = data + off[q];
    const uint64_t len = off[q + 1] - off[q];
    s.epoch = (uint32_t)(q + 1);
    if (len < n) continue;
    uint64_t id = 0;
    for (uint64_t i = 0; i + 1 < n; ++i) id = (id << 8) | b[i];
    for (uint64_t i = n - 1; i < len; ++i) {
      id = ((id << 8) | b[i]) & mask;
      sink_emit(&s, id);
    }
  }
  free(s.stamp);
  return IGO_OK;
}

/* ------------------------------------------------------------ top-k
 * counting.cpp:52-98: canonical top-k of nonzero entries — count
 * descending, then gram bytes ascending (canonical_less, counting.hpp:38-41).
 * All grams of one table share a length, so gram order == key order. */
typedef struct {
  uint64_t count, key;
} entry_t;

/* a ranks strictly before b in canonical order */
static inline int better(const entry_t* a, const entry_t* b) {
  if (a->count != b->count) return a->count > b->count;
  return a->key < b->key;
}

static void heap_down(entry_t* h, uint64_t n, uint64_t i) {
  /* min-heap on canonical order: h[0] is the worst kept entry */
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, w = i;
    if (l < n && better(&h[w], &h[l])) w = l;
    if (r < n && better(&h[w], &h[r])) w = r;
    if (w == i) return;
    entry_t t = h[i];
    h[i] = h[w];
    h[w] = t;
    i = w;
  }
}

static void heap_up(entry_t* h, uint64_t i) {
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (!better(&h[p], &h[i])) return;
    entry_t t = h[i];
    h[i] = h[p];
    h[p] = t;
    i = p;
  }
}

static int cmp_canonical(const void* pa, const void* pb) {
  const entry_t* a = (const entry_t*)pa;
  const entry_t* b = (const entry_t*)pb;
  if (better(a, b)) return -1;
  if (better(b, a)) return 1;
  return 0;
}

uint64_t igo_top_k(const uint64_t* table, uint64_t cap, uint64_t k,
                   const uint64_t* prefix_keys, uint64_t* out_keys,
                   uint64_t* out_counts) {
  if (k == 0) return 0;
  uint64_t hcap = k < cap ? k : cap;
  entry_t* h = (entry_t*)malloc((hcap ? hcap : 1) * sizeof(entry_t));
  uint64_t n = 0;
  for (uint64_t id = 0; id < cap; ++id) {
    if (table[id] == 0) continue; /* counting.cpp:72 */
    entry_t e;
    e.count = table[id];
    e.key = prefix_keys ? ((prefix_keys[id >> 8] << 8) | (id & 255)) : id;
    if (n < hcap) {
      h[n] = e;
      heap_up(h, n++);
    } else if (better(&e, &h[0])) { /* counting.cpp:78-87 */
      h[0] = e;
      heap_down(h, n, 0);
    }
  }
  qsort(h, n, sizeof(entry_t), cmp_canonical); /* counting.cpp:90-97 */
  for (uint64_t i = 0; i < n; ++i) {
    out_keys[i] = h[i].key;
    out_counts[i] = h[i].count;
  }
  free(h);
  return n;
}

/* ------------------------------------------------------------ prefix set
 * PrefixTrie semantics (trie.hpp:18-73, trie.cpp:139-151): window -> rank
 * ordinal, absent otherwise.  Restated as binary search over (key, rank). */
typedef struct {
  uint64_t key;
  uint64_t rank;
} kr_t;

static int cmp_kr(const void* pa, const void* pb) {
  const kr_t* a = (const kr_t*)pa;
  const kr_t* b = (const kr_t*)pb;
  return a->key < b->key ? -1 : a->key > b->key ? 1 : 0;
}

static int64_t kr_find(const kr_t* s, uint64_t n, uint64_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (s[mid].key < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && s[lo].key == key) ? (int64_t)s[lo].rank : -1;
}

/* ------------------------------------------------------------ extension pass
 * intergrams.cpp:44-66. */
int igo_extend_pass(const uint8_t* data, const uint64_t* off, uint64_t m,
                    const uint64_t* prefix_keys, uint64_t nprefix,
                    uint32_t prefix_len, uint32_t j, int mode, uint64_t* table,
                    uint64_t* bytes_processed) {
  const uint32_t depth = nprefix ? prefix_len : 0; /* trie.cpp:23 */
  if (j < 2 || depth != j - 1) return IGO_CONFIG; /* intergrams.cpp:46-48 */
  if (j > 8) return IGO_CONFIG;
  const uint64_t cap = 256 * nprefix; /* intergrams.cpp:49 */
  kr_t* set = (kr_t*)malloc(nprefix * sizeof(kr_t));
  for (uint64_t r = 0; r < nprefix; ++r) {
    set[r].key = prefix_keys[r];
    set[r].rank = r;
  }
  qsort(set, nprefix, sizeof(kr_t), cmp_kr);
  for (uint64_t r = 1; r < nprefix; ++r) {
    if (set[r].key == set[r - 1].key) { /* trie.cpp:45-46 */
      free(set);
      return IGO_CONFIG;
    }
  }
  sink_t s;
  if (sink_init(&s, mode, table, cap)) {
    free(set);
    return IGO_INTERNAL;
  }
  const uint64_t wmask = (j - 1) == 8 ? ~0ULL : ((1ULL << (8 * (j - 1))) - 1);
  uint64_t bytes = 0;
  for (uint64_t q = 0; q < m; ++q) {
    const uint8_t* b = data + off[q];
    const uint64_t len = off[q + 1] - off[q];
    s.epoch = (uint32_t)(q + 1);
    bytes += len; /* intergrams.cpp:53 */
    if (len < j) continue; /* intergrams.cpp:54 */
    uint64_t w = 0;
    for (uint32_t i = 0; i + 1 < j - 1; ++i) w = (w << 8) | b[i];
    for (uint64_t pos = 0; pos + j <= len; ++pos) {
      w = ((w << 8) | b[pos + j - 2]) & wmask; /* window b[pos..pos+j-2] */
      int64_t ord = kr_find(set, nprefix, w);
      if (ord < 0) continue;
      sink_emit(&s, (uint64_t)ord * 256 + b[pos + j - 1]); /* candidate_id */
    }
  }
  if (bytes_processed) *bytes_processed = bytes;
  free(s.stamp);
  free(set);
  return IGO_OK;
}

/* ------------------------------------------------------------ driver
 * run_intergrams, intergrams.cpp:68-166. */
static void add_pass(igo_pass* p, uint32_t* np, const char* label,
                     uint32_t gl, uint64_t bytes, uint64_t cap,
                     uint64_t retained, int shrt) {
  igo_pass* r = &p[(*np)++];
  memset(r, 0, sizeof(*r));
  snprintf(r->label, sizeof(r->label), "%s", label);
  r->gram_len = gl;
  r->bytes_processed = bytes;
  r->candidate_space = cap;
  r->retained = retained;
  r->retained_short = shrt;
}

static void add_diag(char* diag, size_t len, uint32_t pass, uint64_t got,
                     uint64_t want) {
  if (!diag || !len) return;
  size_t used = strlen(diag);
  snprintf(diag + used, len - used,
           "pass %u retained %llu candidates (requested %llu)\n", pass,
           (unsigned long long)got, (unsigned long long)want);
}

int igo_run_intergrams(const uint8_t* data, const uint64_t* off, uint64_t m,
                       uint32_t n, uint64_t k, double z, int mode,
                       uint64_t* out_keys, uint64_t* out_counts,
                       uint64_t* out_len, igo_pass* passes,
                       uint32_t* num_passes, char* diag, size_t diag_len,
                       char* err, size_t err_len) {
  /* IntergramConfig::validate, intergrams.cpp:37-42 */
  if (n < 1) { set_err(err, err_len, "gram length n must be >= 1"); return IGO_CONFIG; }
  if (k < 1) { set_err(err, err_len, "k must be >= 1"); return IGO_CONFIG; }
  if (!(z >= 1.0)) { set_err(err, err_len, "oversample factor z must be >= 1"); return IGO_CONFIG; }
  if (n > 8) { set_err(err, err_len, "oracle supports n <= 8"); return IGO_CONFIG; }
  double kpd = ceil(z * (double)k); /* k_prime, intergrams.hpp:29-31 */
  const uint64_t kp = kpd >= 9.2e18 ? (uint64_t)9.2e18 : (uint64_t)kpd;
  uint32_t np = 0;
  if (diag && diag_len) diag[0] = 0;
  *out_len = 0;

  const uint32_t n0 = n < 3 ? n : 3; /* intergrams.cpp:76 */
  const uint64_t dcap = 1ULL << (8 * n0);
  uint64_t* table = (uint64_t*)malloc(dcap * sizeof(uint64_t));
  if (igo_count_dense(data, off, m, n0, mode, table)) { free(table); return IGO_INTERNAL; }
  uint64_t total = off[m] - off[0];
  char label[48];
  snprintf(label, sizeof label, "%u-gram pass", n0);
  add_pass(passes, &np, label, n0, total, dcap, 0, 0);

  if (n <= 3) { /* intergrams.cpp:105-113 */
    uint64_t got = igo_top_k(table, dcap, k, NULL, out_keys, out_counts);
    *out_len = got;
    snprintf(label, sizeof label, "top-k %u-grams", n);
    add_pass(passes, &np, label, n, 0, 0, got, 0);
    free(table);
    *num_passes = np;
    return IGO_OK;
  }

  /* survivors = topk_trigrams(table, k') (intergrams.cpp:115-116) */
  uint64_t scap = kp < dcap ? kp : dcap;
  uint64_t* skeys = (uint64_t*)malloc((scap ? scap : 1) * sizeof(uint64_t));
  uint64_t* scnt = (uint64_t*)malloc((scap ? scap : 1) * sizeof(uint64_t));
  uint64_t ns = igo_top_k(table, dcap, kp, NULL, skeys, scnt);
  free(table);
  int shrt = ns < kp;
  if (shrt) add_diag(diag, diag_len, 3, ns, kp);
  add_pass(passes, &np, "top-zk 3-grams/trie building", 3, 0, 0, ns, shrt);

  int rc = IGO_OK;
  for (uint32_t j = 4; j <= n; ++j) {
    const uint64_t cap = 256 * ns;
    uint64_t* counts = (uint64_t*)malloc((cap ? cap : 1) * sizeof(uint64_t));
    uint64_t bytes = 0;
    rc = igo_extend_pass(data, off, m, skeys, ns, ns ? j - 1 : 0, j, mode,
                         counts, &bytes);
    if (rc) {
      free(counts);
      set_err(err, err_len, "extension pass needs a trie of depth j-1");
      break;
    }
    snprintf(label, sizeof label, "%u-gram pass", j);
    add_pass(passes, &np, label, j, bytes, cap, 0, 0);
    if (j < n) {
      uint64_t ncap = kp < cap ? kp : cap;
      uint64_t* nk = (uint64_t*)malloc((ncap ? ncap : 1) * sizeof(uint64_t));
      uint64_t* nc = (uint64_t*)malloc((ncap ? ncap : 1) * sizeof(uint64_t));
      uint64_t nn = igo_top_k(counts, cap, kp, skeys, nk, nc);
      shrt = nn < kp;
      if (shrt) add_diag(diag, diag_len, j, nn, kp);
      free(skeys);
      free(scnt);
      skeys = nk;
      scnt = nc;
      ns = nn;
      snprintf(label, sizeof label, "top-zk %u-grams/trie building", j);
      add_pass(passes, &np, label, j, 0, 0, ns, shrt);
    } else {
      uint64_t got = igo_top_k(counts, cap, k, skeys, out_keys, out_counts);
      *out_len = got;
      snprintf(label, sizeof label, "top-k %u-grams", j);
      add_pass(passes, &np, label, j, 0, 0, got, 0);
    }
    free(counts);
  }
  free(skeys);
  free(scnt);
  *num_passes = np;
  return rc;
}

/* ------------------------------------------------------------ naive oracle
 * naive_count + naive_topk, oracle.cpp:7-47 (exact dictionary counting of
 * Eq. 1 / Eq. 2), restated as sort + run-length over packed keys. */
static int cmp_u64(const void* pa, const void* pb) {
  uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
  return a < b ? -1 : a > b ? 1 : 0;
}

int igo_naive_topk(const uint8_t* data, const uint64_t* off, uint64_t m,
                   uint32_t n, int mode, uint64_t k, uint64_t* out_keys,
                   uint64_t* out_counts, uint64_t* out_len) {
  if (n < 1 || n > 8 || k < 1) return IGO_CONFIG;
  uint64_t total = 0;
  for (uint64_t q = 0; q < m; ++q) {
    uint64_t len = off[q + 1] - off[q];
    if (len >= n) total += len - n + 1;
  }
  uint64_t* keys = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
  uint64_t nk = 0;
  const uint64_t mask = n == 8 ? ~0ULL : ((1ULL << (8 * n)) - 1);
  for (uint64_t q = 0; q < m; ++q) {
    const uint8_t* b = data + off[q];
    uint64_t len = off[q + 1] - off[q];
    if (len < n) continue;
    uint64_t start = nk, w = 0;
    for (uint64_t i = 0; i < len; ++i) {
      w = ((w << 8) | b[i]) & mask;
      if (i + 1 >= n) keys[nk++] = w;
    }
    if (mode == IGO_ONCE) { /* per-sequence set, oracle.cpp:22-29 */
      qsort(keys + start, nk - start, sizeof(uint64_t), cmp_u64);
      uint64_t u = start;
      for (uint64_t i = start; i < nk; ++i)
        if (i == start || keys[i] != keys[i - 1]) keys[u++] = keys[i];
      nk = u;
    }
  }
  qsort(keys, nk, sizeof(uint64_t), cmp_u64);
  entry_t* e = (entry_t*)malloc((nk ? nk : 1) * sizeof(entry_t));
  uint64_t ne = 0;
  for (uint64_t i = 0; i < nk;) {
    uint64_t j = i;
    while (j < nk && keys[j] == keys[i]) ++j;
    e[ne].key = keys[i];
    e[ne].count = j - i;
    ++ne;
    i = j;
  }
  qsort(e, ne, sizeof(entry_t), cmp_canonical); /* naive_topk, oracle.cpp:37-47 */
  uint64_t out = ne < k ? ne : k;
  for (uint64_t i = 0; i < out; ++i) {
    out_keys[i] = e[i].key;
    out_counts[i] = e[i].count;
  }
  *out_len = out;
  free(keys);
  free(e);
  return IGO_OK;
}

/* ------------------------------------------------------ hash-gramming
 * The two-pass baseline (run_hashgram, hashgram.cpp:325-383).  Bucket
 * tables are kept sparse here (sorted bucket ids), which gives the same
 * counts as the reference's dense CountTable(B). */

/* mix64, hashgram.cpp:22-59 (MurmurHash64A over little-endian 8-byte blocks). */
uint64_t igo_mix64(const uint8_t* bytes, uint64_t len, uint64_t seed) {
  const uint64_t mm = 0xc6a4a7935bd1e995ULL;
  const int r = 47;
  uint64_t h = seed ^ (len * mm);
  while (len >= 8) {
    uint64_t k = 0;
    for (int b = 7; b >= 0; --b) k = (k << 8) | bytes[b];
    k *= mm;
    k ^= k >> r;
    k *= mm;
    h ^= k;
    h *= mm;
    bytes += 8;
    len -= 8;
  }
  uint64_t tail = 0;
  for (uint64_t i = len; i-- > 0;) tail = (tail << 8) | bytes[i];
  if (len > 0) {
    h ^= tail;
    h *= mm;
  }
  h ^= h >> r;
  h *= mm;
  h ^= h >> r;
  return h;
}

typedef struct {
  uint32_t n;
  uint64_t seed, buckets;
  const uint64_t* kept; /* sorted kept buckets (pass 2), or NULL */
  uint64_t nkept;
  int bucket_ids;       /* 1: emit bucket ids (pass 1), 0: emit gram keys */
} hg_ctx;

static int kept_has(const hg_ctx* c, uint64_t b) {
  uint64_t lo = 0, hi = c->nkept;
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (c->kept[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  return lo < c->nkept && c->kept[lo] == b;
}

/* Exact counts of the ids a hash-gramming pass emits; ONCE dedups per
 * sequence (count_sequences' SeenBitset for pass 1, the last-seen stamp of
 * MapDictionary for pass 2, hashgram.cpp:136-148).  Returns entries sorted
 * by id; *ne receives their number. */
static entry_t* hg_count(const uint8_t* data, const uint64_t* off, uint64_t m,
                         int mode, const hg_ctx* c, uint64_t* ne) {
  const uint32_t n = c->n;
  uint64_t total = 0;
  for (uint64_t q = 0; q < m; ++q) {
    uint64_t len = off[q + 1] - off[q];
    if (len >= n) total += len - n + 1;
  }
  uint64_t* ids = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
  uint64_t ni = 0;
  for (uint64_t q = 0; q < m; ++q) {
    const uint8_t* b = data + off[q];
    uint64_t len = off[q + 1] - off[q];
    if (len < n) continue;
    uint64_t start = ni;
    for (uint64_t pos = 0; pos + n <= len; ++pos) {
      uint64_t bucket = igo_mix64(b + pos, n, c->seed) % c->buckets;
      if (c->bucket_ids) {
        ids[ni++] = bucket;
      } else if (kept_has(c, bucket)) {
        uint64_t key = 0;
        for (uint32_t i = 0; i < n; ++i) key = (key << 8) | b[pos + i];
        ids[ni++] = key;
      }
    }
    if (mode == IGO_ONCE) {
      qsort(ids + start, ni - start, sizeof(uint64_t), cmp_u64);
      uint64_t u = start;
      for (uint64_t i = start; i < ni; ++i)
        if (i == start || ids[i] != ids[i - 1]) ids[u++] = ids[i];
      ni = u;
    }
  }
  qsort(ids, ni, sizeof(uint64_t), cmp_u64);
  entry_t* e = (entry_t*)malloc((ni ? ni : 1) * sizeof(entry_t));
  uint64_t k = 0;
  for (uint64_t i = 0; i < ni;) {
    uint64_t j = i;
    while (j < ni && ids[j] == ids[i]) ++j;
    e[k].key = ids[i];
    e[k].count = j - i;
    ++k;
    i = j;
  }
  free(ids);
  *ne = k;
  return e;
}

int igo_hashgram_topk(const uint8_t* data, const uint64_t* off, uint64_t m,
                      uint32_t n, uint64_t k, int mode, uint64_t buckets,
                      uint64_t seed, uint64_t* out_keys, uint64_t* out_counts,
                      uint64_t* out_len, uint64_t* kept_buckets,
                      uint64_t* exact_size) {
  if (buckets < 1 || n < 1 || k < 1 || n > 8) return IGO_CONFIG; /* :16-20 */
  hg_ctx c = {n, seed, buckets, NULL, 0, 1};
  uint64_t ne = 0;
  entry_t* e = hg_count(data, off, m, mode, &c, &ne); /* pass 1, :336-351 */
  qsort(e, ne, sizeof(entry_t), cmp_canonical);      /* topk_buckets, :74-98 */
  uint64_t nk = ne < k ? ne : k;
  uint64_t* kept = (uint64_t*)malloc((nk ? nk : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < nk; ++i) kept[i] = e[i].key;
  free(e);
  qsort(kept, nk, sizeof(uint64_t), cmp_u64);
  *kept_buckets = nk;
  c.bucket_ids = 0;
  c.kept = kept;
  c.nkept = nk;
  e = hg_count(data, off, m, mode, &c, &ne); /* pass 2, :364-375 */
  *exact_size = ne;
  qsort(e, ne, sizeof(entry_t), cmp_canonical); /* naive_topk, :377-380 */
  uint64_t out = ne < k ? ne : k;
  for (uint64_t i = 0; i < out; ++i) {
    out_keys[i] = e[i].key;
    out_counts[i] = e[i].count;
  }
  *out_len = out;
  free(e);
  free(kept);
  return IGO_OK;
}

/* ---------------------------------------------------------- featurize
 * metrics.cpp:83-132: entry (row, col) when vocabulary gram col occurs in
 * sequence row; a repeated vocabulary gram keeps its first column
 * (columns.emplace, :101-104).  Entries sorted by row then col (:130).
 * Returns a malloc'd array of (row << 32 | col) (free with igo_free). */
uint64_t* igo_featurize(const uint8_t* data, const uint64_t* off, uint64_t m,
                        const uint64_t* vocab, uint64_t ncols, uint32_t n,
                        uint64_t* nnz) {
  /* sorted (key, first column) pairs */
  entry_t* v = (entry_t*)malloc((ncols ? ncols : 1) * sizeof(entry_t));
  for (uint64_t j = 0; j < ncols; ++j) {
    v[j].key = vocab[j];
    v[j].count = j; /* column */
  }
  /* stable by key then column: sort on (key, column) */
  for (uint64_t a = 1; a < ncols; ++a) { /* insertion sort is fine for tests */
    entry_t t = v[a];
    uint64_t b = a;
    while (b > 0 && (v[b - 1].key > t.key ||
                     (v[b - 1].key == t.key && v[b - 1].count > t.count))) {
      v[b] = v[b - 1];
      --b;
    }
    v[b] = t;
  }
  uint64_t cap = 1024, cnt = 0;
  uint64_t* out = (uint64_t*)malloc(cap * sizeof(uint64_t));
  for (uint64_t q = 0; q < m && ncols; ++q) {
    const uint8_t* b = data + off[q];
    uint64_t len = off[q + 1] - off[q];
    if (len < n) continue;
    uint64_t start = cnt;
    for (uint64_t pos = 0; pos + n <= len; ++pos) {
      uint64_t key = 0;
      for (uint32_t i = 0; i < n; ++i) key = (key << 8) | b[pos + i];
      uint64_t lo = 0, hi = ncols;
      while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (v[mid].key < key) lo = mid + 1;
        else hi = mid;
      }
      if (lo < ncols && v[lo].key == key) {
        if (cnt == cap) {
          cap *= 2;
          out = (uint64_t*)realloc(out, cap * sizeof(uint64_t));
        }
        out[cnt++] = (q << 32) | v[lo].count;
      }
    }
    qsort(out + start, cnt - start, sizeof(uint64_t), cmp_u64);
    uint64_t u = start;
    for (uint64_t i = start; i < cnt; ++i)
      if (i == start || out[i] != out[i - 1]) out[u++] = out[i];
    cnt = u;
  }
  free(v);
  *nnz = cnt;
  return out;
}

void igo_free(void* p) { free(p); }
