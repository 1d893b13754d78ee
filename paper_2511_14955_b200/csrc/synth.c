/* synth.c — seeded synthetic corpora with the shapes of BASELINE.json's five
 * configs (the paper's corpora are not available; these stand in for them).
 *
 * Pinned generator (documented in DESIGN.md §5 and echoed in every bench line):
 *   PRNG      xoshiro256** seeded by SplitMix64 from
 *             seed ^ (purpose * 0x9E3779B97F4A7C15) ^ (index * 0xD1B54A32D192ED03);
 *             one independent stream per (purpose, sequence index), so any
 *             subset of sequences regenerates byte-identically in parallel.
 *   vocab     65536 tokens (purpose VOCAB, index 0, vocab_seed): length
 *             1 + x % 16, bytes x >> 56, one draw per value.
 *   Zipf      s = 1.1 over ranks 1..65536 (rank r -> token r-1), Walker alias
 *             table; a draw x picks column x >> 48 and accepts it when
 *             (x & (2^48-1)) < prob48[col], else takes alias[col].
 *   zipf seq  concatenate Zipf tokens until the length is reached; truncate.
 *   lognormal len = round(exp(12 + 1.5 * N(0,1))) clipped to [256, 64 MiB],
 *             N(0,1) by Box-Muller from two 53-bit uniforms (purpose LEN);
 *             sequences are drawn until the running total reaches the target;
 *             the last one is truncated to hit the total exactly.
 *   markov    order-5 over {A,C,G,T}: row s (1024 rows) = Dirichlet(0.3)^4 via
 *             Gamma(0.3) = Gamma(1.3) * U^(1/0.3) (Marsaglia-Tsang), as 64-bit
 *             cumulative thresholds; first 5-mer uniform (x & 1023); then
 *             b = row[state] sampled with one draw, state = (state<<2 | b) & 1023.
 *   mixed     every byte uniform (x >> 56 per byte, 8 per draw), then runs of
 *             L = 64 + x % 4033 Zipf-token bytes at offset x % (len - L + 1) are
 *             written (later runs overwrite) until the summed run lengths reach
 *             len / 10.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IGS_API __attribute__((visibility("default")))

enum { P_VOCAB = 1, P_SEQ = 2, P_LEN = 3, P_MARKOV = 4 };
enum { K_ZIPF = 1, K_LOGNORMAL = 3, K_MARKOV = 4, K_MIXED = 5 };

typedef struct {
  uint64_t s[4];
} xo_t;

static inline uint64_t splitmix(uint64_t* x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static void xo_seed(xo_t* r, uint64_t seed, uint64_t purpose, uint64_t index) {
  uint64_t x = seed ^ (purpose * 0x9E3779B97F4A7C15ULL) ^ (index * 0xD1B54A32D192ED03ULL);
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix(&x);
}

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static inline uint64_t xo_next(xo_t* r) {
  uint64_t* s = r->s;
  const uint64_t out = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return out;
}

static inline double xo_unit(xo_t* r) { return (double)(xo_next(r) >> 11) * 0x1.0p-53; }

/* ------------------------------------------------------------ vocabulary + Zipf */
#define VOCAB 65536
typedef struct {
  uint64_t seed;
  uint8_t bytes[VOCAB * 16];
  uint8_t len[VOCAB];
  uint32_t off[VOCAB];
  uint64_t prob48[VOCAB];
  uint32_t alias[VOCAB];
} zipf_t;

static zipf_t* zipf_build(uint64_t vocab_seed, double s_exp) {
  zipf_t* z = (zipf_t*)calloc(1, sizeof(zipf_t));
  xo_t r;
  xo_seed(&r, vocab_seed, P_VOCAB, 0);
  uint32_t o = 0;
  for (int t = 0; t < VOCAB; ++t) {
    const int L = 1 + (int)(xo_next(&r) % 16);
    z->len[t] = (uint8_t)L;
    z->off[t] = o;
    for (int i = 0; i < L; ++i) z->bytes[o + i] = (uint8_t)(xo_next(&r) >> 56);
    o += (uint32_t)L;
  }
  /* Walker alias over w_r = r^-s (Vose's construction, stable order) */
  double* p = (double*)malloc(sizeof(double) * VOCAB);
  double sum = 0;
  for (int t = 0; t < VOCAB; ++t) sum += pow((double)(t + 1), -s_exp);
  for (int t = 0; t < VOCAB; ++t) p[t] = pow((double)(t + 1), -s_exp) / sum * VOCAB;
  uint32_t* small = (uint32_t*)malloc(4 * VOCAB);
  uint32_t* large = (uint32_t*)malloc(4 * VOCAB);
  int ns = 0, nl = 0;
  for (int t = 0; t < VOCAB; ++t) {
    if (p[t] < 1.0) small[ns++] = (uint32_t)t;
    else large[nl++] = (uint32_t)t;
  }
  while (ns && nl) {
    const uint32_t a = small[--ns], g = large[--nl];
    z->prob48[a] = (uint64_t)(p[a] * 281474976710656.0);
    z->alias[a] = g;
    p[g] = (p[g] + p[a]) - 1.0;
    if (p[g] < 1.0) small[ns++] = g;
    else large[nl++] = g;
  }
  while (nl) {
    const uint32_t g = large[--nl];
    z->prob48[g] = 281474976710656ULL;
    z->alias[g] = g;
  }
  while (ns) {
    const uint32_t a = small[--ns];
    z->prob48[a] = 281474976710656ULL;
    z->alias[a] = a;
  }
  free(p);
  free(small);
  free(large);
  return z;
}

static inline uint32_t zipf_draw(const zipf_t* z, xo_t* r) {
  const uint64_t x = xo_next(r);
  const uint32_t col = (uint32_t)(x >> 48);
  return (x & 0xFFFFFFFFFFFFULL) < z->prob48[col] ? col : z->alias[col];
}

static void fill_zipf(const zipf_t* z, xo_t* r, uint8_t* out, uint64_t len) {
  uint64_t w = 0;
  while (w < len) {
    const uint32_t t = zipf_draw(z, r);
    uint64_t L = z->len[t];
    if (L > len - w) L = len - w;
    memcpy(out + w, z->bytes + z->off[t], L);
    w += L;
  }
}

/* ------------------------------------------------------------ Markov */
static double gamma_mt(xo_t* r, double a) { /* Marsaglia-Tsang, a >= 1 */
  const double d = a - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      const double u1 = xo_unit(r), u2 = xo_unit(r);
      x = sqrt(-2.0 * log(u1 > 0 ? u1 : 1e-300)) * cos(6.283185307179586 * u2);
      v = 1.0 + c * x;
    } while (v <= 0);
    v = v * v * v;
    const double u = xo_unit(r);
    if (u < 1.0 - 0.0331 * x * x * x * x) return d * v;
    if (log(u > 0 ? u : 1e-300) < 0.5 * x * x + d * (1.0 - v + log(v))) return d * v;
  }
}

static void markov_rows(uint64_t seed, double alpha, uint64_t thr[1024][3]) {
  xo_t r;
  xo_seed(&r, seed, P_MARKOV, 0);
  for (int s = 0; s < 1024; ++s) {
    double g[4], sum = 0;
    for (int b = 0; b < 4; ++b) {
      const double u = xo_unit(&r);
      g[b] = gamma_mt(&r, alpha + 1.0) * pow(u > 0 ? u : 1e-300, 1.0 / alpha);
      sum += g[b];
    }
    double c = 0;
    for (int b = 0; b < 3; ++b) {
      c += g[b] / sum;
      const double v = c * 18446744073709551616.0;
      thr[s][b] = v >= 18446744073709551615.0 ? ~0ULL : (uint64_t)v;
    }
  }
}

/* ------------------------------------------------------------ public API */
typedef struct {
  int32_t kind;
  uint64_t num_seqs;   /* fixed-length kinds */
  uint64_t seq_len;    /* fixed-length kinds */
  uint64_t total;      /* lognormal: exact total bytes */
  uint64_t seed;
  uint64_t vocab_seed;
} igs_spec;

/* Number of sequences and offsets (m+1).  off may be NULL to query m. */
IGS_API uint64_t igs_offsets(const igs_spec* sp, uint64_t* off) {
  if (sp->kind != K_LOGNORMAL) {
    if (off)
      for (uint64_t i = 0; i <= sp->num_seqs; ++i) off[i] = i * sp->seq_len;
    return sp->num_seqs;
  }
  xo_t r;
  xo_seed(&r, sp->seed, P_LEN, 0);
  uint64_t total = 0, m = 0;
  if (off) off[0] = 0;
  while (total < sp->total) {
    const double u1 = xo_unit(&r), u2 = xo_unit(&r);
    const double nz = sqrt(-2.0 * log(u1 > 0 ? u1 : 1e-300)) * cos(6.283185307179586 * u2);
    double lf = floor(exp(12.0 + 1.5 * nz) + 0.5);
    if (lf < 256) lf = 256;
    if (lf > 67108864.0) lf = 67108864.0;
    uint64_t L = (uint64_t)lf;
    if (L > sp->total - total) L = sp->total - total;
    total += L;
    ++m;
    if (off) off[m] = total;
  }
  return m;
}

typedef struct {
  const igs_spec* sp;
  const zipf_t* z;
  uint64_t (*thr)[3];
  const uint64_t* off;
  uint8_t* base;
  uint64_t first, count;
  int tid, nthreads;
} job_t;

static void gen_one(const job_t* j, uint64_t i) {
  const igs_spec* sp = j->sp;
  const uint64_t len = j->off[i + 1] - j->off[i];
  uint8_t* out = j->base + (j->off[i] - j->off[j->first]);
  xo_t r;
  xo_seed(&r, sp->seed, P_SEQ, i);
  if (sp->kind == K_ZIPF || sp->kind == K_LOGNORMAL) {
    fill_zipf(j->z, &r, out, len);
  } else if (sp->kind == K_MARKOV) {
    static const uint8_t acgt[4] = {0x41, 0x43, 0x47, 0x54};
    uint32_t state = (uint32_t)(xo_next(&r) & 1023);
    for (uint64_t w = 0; w < len && w < 5; ++w) out[w] = acgt[(state >> (2 * (4 - w))) & 3];
    for (uint64_t w = 5; w < len; ++w) {
      const uint64_t x = xo_next(&r);
      const uint64_t* t = j->thr[state];
      const uint32_t b = x < t[0] ? 0 : x < t[1] ? 1 : x < t[2] ? 2 : 3;
      out[w] = acgt[b];
      state = ((state << 2) | b) & 1023;
    }
  } else { /* K_MIXED */
    uint64_t w = 0;
    while (w < len) {
      uint64_t x = xo_next(&r);
      for (int q = 0; q < 8 && w < len; ++q, ++w, x <<= 8) out[w] = (uint8_t)(x >> 56);
    }
    uint64_t covered = 0;
    while (len >= 64 && covered < len / 10) {
      uint64_t L = 64 + xo_next(&r) % 4033;
      if (L > len) L = len;
      const uint64_t at = xo_next(&r) % (len - L + 1);
      fill_zipf(j->z, &r, out + at, L);
      covered += L;
    }
  }
}

static void* worker(void* arg) {
  const job_t* j = (const job_t*)arg;
  for (uint64_t i = j->first + (uint64_t)j->tid; i < j->first + j->count; i += (uint64_t)j->nthreads)
    gen_one(j, i);
  return NULL;
}

/* Generates sequences [first, first+count) into base (sequence first at base). */
IGS_API int igs_fill(const igs_spec* sp, const uint64_t* off, uint64_t first, uint64_t count,
                     uint8_t* base, int threads) {
  zipf_t* z = NULL;
  uint64_t(*thr)[3] = NULL;
  if (sp->kind == K_ZIPF || sp->kind == K_LOGNORMAL || sp->kind == K_MIXED)
    z = zipf_build(sp->vocab_seed, 1.1);
  if (sp->kind == K_MARKOV) {
    thr = (uint64_t(*)[3])malloc(sizeof(uint64_t) * 3 * 1024);
    markov_rows(sp->seed, 0.3, thr);
  }
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].sp = sp;
    jobs[t].z = z;
    jobs[t].thr = thr;
    jobs[t].off = off;
    jobs[t].base = base;
    jobs[t].first = first;
    jobs[t].count = count;
    jobs[t].tid = t;
    jobs[t].nthreads = threads;
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(z);
  free(thr);
  return 0;
}
