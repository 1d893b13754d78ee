/* ig_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference Intergrams CPU
 * algorithm (/root/reference/proj, arxiv 2511.14955).  It is the parity
 * checker for the CUDA path: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it.  The product library
 * (paper_2511_14955_b200) never links or calls it.
 *
 * Parity pinning: this restatement is checked against (a) the reference's own
 * known-answer tests (proj/tests/test_*.cpp, restated in tests/test_oracle_kat.py)
 * and (b) the reference itself compiled from its sources into oracle/_ref/
 * (see oracle/Makefile), through golden vectors under tests/golden/ generated
 * by tests/golden/make_golden.py.
 *
 * Gram convention: a gram of L <= 8 bytes is packed big-endian into a u64,
 * key = sum b_i << 8*(L-1-i).  For equal L, numeric key order equals the
 * unsigned-byte lexicographic order of std::string::operator< that the
 * reference uses as its tie-break (proj/include/intergrams/counting.hpp:38-41).
 *
 * Corpus layout: CSR — data[] bytes, offsets[m+1] (u64), sequence i is
 * data[offsets[i] .. offsets[i+1]).
 */
#ifndef IG_ORACLE_H
#define IG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { IGO_OK = 0, IGO_CONFIG = 2, IGO_INTERNAL = 4 };
enum { IGO_ONCE = 0, IGO_ALL = 1 }; /* CountMode::kOnce / kAll, counting.hpp:19 */

/* std::mt19937_64 (the reference tests' RNG, tests/helpers.hpp:46-65). */
typedef struct {
  uint64_t mt[312];
  int idx;
} igo_mt64;
void igo_mt64_seed(igo_mt64* r, uint64_t seed);
uint64_t igo_mt64_next(igo_mt64* r);

/* One row of IntergramsResult::passes (intergrams.hpp:35-47), minus timing. */
typedef struct {
  char label[48];
  uint32_t gram_len;
  uint64_t bytes_processed;
  uint64_t candidate_space;
  uint64_t retained;
  int32_t retained_short;
} igo_pass;

/* Dense exact count over 256^n ids, n in [1,3]
 * (dense_pass.cpp:21-39; driver copy intergrams.cpp:79-100).
 * table: 256^n u64, overwritten. */
int igo_count_dense(const uint8_t* data, const uint64_t* off, uint64_t m,
                    uint32_t n, int mode, uint64_t* table);

/* Canonical top-k of the nonzero entries of table[0..cap)
 * (counting.cpp:52-98).  Gram key of id: id itself when prefix_keys == NULL
 * (dense_gram, dense_pass.cpp:12-19), else (prefix_keys[id>>8] << 8) | (id&255)
 * (candidate_gram, intergrams.hpp:62-66).  Returns the number written
 * (<= k).  out arrays need room for min(k, cap). */
uint64_t igo_top_k(const uint64_t* table, uint64_t cap, uint64_t k,
                   const uint64_t* prefix_keys, uint64_t* out_keys,
                   uint64_t* out_counts);

/* extend_pass (intergrams.cpp:44-66): counts j-grams whose (j-1)-byte prefix
 * is prefix_keys[ord] (ord = rank); id = ord*256 + last byte.  prefix_len is
 * the trie depth (0 for an empty trie).  table: 256*nprefix u64.  Returns
 * IGO_CONFIG when the trie depth is not j-1 (intergrams.cpp:46-48). */
int igo_extend_pass(const uint8_t* data, const uint64_t* off, uint64_t m,
                    const uint64_t* prefix_keys, uint64_t nprefix,
                    uint32_t prefix_len, uint32_t j, int mode, uint64_t* table,
                    uint64_t* bytes_processed);

/* run_intergrams (intergrams.cpp:68-166) for n <= 8.
 * out_keys/out_counts: room for k entries.  passes: room for 2*max(n,3)
 * rows.  diag: newline-separated diagnostics (may be NULL). */
int igo_run_intergrams(const uint8_t* data, const uint64_t* off, uint64_t m,
                       uint32_t n, uint64_t k, double z, int mode,
                       uint64_t* out_keys, uint64_t* out_counts,
                       uint64_t* out_len, igo_pass* passes,
                       uint32_t* num_passes, char* diag, size_t diag_len,
                       char* err, size_t err_len);

/* naive_count + naive_topk (oracle.cpp:7-47) for n <= 8. */
int igo_naive_topk(const uint8_t* data, const uint64_t* off, uint64_t m,
                   uint32_t n, int mode, uint64_t k, uint64_t* out_keys,
                   uint64_t* out_counts, uint64_t* out_len);

/* run_hashgram (hashgram.cpp:325-383) for n <= 8: top-k grams plus the
 * retained counts of its "top-k buckets" and "exact pass" rows. */
uint64_t igo_mix64(const uint8_t* bytes, uint64_t len, uint64_t seed);
int igo_hashgram_topk(const uint8_t* data, const uint64_t* off, uint64_t m,
                      uint32_t n, uint64_t k, int mode, uint64_t buckets,
                      uint64_t seed, uint64_t* out_keys, uint64_t* out_counts,
                      uint64_t* out_len, uint64_t* kept_buckets,
                      uint64_t* exact_size);

/* featurize (metrics.cpp:83-132) for grams of n <= 8 bytes: malloc'd
 * (row << 32 | col) entries sorted by row then col; free with igo_free. */
uint64_t* igo_featurize(const uint8_t* data, const uint64_t* off, uint64_t m,
                        const uint64_t* vocab, uint64_t ncols, uint32_t n,
                        uint64_t* nnz);
void igo_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
