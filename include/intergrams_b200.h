/* intergrams_b200.h — the C-ABI drop-in boundary of the B200-native Intergrams
 * top-k n-gram counter (arxiv 2511.14955).
 *
 * The reference exposes its hot path as the C++ API in
 * /root/reference/proj/include/intergrams/ (no FFI of its own):
 *   run_intergrams   intergrams.hpp:74-75   (driver, src/intergrams.cpp:68-166)
 *   extend_pass      intergrams.hpp:70-72   (src/intergrams.cpp:44-66)
 *   count_dense      dense_pass.hpp:25-28   (src/dense_pass.cpp:21-39)
 *   top_k            counting.hpp:112-113   (src/counting.cpp:52-98)
 * Every entry point below replaces one of those; the C++ drop-in headers in
 * include/intergrams/ re-expose the reference's own signatures on top of it.
 * Plain pointers and sizes only; no torch or STL types cross this boundary.
 *
 * Corpus layout (CSR): data[0..offsets[m]) bytes, offsets[m+1] u64 with
 * offsets[0] == 0; sequence i is data[offsets[i] .. offsets[i+1]).  This is
 * the enumeration order of Corpus::for_each (corpus.hpp:46-64).
 *
 * Gram keys: a gram of L <= 8 bytes is a u64, key = sum b_i << 8*(L-1-i)
 * (big-endian), so for one L numeric order == the reference's unsigned-byte
 * tie-break order (counting.hpp:38-41).  Output lists are canonical: count
 * descending, then key ascending.
 *
 * Return codes mirror the reference's exception classes (common.hpp:12-22,
 * cli.cpp:427-439):  IG_OK 0, IG_ECONFIG 2 (ConfigError), IG_EIO 3 (IoError),
 * IG_EINTERNAL 4 (CUDA / collective / allocation failure), IG_EINVALID 5
 * (std::invalid_argument from PrefixTrie::build / lookup, trie.cpp:26-46,142).
 * On error `err` (if non-NULL) receives a NUL-terminated message.
 *
 * Threading: calls on one session are serialised by the caller; sessions on
 * different devices are independent.  No global mutable state.
 */
#ifndef INTERGRAMS_B200_H
#define INTERGRAMS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define IG_API __attribute__((visibility("default")))
#else
#define IG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define IG_OK 0
#define IG_ECONFIG 2
#define IG_EIO 3
#define IG_EINTERNAL 4
#define IG_EINVALID 5
#define IG_ECALLBACK 6 /* a caller callback asked to stop (its own exception is rethrown by the C++ layer) */

/* CountMode (counting.hpp:19). */
#define IG_MODE_ONCE 0
#define IG_MODE_ALL 1

/* Where ig_corpus pointers live. */
#define IG_HOST 0
#define IG_DEVICE 1

/* Largest gram length of the packed-u64 key forms (ig_result.keys,
 * extend_pass, naive / hashgram / featurize).  run_intergrams itself takes
 * any n, as the reference does (intergrams.cpp:37-42): grams longer than 8
 * bytes come back in ig_result.grams only. */
#define IG_MAX_N 8

typedef struct {
  const uint8_t* data;      /* bytes; host or device per `location` */
  const uint64_t* offsets;  /* num_seqs + 1 entries, same location as data */
  uint64_t num_seqs;        /* m */
  int32_t location;         /* IG_HOST or IG_DEVICE */
} ig_corpus;

/* IntergramConfig (intergrams.hpp:19-33).  merge / workers /
 * flush_batch_size / frequency_ordered_trie never change results in the
 * reference (tests/test_dense_pass.cpp:141-161, test_trie.cpp:134-150) and
 * have no GPU meaning; flush_batch_size is still validated. */
typedef struct {
  uint32_t n;
  uint64_t k;
  double z;
  int32_t mode;             /* IG_MODE_ONCE / IG_MODE_ALL */
  uint64_t flush_batch_size;/* validated only (>= 1) */
  int32_t device;           /* CUDA ordinal; -1 = current */
} ig_params;

/* PassResult (intergrams.hpp:35-47). seconds are device-event times. */
typedef struct {
  char label[48];
  uint32_t gram_len;
  double seconds;
  uint64_t bytes_processed;
  uint64_t candidate_space;
  uint64_t retained;
  int32_t retained_short;
} ig_pass_stat;

/* IntergramsResult (intergrams.hpp:49-53); library-allocated, release with
 * ig_result_free. */
typedef struct {
  uint64_t len;            /* entries in keys/counts */
  uint32_t gram_len;       /* n */
  uint64_t* keys;          /* packed big-endian grams, canonical order */
  uint64_t* counts;
  ig_pass_stat* passes;
  uint32_t num_passes;
  char* diagnostics;       /* '\n'-separated, NUL-terminated */
  uint8_t* grams;          /* len * gram_len gram bytes, canonical order (every n;
                              for n > 8 the only form: keys is NULL) */
} ig_result;

/* Optional cross-rank hook for multi-GPU runs (one process per GPU).  The
 * library shards nothing itself: each rank passes its own whole-sequence
 * shard (see ig_shard_range) and the library calls allreduce once per
 * counting pass on the device count table (sum, in place, on `stream`).
 * A u64 table is preceded by a one-element u64 call (the sum of the ranks'
 * largest entries); when that sum is below 2^32 the table itself follows as
 * u32 (exact, half the bytes).  Every rank makes the same calls in the same
 * order.  dtype: 0 = u32, 1 = u64.  bytes_total / seqs_total are the GLOBAL corpus
 * totals (they choose the counter width identically on every rank and are
 * what PassResult::bytes_processed reports). */
typedef struct {
  int32_t rank;
  int32_t world;
  uint64_t bytes_total;
  uint64_t seqs_total;
  int (*allreduce)(void* dev_buf, uint64_t count, int32_t dtype,
                   void* cuda_stream, void* user);
  void* user;
} ig_collective;

/* ---- one-shot entry point: run_intergrams (src/intergrams.cpp:68-166) ---- */
IG_API int ig_topk_ngrams(const ig_corpus* corpus, const ig_params* params,
                   ig_result* out, char* err, size_t err_len);
IG_API void ig_result_free(ig_result* r);
/* run_intergrams over the reference's in-memory Corpus (a list of sequences,
 * corpus.hpp:60-62 / make_memory_corpus) without packing it first: sequence
 * q is seqs[q][0 .. lens[q]) in ordinary host memory.  Host threads gather
 * the bytes into pinned slabs that stream to HBM under the dense pass.  A
 * host ig_corpus that is not page-locked takes the same path in
 * ig_topk_ngrams / ig_session_run_host. */
IG_API int ig_topk_ngrams_seqs(const uint8_t* const* seqs, const uint64_t* lens,
                               uint64_t num_seqs, const ig_params* params, ig_result* out,
                               char* err, size_t err_len);

/* ---- session API: corpus resident in HBM across runs ---------------------
 * ig_session_create binds a device and (optionally) a collective.  load
 * copies a host corpus (or adopts a device corpus without copying).  run
 * executes run_intergrams on the resident corpus.  stream: cudaStream_t or
 * NULL for a library-owned stream. */
typedef struct ig_session ig_session;
IG_API int ig_session_create(int32_t device, void* cuda_stream,
                      const ig_collective* coll, ig_session** out, char* err,
                      size_t err_len);
IG_API int ig_session_load(ig_session* s, const ig_corpus* corpus, char* err,
                    size_t err_len);
IG_API int ig_session_run(ig_session* s, const ig_params* params, ig_result* out,
                   char* err, size_t err_len);
/* load + run with the host->device copy pipelined under the dense pass (the
 * corpus stays resident afterwards, as after ig_session_load). */
IG_API int ig_session_run_host(ig_session* s, const ig_corpus* corpus, const ig_params* params,
                               ig_result* out, char* err, size_t err_len);
/* ---- multi-GPU with the library's own NCCL communicators --------------
 * The reference's data parallelism (pipeline.hpp:101-199: whole sequences per
 * worker, per-pass tables merged into one) on GPUs: each device counts a
 * byte-balanced shard of whole sequences (ig_shard_range) and every pass
 * table is summed in place by one NCCL all-reduce; selection then runs
 * identically everywhere.  NCCL (libnccl.so.2) is loaded at first use.
 *
 * One process per GPU: rank 0 calls ig_nccl_unique_id and the caller moves
 * the 128 bytes to every rank; each rank then creates its session with
 * ig_session_create_nccl (ncclCommInitRank; collective over all ranks),
 * loads its shard and runs.  bytes_total / seqs_total are the whole
 * corpus's (count-table widths).  One process, several GPUs:
 * ig_topk_ngrams_multi shards a host corpus over `devices`
 * (ncclCommInitAll, one host thread per device) and returns the list. */
IG_API int ig_nccl_unique_id(uint8_t id_out[128], char* err, size_t err_len);
IG_API int ig_session_create_nccl(int32_t device, void* cuda_stream, int32_t rank, int32_t world,
                                  const uint8_t id[128], uint64_t bytes_total,
                                  uint64_t seqs_total, ig_session** out, char* err,
                                  size_t err_len);
IG_API int ig_topk_ngrams_multi(const ig_corpus* corpus, const int32_t* devices, int32_t ndev,
                                const ig_params* params, ig_result* out, char* err,
                                size_t err_len);
/* Debugging: with IG_GUARD=1 in the environment every device buffer carries
 * guard bytes and every call checks them afterwards (out-of-bounds device
 * writes become IG_EINTERNAL).  ig_guard_selftest writes byte `at` of a
 * 100-byte guarded buffer and runs that check. */
IG_API int ig_guard_selftest(int32_t device, int64_t at, char* err, size_t err_len);
/* Kernel launches issued by the session so far (for launch accounting). */
IG_API uint64_t ig_session_launches(const ig_session* s);

/* Per-kernel-family device timing (CUDA events on the session stream; off by
 * default).  ig_session_kernel_stats fills ms[i] / launches[i] for families
 * i < n (IG_KF_*) accumulated since the last reset. */
#define IG_KF_ROUTE_COUNT 0   /* count-once: owner histogram pass        */
#define IG_KF_ROUTE_SCATTER 1 /* count-once: dedup + lookup + route       */
#define IG_KF_ROUTE_CONSUME 2 /* count-once: per-sequence dedup + counts  */
#define IG_KF_COUNT_ALL 3     /* count-all counting kernels               */
#define IG_KF_SELECT 4        /* canonical top-k selection (all kernels)  */
#define IG_KF_ONCE_SHORT 5    /* count-once: short sequences, no routing  */
#define IG_KF_ONCE_DIRECT 6   /* count-once: small-alphabet bitmap passes */
IG_API void ig_session_set_profiling(ig_session* s, int32_t on);
IG_API int ig_session_kernel_stats(ig_session* s, double* ms, uint64_t* launches, int32_t n,
                                   int32_t reset);
IG_API void ig_session_destroy(ig_session* s);

/* ---- pass-level entry points (parity of the reference's tables) ---------- */
/* count_dense (dense_pass.cpp:21-39): table_out receives 256^n u64, n 1..3. */
IG_API int ig_count_dense(const ig_corpus* corpus, uint32_t n, int32_t mode,
                   int32_t device, uint64_t* table_out, char* err,
                   size_t err_len);

/* extend_pass (intergrams.cpp:44-66) over the prefix list `prefix_keys`
 * (nprefix keys of prefix_len bytes, rank order; ordinal = index).
 * table_out receives 256*nprefix u64 indexed ordinal*256 + last byte
 * (candidate_id, intergrams.hpp:56-59).  An empty list is a depth-0 trie. */
IG_API int ig_extend_pass(const ig_corpus* corpus, const uint64_t* prefix_keys,
                   uint64_t nprefix, uint32_t prefix_len, uint32_t j,
                   int32_t mode, int32_t device, uint64_t* table_out,
                   uint64_t* bytes_processed, char* err, size_t err_len);

/* top_k (counting.cpp:52-98) of a host u64 table whose gram key is the id
 * (prefix_keys == NULL) or (prefix_keys[id>>8] << 8) | (id & 255).  Writes
 * min(k, nonzero) entries; returns IG_ECONFIG for k < 1. */
IG_API int ig_top_k(const uint64_t* table, uint64_t cap, uint64_t k,
             const uint64_t* prefix_keys, int32_t device, uint64_t* keys_out,
             uint64_t* counts_out, uint64_t* len_out, char* err,
             size_t err_len);

/* ---- corpus ingestion from files (corpus.cpp:13-152) ---------------------
 * The reference's CorpusSpec: roots are regular files or directories (of
 * regular files, recursively when `recurse`); all files are taken in path
 * order; each file gives one sequence, or one per '\n'-terminated line
 * (`line_mode`; a final unterminated line counts when non-empty), or one per
 * `chunk_size` bytes (the last one short).  Files are read by host threads
 * into pinned slabs and copied to HBM as they are read; line splitting runs
 * on the GPU.  A missing root is IG_ECONFIG, an unreadable file IG_EIO. */
typedef struct {
  const char* const* roots;
  uint64_t num_roots;
  int32_t recurse;
  int32_t line_mode;
  uint64_t chunk_size;
} ig_file_corpus;

/* run_intergrams(Corpus(spec), cfg) on a file corpus. */
IG_API int ig_topk_ngrams_files(const ig_file_corpus* spec, const ig_params* params,
                                ig_result* out, char* err, size_t err_len);
/* Session variants: load (corpus stays resident), load + run. */
IG_API int ig_session_load_files(ig_session* s, const ig_file_corpus* spec, char* err,
                                 size_t err_len);
IG_API int ig_session_run_files(ig_session* s, const ig_file_corpus* spec,
                                const ig_params* params, ig_result* out, char* err,
                                size_t err_len);
/* The resident corpus of a session, copied back (data / offsets may be NULL;
 * each is filled only when its capacity suffices). */
IG_API int ig_session_corpus(ig_session* s, uint8_t* data, uint64_t data_cap, uint64_t* offsets,
                             uint64_t offsets_cap, uint64_t* num_seqs, uint64_t* total_bytes,
                             char* err, size_t err_len);
/* Host-only: the spec's files in enumeration order, one callback each
 * (path, size); a nonzero return stops the walk with IG_ECALLBACK. */
typedef int (*ig_file_fn)(const char* path, uint64_t size, void* user);
IG_API int ig_file_corpus_list(const ig_file_corpus* spec, ig_file_fn fn, void* user, char* err,
                               size_t err_len);
/* Host-only: every record of the spec in enumeration order (Corpus::for_each,
 * corpus.hpp:51), as (id, bytes, len) views valid during the callback; a
 * nonzero return stops the walk with IG_ECALLBACK. */
typedef int (*ig_record_fn)(uint64_t id, const uint8_t* bytes, uint64_t len, void* user);
IG_API int ig_file_corpus_records(const ig_file_corpus* spec, ig_record_fn fn, void* user,
                                  char* err, size_t err_len);
/* Host-only: the files a spec enumerates (count, total bytes). */
IG_API int ig_file_corpus_files(const ig_file_corpus* spec, uint64_t* num_files,
                                uint64_t* total_bytes, char* err, size_t err_len);

/* ---- exact counting paths (sort-based, same sm_100a library) ------------ */
/* naive_count + naive_topk (proj/src/oracle.cpp:7-47, oracle.hpp:17-27):
 * exact counts of every n-gram, canonical top-k.  A corpus of more than
 * max_corpus_bytes is a ConfigError, like the reference's guard; pass
 * IG_ORACLE_GUARD for the reference default.  out->passes is empty. */
#define IG_ORACLE_GUARD (256ull << 20)
IG_API int ig_naive_topk(const ig_corpus* corpus, uint32_t n, uint64_t k, int32_t mode,
                         uint64_t max_corpus_bytes, int32_t device, ig_result* out,
                         char* err, size_t err_len);

/* HashgramConfig (hashgram.hpp:19-31).  merge / workers / flush_batch_size /
 * trie_second_pass never change results and are accepted unused. */
typedef struct {
  uint64_t buckets;          /* B */
  uint32_t n;
  uint64_t k;
  int32_t mode;
  uint64_t seed;
  uint64_t flush_batch_size;
  int32_t trie_second_pass;
  int32_t device;
} ig_hashgram_params;

/* run_hashgram (hashgram.cpp:325-383): bucket pass, top-k buckets (count
 * desc, bucket asc), exact pass over grams of kept buckets, top-k grams.
 * out->passes holds the reference's four rows ("hash pass", "top-k buckets",
 * "exact pass", "top-k grams"). */
IG_API int ig_hashgram_topk(const ig_corpus* corpus, const ig_hashgram_params* params,
                            ig_result* out, char* err, size_t err_len);

/* mix64 (hashgram.cpp:22-59, MurmurHash64A).  Host-only. */
IG_API uint64_t ig_mix64(const uint8_t* bytes, uint64_t len, uint64_t seed);

/* FeatureMatrix (metrics.hpp:39-46): rows = sequences, cols = vocabulary
 * entries, (row[i], col[i]) the set entries sorted by row then col. */
typedef struct {
  uint64_t rows;
  uint64_t cols;
  uint64_t nnz;
  uint64_t* row;
  uint32_t* col;
} ig_matrix;

/* featurize (metrics.cpp:83-132): entry (r, j) when vocabulary gram j (a
 * packed key of gram_len bytes) occurs in sequence r.  A repeated vocabulary
 * gram maps to its first column.  Release with ig_matrix_free. */
IG_API int ig_featurize(const ig_corpus* corpus, const uint64_t* vocab_keys, uint64_t ncols,
                        uint32_t gram_len, int32_t device, ig_matrix* out, char* err,
                        size_t err_len);
IG_API void ig_matrix_free(ig_matrix* m);

/* Byte-balanced whole-sequence shard [*first, *last) of rank r of world w:
 * cut at the sequence boundary nearest r*total/w.  Host-only, no device. */
IG_API void ig_shard_range(const uint64_t* offsets, uint64_t num_seqs, int32_t rank,
                    int32_t world, uint64_t* first, uint64_t* last);

/* Library version string. */
IG_API const char* ig_version(void);

#ifdef __cplusplus
}
#endif
#endif
