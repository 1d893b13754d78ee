"""ctypes binding of include/intergrams_b200.h (the C-ABI boundary).

The library is built in-tree (``make -C paper_2511_14955_b200``) into
``paper_2511_14955_b200/_lib/libintergrams_b200.so``.  There is no fallback:
if the shared library is missing, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libintergrams_b200.so")

IG_OK, IG_ECONFIG, IG_EIO, IG_EINTERNAL, IG_EINVALID = 0, 2, 3, 4, 5
IG_MODE_ONCE, IG_MODE_ALL = 0, 1
IG_HOST, IG_DEVICE = 0, 1
IG_MAX_N = 8
KERNEL_FAMILIES = ["route_count", "route_scatter", "route_consume", "count_all", "select",
                   "once_short", "once_direct"]


class ig_corpus(C.Structure):
    _fields_ = [("data", C.c_void_p), ("offsets", C.c_void_p),
                ("num_seqs", C.c_uint64), ("location", C.c_int32)]


class ig_params(C.Structure):
    _fields_ = [("n", C.c_uint32), ("k", C.c_uint64), ("z", C.c_double),
                ("mode", C.c_int32), ("flush_batch_size", C.c_uint64),
                ("device", C.c_int32)]


class ig_pass_stat(C.Structure):
    _fields_ = [("label", C.c_char * 48), ("gram_len", C.c_uint32),
                ("seconds", C.c_double), ("bytes_processed", C.c_uint64),
                ("candidate_space", C.c_uint64), ("retained", C.c_uint64),
                ("retained_short", C.c_int32)]


class ig_result(C.Structure):
    _fields_ = [("len", C.c_uint64), ("gram_len", C.c_uint32),
                ("keys", C.POINTER(C.c_uint64)), ("counts", C.POINTER(C.c_uint64)),
                ("passes", C.POINTER(ig_pass_stat)), ("num_passes", C.c_uint32),
                ("diagnostics", C.c_char_p), ("grams", C.POINTER(C.c_uint8))]


class ig_hashgram_params(C.Structure):
    _fields_ = [("buckets", C.c_uint64), ("n", C.c_uint32), ("k", C.c_uint64),
                ("mode", C.c_int32), ("seed", C.c_uint64), ("flush_batch_size", C.c_uint64),
                ("trie_second_pass", C.c_int32), ("device", C.c_int32)]


class ig_matrix(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64),
                ("row", C.POINTER(C.c_uint64)), ("col", C.POINTER(C.c_uint32))]


class ig_file_corpus(C.Structure):
    _fields_ = [("roots", C.POINTER(C.c_char_p)), ("num_roots", C.c_uint64),
                ("recurse", C.c_int32), ("line_mode", C.c_int32), ("chunk_size", C.c_uint64)]


IG_ORACLE_GUARD = 256 << 20

FILE_FN = C.CFUNCTYPE(C.c_int, C.c_char_p, C.c_uint64, C.c_void_p)
RECORD_FN = C.CFUNCTYPE(C.c_int, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p)


class ig_collective(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32),
                ("bytes_total", C.c_uint64), ("seqs_total", C.c_uint64),
                ("allreduce", ALLREDUCE_FN), ("user", C.c_void_p)]


# (name, restype, argtypes) for every symbol include/intergrams_b200.h declares.
SYMBOLS = [
    ("ig_topk_ngrams", C.c_int, [C.POINTER(ig_corpus), C.POINTER(ig_params),
                                 C.POINTER(ig_result), C.c_char_p, C.c_size_t]),
    ("ig_result_free", None, [C.POINTER(ig_result)]),
    ("ig_topk_ngrams_seqs", C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), C.c_uint64,
                                      C.POINTER(ig_params), C.POINTER(ig_result), C.c_char_p,
                                      C.c_size_t]),
    ("ig_session_create", C.c_int, [C.c_int32, C.c_void_p, C.POINTER(ig_collective),
                                    C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    ("ig_session_load", C.c_int, [C.c_void_p, C.POINTER(ig_corpus), C.c_char_p, C.c_size_t]),
    ("ig_session_run", C.c_int, [C.c_void_p, C.POINTER(ig_params), C.POINTER(ig_result),
                                 C.c_char_p, C.c_size_t]),
    ("ig_session_run_host", C.c_int, [C.c_void_p, C.POINTER(ig_corpus), C.POINTER(ig_params),
                                      C.POINTER(ig_result), C.c_char_p, C.c_size_t]),
    ("ig_session_launches", C.c_uint64, [C.c_void_p]),
    ("ig_nccl_unique_id", C.c_int, [C.c_char_p, C.c_char_p, C.c_size_t]),
    ("ig_guard_selftest", C.c_int, [C.c_int32, C.c_int64, C.c_char_p, C.c_size_t]),
    ("ig_session_create_nccl", C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                         C.c_char_p, C.c_uint64, C.c_uint64,
                                         C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    ("ig_topk_ngrams_multi", C.c_int, [C.POINTER(ig_corpus), C.POINTER(C.c_int32), C.c_int32,
                                       C.POINTER(ig_params), C.POINTER(ig_result), C.c_char_p,
                                       C.c_size_t]),
    ("ig_session_set_profiling", None, [C.c_void_p, C.c_int32]),
    ("ig_session_kernel_stats", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                          C.c_int32]),
    ("ig_session_destroy", None, [C.c_void_p]),
    ("ig_count_dense", C.c_int, [C.POINTER(ig_corpus), C.c_uint32, C.c_int32, C.c_int32,
                                 C.c_void_p, C.c_char_p, C.c_size_t]),
    ("ig_extend_pass", C.c_int, [C.POINTER(ig_corpus), C.c_void_p, C.c_uint64, C.c_uint32,
                                 C.c_uint32, C.c_int32, C.c_int32, C.c_void_p,
                                 C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    ("ig_top_k", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int32,
                           C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_char_p,
                           C.c_size_t]),
    ("ig_naive_topk", C.c_int, [C.POINTER(ig_corpus), C.c_uint32, C.c_uint64, C.c_int32,
                                C.c_uint64, C.c_int32, C.POINTER(ig_result), C.c_char_p,
                                C.c_size_t]),
    ("ig_hashgram_topk", C.c_int, [C.POINTER(ig_corpus), C.POINTER(ig_hashgram_params),
                                   C.POINTER(ig_result), C.c_char_p, C.c_size_t]),
    ("ig_mix64", C.c_uint64, [C.c_void_p, C.c_uint64, C.c_uint64]),
    ("ig_featurize", C.c_int, [C.POINTER(ig_corpus), C.c_void_p, C.c_uint64, C.c_uint32,
                               C.c_int32, C.POINTER(ig_matrix), C.c_char_p, C.c_size_t]),
    ("ig_matrix_free", None, [C.POINTER(ig_matrix)]),
    ("ig_topk_ngrams_files", C.c_int, [C.POINTER(ig_file_corpus), C.POINTER(ig_params),
                                       C.POINTER(ig_result), C.c_char_p, C.c_size_t]),
    ("ig_session_load_files", C.c_int, [C.c_void_p, C.POINTER(ig_file_corpus), C.c_char_p,
                                        C.c_size_t]),
    ("ig_session_run_files", C.c_int, [C.c_void_p, C.POINTER(ig_file_corpus),
                                       C.POINTER(ig_params), C.POINTER(ig_result), C.c_char_p,
                                       C.c_size_t]),
    ("ig_session_corpus", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_char_p,
                                    C.c_size_t]),
    ("ig_file_corpus_list", C.c_int, [C.POINTER(ig_file_corpus), FILE_FN, C.c_void_p,
                                      C.c_char_p, C.c_size_t]),
    ("ig_file_corpus_records", C.c_int, [C.POINTER(ig_file_corpus), RECORD_FN, C.c_void_p,
                                         C.c_char_p, C.c_size_t]),
    ("ig_file_corpus_files", C.c_int, [C.POINTER(ig_file_corpus), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    ("ig_shard_range", None, [C.c_void_p, C.c_uint64, C.c_int32, C.c_int32,
                              C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("ig_version", C.c_char_p, []),
]

_lib = None


def lib() -> C.CDLL:
    """Loads the CUDA library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2511_14955_b200` "
                "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib
