"""TEST INFRASTRUCTURE ONLY.

ctypes access to the two CPU checkers of the GPU path:
  * ``c_oracle()``  — oracle/ig_oracle.c, a plain-C restatement of the reference
    algorithm (built into oracle/_build/libigoracle.so);
  * ``ref()``       — the unmodified reference sources compiled in place from
    /root/reference/proj/src (oracle/_ref/libigref.so, see oracle/Makefile).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product library never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libigoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libigref.so")
REF_SRC = "/root/reference/proj"

ONCE, ALL = 0, 1


class igo_mt64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class igo_pass(C.Structure):
    _fields_ = [("label", C.c_char * 48), ("gram_len", C.c_uint32),
                ("bytes_processed", C.c_uint64), ("candidate_space", C.c_uint64),
                ("retained", C.c_uint64), ("retained_short", C.c_int32)]


class igref_pass(C.Structure):
    _fields_ = [("label", C.c_char * 48), ("gram_len", C.c_uint32), ("seconds", C.c_double),
                ("bytes_processed", C.c_uint64), ("candidate_space", C.c_uint64),
                ("retained", C.c_uint64), ("retained_short", C.c_int32)]


_oracle = None
_ref = None


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def build_ref() -> bool:
    """Compiles the reference CPU path from /root/reference (only where it exists)."""
    if not os.path.isdir(REF_SRC):
        return os.path.exists(REF_SO)
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return True


def c_oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        L.igo_mt64_seed.argtypes = [C.POINTER(igo_mt64), C.c_uint64]
        L.igo_mt64_next.argtypes = [C.POINTER(igo_mt64)]
        L.igo_mt64_next.restype = C.c_uint64
        L.igo_count_dense.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int,
                                      C.c_void_p]
        L.igo_top_k.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                C.c_void_p]
        L.igo_top_k.restype = C.c_uint64
        L.igo_extend_pass.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                      C.c_uint32, C.c_uint32, C.c_int, C.c_void_p,
                                      C.POINTER(C.c_uint64)]
        L.igo_run_intergrams.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                         C.c_uint64, C.c_double, C.c_int, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_uint64), C.c_void_p,
                                         C.POINTER(C.c_uint32), C.c_char_p, C.c_size_t,
                                         C.c_char_p, C.c_size_t]
        L.igo_naive_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int,
                                     C.c_uint64, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
        L.igo_mix64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.igo_mix64.restype = C.c_uint64
        L.igo_hashgram_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                        C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.igo_featurize.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                    C.c_uint32, C.POINTER(C.c_uint64)]
        L.igo_featurize.restype = C.c_void_p
        L.igo_free.argtypes = [C.c_void_p]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if not build_ref():
                raise RuntimeError("reference build unavailable (no /root/reference and no "
                                   "prebuilt oracle/_ref/libigref.so)")
        L = C.CDLL(REF_SO)
        L.igref_hardware_concurrency.restype = C.c_uint
        L.igref_run_intergrams.argtypes = [
            C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, C.c_int,
            C.c_uint32, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p, C.c_uint32,
            C.POINTER(C.c_uint32), C.c_char_p, C.c_size_t, C.POINTER(C.c_double), C.c_char_p,
            C.c_size_t]
        L.igref_count_dense.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int,
                                        C.c_uint32, C.c_void_p, C.c_char_p, C.c_size_t]
        L.igref_extend_pass.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                        C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p,
                                        C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
        L.igref_naive_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int,
                                       C.c_uint64, C.c_void_p, C.c_void_p,
                                       C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
        L.igref_mix64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.igref_mix64.restype = C.c_uint64
        L.igref_hashgram.argtypes = [
            C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.c_uint64,
            C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
            C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_char_p, C.c_size_t]
        L.igref_featurize.argtypes = [
            C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
            C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_char_p,
            C.c_size_t]
        L.igref_corpus_files.argtypes = [
            C.POINTER(C.c_char_p), C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_void_p,
            C.c_uint64, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
            C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
        L.igref_jaccard_tsv.argtypes = [C.c_char_p, C.c_char_p]
        L.igref_jaccard_tsv.restype = C.c_double
        L.igref_report.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_uint32, C.c_int,
                                   C.c_double, C.c_int, C.c_char_p, C.c_size_t]
        _ref = L
    return _ref


# ------------------------------------------------------------------ corpora

def csr(seqs: Sequence[bytes]) -> Tuple[np.ndarray, np.ndarray]:
    lens = np.fromiter((len(s) for s in seqs), dtype=np.uint64, count=len(seqs))
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    np.cumsum(lens, out=off[1:])
    data = np.frombuffer(b"".join(seqs) + b"\0", dtype=np.uint8)[:-1].copy()
    return data, off


class Mt64:
    """std::mt19937_64 via the C oracle (tests/helpers.hpp uses it)."""

    def __init__(self, seed: int):
        self.s = igo_mt64()
        c_oracle().igo_mt64_seed(C.byref(self.s), seed)

    def __call__(self) -> int:
        return int(c_oracle().igo_mt64_next(C.byref(self.s)))


def random_bytes(rng: Mt64, n: int, alphabet: int) -> bytes:
    """tests/helpers.hpp:46-53."""
    return bytes(rng() % alphabet for _ in range(n))


def random_corpus(rng: Mt64, max_m: int, max_len: int, alphabet: int) -> List[bytes]:
    """tests/helpers.hpp:55-65: m in [1, max_m], lengths in [0, max_len]."""
    m = 1 + rng() % max_m
    return [random_bytes(rng, rng() % (max_len + 1), alphabet) for _ in range(m)]


# ------------------------------------------------------------------ C oracle calls

def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def oracle_run(data: np.ndarray, off: np.ndarray, n: int, k: int, z: float, mode: int):
    """igo_run_intergrams -> (rc, keys, counts, passes, diagnostics)."""
    L = c_oracle()
    keys = np.zeros(k, np.uint64)
    counts = np.zeros(k, np.uint64)
    ln = C.c_uint64(0)
    passes = (igo_pass * 32)()
    np_ = C.c_uint32(0)
    diag = C.create_string_buffer(4096)
    err = C.create_string_buffer(512)
    rc = L.igo_run_intergrams(_ptr(data), off.ctypes.data, off.size - 1, n, k, z, mode,
                              keys.ctypes.data, counts.ctypes.data, C.byref(ln), passes,
                              C.byref(np_), diag, len(diag), err, len(err))
    rows = [dict(label=passes[i].label.decode(), gram_len=passes[i].gram_len,
                 bytes_processed=passes[i].bytes_processed,
                 candidate_space=passes[i].candidate_space, retained=passes[i].retained,
                 retained_short=bool(passes[i].retained_short)) for i in range(np_.value)]
    n_ = ln.value
    return rc, keys[:n_], counts[:n_], rows, [d for d in diag.value.decode().split("\n") if d]


def oracle_count_dense(data, off, n, mode) -> np.ndarray:
    t = np.zeros(1 << (8 * n), np.uint64)
    rc = c_oracle().igo_count_dense(_ptr(data), off.ctypes.data, off.size - 1, n, mode,
                                    t.ctypes.data)
    assert rc == 0
    return t


def oracle_extend(data, off, prefix_keys: np.ndarray, plen: int, j: int, mode: int):
    pk = np.ascontiguousarray(prefix_keys, np.uint64)
    t = np.zeros(max(256 * pk.size, 1), np.uint64)
    b = C.c_uint64(0)
    rc = c_oracle().igo_extend_pass(_ptr(data), off.ctypes.data, off.size - 1, _ptr(pk), pk.size,
                                    plen, j, mode, t.ctypes.data, C.byref(b))
    return rc, t[:256 * pk.size], b.value


def oracle_top_k(table: np.ndarray, k: int, prefix_keys: Optional[np.ndarray] = None):
    t = np.ascontiguousarray(table, np.uint64)
    kk = max(min(k, t.size), 1)
    keys = np.zeros(kk, np.uint64)
    counts = np.zeros(kk, np.uint64)
    pk = None if prefix_keys is None else np.ascontiguousarray(prefix_keys, np.uint64)
    n = c_oracle().igo_top_k(t.ctypes.data, t.size, k, pk.ctypes.data if pk is not None else None,
                             keys.ctypes.data, counts.ctypes.data)
    return keys[:n], counts[:n]


def oracle_naive(data, off, n: int, mode: int, k: int):
    keys = np.zeros(k, np.uint64)
    counts = np.zeros(k, np.uint64)
    ln = C.c_uint64(0)
    rc = c_oracle().igo_naive_topk(_ptr(data), off.ctypes.data, off.size - 1, n, mode, k,
                                   keys.ctypes.data, counts.ctypes.data, C.byref(ln))
    assert rc == 0
    return keys[:ln.value], counts[:ln.value]


# ------------------------------------------------------------------ reference calls

def ref_run(data: np.ndarray, off: np.ndarray, n: int, k: int, z: float, mode: int,
            workers: int = 0):
    """ig_ref::run_intergrams -> (rc, keys, counts, passes, diagnostics, seconds, err)."""
    L = ref()
    grams = np.zeros(max(k * n, 1), np.uint8)
    counts = np.zeros(k, np.uint64)
    ln = C.c_uint64(0)
    passes = (igref_pass * 32)()
    np_ = C.c_uint32(0)
    diag = C.create_string_buffer(4096)
    err = C.create_string_buffer(512)
    secs = C.c_double(0)
    rc = L.igref_run_intergrams(_ptr(data), off.ctypes.data, off.size - 1, n, k, z, mode, workers,
                                grams.ctypes.data, counts.ctypes.data, C.byref(ln), passes, 32,
                                C.byref(np_), diag, len(diag), C.byref(secs), err, len(err))
    m = ln.value
    g = grams[:m * n].reshape(m, n) if m else np.zeros((0, n), np.uint8)
    keys = np.zeros(m, np.uint64)
    for i in range(n):
        keys = (keys << np.uint64(8)) | g[:, i].astype(np.uint64)
    rows = [dict(label=passes[i].label.decode(), gram_len=passes[i].gram_len,
                 seconds=passes[i].seconds, bytes_processed=passes[i].bytes_processed,
                 candidate_space=passes[i].candidate_space, retained=passes[i].retained,
                 retained_short=bool(passes[i].retained_short)) for i in range(np_.value)]
    return (rc, keys, counts[:m], rows, [d for d in diag.value.decode().split("\n") if d],
            secs.value, err.value.decode())


def ref_run_grams(data: np.ndarray, off: np.ndarray, n: int, k: int, z: float, mode: int,
                  workers: int = 0):
    """ig_ref::run_intergrams for any n -> (rc, grams (len, n) uint8, counts,
    passes, diagnostics, err): the gram bytes themselves (n > 8 does not fit
    the packed keys ref_run returns)."""
    L = ref()
    grams = np.zeros(max(k * n, 1), np.uint8)
    counts = np.zeros(k, np.uint64)
    ln = C.c_uint64(0)
    passes = (igref_pass * 64)()
    np_ = C.c_uint32(0)
    diag = C.create_string_buffer(8192)
    err = C.create_string_buffer(512)
    secs = C.c_double(0)
    rc = L.igref_run_intergrams(_ptr(data), off.ctypes.data, off.size - 1, n, k, z, mode, workers,
                                grams.ctypes.data, counts.ctypes.data, C.byref(ln), passes, 64,
                                C.byref(np_), diag, len(diag), C.byref(secs), err, len(err))
    m = ln.value
    rows = [dict(label=passes[i].label.decode(), gram_len=passes[i].gram_len,
                 bytes_processed=passes[i].bytes_processed,
                 candidate_space=passes[i].candidate_space, retained=passes[i].retained,
                 retained_short=bool(passes[i].retained_short)) for i in range(np_.value)]
    return (rc, grams[:m * n].reshape(m, n).copy(), counts[:m], rows,
            [d for d in diag.value.decode().split("\n") if d], err.value.decode())


def ref_run_file(path: str, chunk_size: int, n: int, k: int, z: float, mode: int,
                 workers: int = 0):
    """ig_ref::run_intergrams over a file corpus (one root; chunk_size records,
    or whole-file records when 0) -> the same tuple as ref_run."""
    L = ref()
    if not hasattr(L, "_file_bound"):
        L.igref_run_intergrams_file.argtypes = [
            C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, C.c_int, C.c_uint32,
            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_char_p,
            C.c_size_t, C.c_void_p, C.c_char_p, C.c_size_t]
        L._file_bound = True
    grams = np.zeros(max(k * n, 1), np.uint8)
    counts = np.zeros(k, np.uint64)
    ln = C.c_uint64(0)
    passes = (igref_pass * 32)()
    np_ = C.c_uint32(0)
    diag = C.create_string_buffer(4096)
    err = C.create_string_buffer(512)
    secs = C.c_double(0)
    rc = L.igref_run_intergrams_file(path.encode(), chunk_size, n, k, z, mode, workers,
                                     grams.ctypes.data, counts.ctypes.data, C.byref(ln), passes,
                                     32, C.byref(np_), diag, len(diag), C.byref(secs), err,
                                     len(err))
    m = ln.value
    g = grams[:m * n].reshape(m, n) if m else np.zeros((0, n), np.uint8)
    keys = np.zeros(m, np.uint64)
    for i in range(n):
        keys = (keys << np.uint64(8)) | g[:, i].astype(np.uint64)
    rows = [dict(label=passes[i].label.decode(), gram_len=passes[i].gram_len,
                 seconds=passes[i].seconds, bytes_processed=passes[i].bytes_processed,
                 candidate_space=passes[i].candidate_space, retained=passes[i].retained,
                 retained_short=bool(passes[i].retained_short)) for i in range(np_.value)]
    return (rc, keys, counts[:m], rows, [d for d in diag.value.decode().split("\n") if d],
            secs.value, err.value.decode())


def ref_count_dense(data, off, n, mode, workers=1) -> np.ndarray:
    t = np.zeros(1 << (8 * n), np.uint64)
    err = C.create_string_buffer(512)
    rc = ref().igref_count_dense(_ptr(data), off.ctypes.data, off.size - 1, n, mode, workers,
                                 t.ctypes.data, err, len(err))
    assert rc == 0, err.value
    return t


def ref_extend(data, off, prefixes: Sequence[bytes], j: int, mode: int):
    plen = len(prefixes[0]) if prefixes else 0
    flat = np.frombuffer(b"".join(prefixes) + b"\0", np.uint8)[:-1].copy()
    t = np.zeros(max(256 * len(prefixes), 1), np.uint64)
    b = C.c_uint64(0)
    err = C.create_string_buffer(512)
    rc = ref().igref_extend_pass(_ptr(data), off.ctypes.data, off.size - 1, _ptr(flat),
                                 len(prefixes), plen, j, mode, t.ctypes.data, C.byref(b), err,
                                 len(err))
    return rc, t[:256 * len(prefixes)], b.value, err.value.decode()


def ref_naive(data, off, n: int, mode: int, k: int):
    grams = np.zeros(max(k * n, 1), np.uint8)
    counts = np.zeros(k, np.uint64)
    ln = C.c_uint64(0)
    err = C.create_string_buffer(512)
    rc = ref().igref_naive_topk(_ptr(data), off.ctypes.data, off.size - 1, n, mode, k,
                                grams.ctypes.data, counts.ctypes.data, C.byref(ln), err, len(err))
    assert rc == 0, err.value
    m = ln.value
    g = grams[:m * n].reshape(m, n) if m else np.zeros((0, n), np.uint8)
    keys = np.zeros(m, np.uint64)
    for i in range(n):
        keys = (keys << np.uint64(8)) | g[:, i].astype(np.uint64)
    return keys, counts[:m]


# ------------------------------------------------------- hash-gramming / featurize

def oracle_mix64(b: bytes, seed: int) -> int:
    buf = np.frombuffer(b + b"\0", np.uint8)
    return int(c_oracle().igo_mix64(buf.ctypes.data, len(b), seed))


def oracle_hashgram(data, off, n: int, k: int, mode: int, buckets: int, seed: int):
    """igo_hashgram_topk -> (rc, keys, counts, kept_buckets, exact_size)."""
    keys = np.zeros(k, np.uint64)
    counts = np.zeros(k, np.uint64)
    ln, kept, ex = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    rc = c_oracle().igo_hashgram_topk(_ptr(data), off.ctypes.data, off.size - 1, n, k, mode,
                                      buckets, seed, keys.ctypes.data, counts.ctypes.data,
                                      C.byref(ln), C.byref(kept), C.byref(ex))
    return rc, keys[:ln.value], counts[:ln.value], kept.value, ex.value


def oracle_featurize(data, off, vocab_keys, n: int) -> np.ndarray:
    """igo_featurize -> sorted (row << 32 | col) entries."""
    v = np.ascontiguousarray(vocab_keys, np.uint64)
    nnz = C.c_uint64(0)
    L = c_oracle()
    p = L.igo_featurize(_ptr(data), off.ctypes.data, off.size - 1, _ptr(v), v.size, n,
                        C.byref(nnz))
    out = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), (max(nnz.value, 1),))
    out = out[:nnz.value].copy()
    L.igo_free(p)
    return out


def ref_mix64(b: bytes, seed: int) -> int:
    buf = np.frombuffer(b + b"\0", np.uint8)
    return int(ref().igref_mix64(buf.ctypes.data, len(b), seed))


def ref_hashgram(data, off, n: int, k: int, mode: int, buckets: int, seed: int,
                 workers: int = 1, trie: bool = False):
    """ig_ref::run_hashgram -> (rc, keys, counts, rows, err)."""
    grams = np.zeros(max(k * n, 1), np.uint8)
    counts = np.zeros(k, np.uint64)
    ln = C.c_uint64(0)
    passes = (igref_pass * 8)()
    np_ = C.c_uint32(0)
    err = C.create_string_buffer(512)
    rc = ref().igref_hashgram(_ptr(data), off.ctypes.data, off.size - 1, n, k, mode, buckets,
                              seed, workers, int(trie), grams.ctypes.data, counts.ctypes.data,
                              C.byref(ln), passes, 8, C.byref(np_), err, len(err))
    m = ln.value
    g = grams[:m * n].reshape(m, n) if m else np.zeros((0, n), np.uint8)
    keys = np.zeros(m, np.uint64)
    for i in range(n):
        keys = (keys << np.uint64(8)) | g[:, i].astype(np.uint64)
    rows = [dict(label=passes[i].label.decode(), gram_len=passes[i].gram_len,
                 seconds=passes[i].seconds, bytes_processed=passes[i].bytes_processed,
                 candidate_space=passes[i].candidate_space, retained=passes[i].retained,
                 retained_short=bool(passes[i].retained_short)) for i in range(np_.value)]
    return rc, keys, counts[:m], rows, err.value.decode()


def ref_featurize(data, off, vocab: Sequence[bytes], workers: int = 1):
    """ig_ref::featurize -> (rc, entries (row << 32 | col), rows, err)."""
    n = len(vocab[0]) if vocab else 0
    flat = np.frombuffer(b"".join(vocab) + b"\0", np.uint8)[:-1].copy()
    cap = int(off[-1]) + int(off.size) + 16
    ent = np.zeros(cap, np.uint64)
    nnz, rows = C.c_uint64(0), C.c_uint64(0)
    err = C.create_string_buffer(512)
    rc = ref().igref_featurize(_ptr(data), off.ctypes.data, off.size - 1, _ptr(flat), len(vocab),
                               n, workers, ent.ctypes.data, cap, C.byref(nnz), C.byref(rows), err,
                               len(err))
    return rc, ent[:nnz.value].copy(), rows.value, err.value.decode()


def ref_jaccard_tsv(a: str, b: str) -> float:
    return float(ref().igref_jaccard_tsv(a.encode(), b.encode()))


def ref_report(algorithm: str, echo: str, rows, jaccard: Optional[float] = None,
               json: bool = False) -> str:
    """RunReport(algorithm, echo, rows).to_tsv() / to_json() of the reference."""
    arr = (igref_pass * max(len(rows), 1))()
    for i, r in enumerate(rows):
        arr[i].label = r["label"].encode()
        arr[i].gram_len = r["gram_len"]
        arr[i].seconds = r["seconds"]
        arr[i].bytes_processed = r["bytes_processed"]
        arr[i].candidate_space = r["candidate_space"]
        arr[i].retained = r["retained"]
        arr[i].retained_short = int(r["retained_short"])
    out = C.create_string_buffer(1 << 20)
    rc = ref().igref_report(algorithm.encode(), echo.encode(), arr, len(rows),
                            int(jaccard is not None), float(jaccard or 0.0), int(json), out,
                            len(out))
    assert rc == 0, out.value
    return out.value.decode()


def ref_corpus_files(roots, recurse=False, line_mode=False, chunk_size=0):
    """ig_ref::Corpus(CorpusSpec{roots, ...}) -> (rc, data, offsets, num_files, err)."""
    arr = (C.c_char_p * max(len(roots), 1))(*[os.fsencode(r) for r in roots])
    m, tot, nf = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    err = C.create_string_buffer(512)
    L = ref()
    rc = L.igref_corpus_files(arr, len(roots), int(recurse), int(line_mode), chunk_size, None, 0,
                              None, 0, C.byref(m), C.byref(tot), C.byref(nf), err, len(err))
    if rc != 0:
        return rc, None, None, 0, err.value.decode()
    data = np.zeros(max(tot.value, 1), np.uint8)
    off = np.zeros(m.value + 1, np.uint64)
    rc = L.igref_corpus_files(arr, len(roots), int(recurse), int(line_mode), chunk_size,
                              data.ctypes.data, data.size, off.ctypes.data, off.size, C.byref(m),
                              C.byref(tot), C.byref(nf), err, len(err))
    return rc, data[:tot.value], off, nf.value, err.value.decode()
