"""Python mirror of the reference's hot-path API (proj/include/intergrams/).

Names, fields, defaults and error classes follow the reference so the parity
tests read like its own doctest suite:

  IntergramConfig   intergrams.hpp:19-33      run_intergrams  intergrams.hpp:74-75
  PassResult        intergrams.hpp:35-47      extend_pass     intergrams.hpp:70-72
  IntergramsResult  intergrams.hpp:49-53      count_dense     dense_pass.hpp:25-28
  CountMode         counting.hpp:19           top_k           counting.hpp:112-113
  GramCount         counting.hpp:27-33        candidate_id    intergrams.hpp:56-59
  ConfigError/IoError common.hpp:12-22        make_memory_corpus corpus.hpp:67
  naive_topk        oracle.cpp:7-47           run_hashgram    hashgram.hpp:19-75
  featurize         metrics.hpp:39-49         mix64           hashgram.hpp:33-39

Every call goes through the C-ABI (include/intergrams_b200.h) into the sm_100a
kernels; nothing here computes counts on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N


class ConfigError(RuntimeError):
    """Unusable configuration (common.hpp:12-15; CLI exit code 2)."""


class IoError(RuntimeError):
    """Filesystem or read failure (common.hpp:19-22; CLI exit code 3)."""


class InternalError(RuntimeError):
    """CUDA / collective / allocation failure (CLI exit code 4)."""


class CountMode(IntEnum):
    """counting.hpp:19 — ONCE: once per sequence; ALL: every occurrence."""
    kOnce = 0
    kAll = 1


class MergeStrategy(IntEnum):
    """counting.hpp:25 — accepted for API parity; never changes results."""
    kBatchedFlush = 0
    kAtomic = 1


def _raise(rc: int, err: C.Array) -> None:
    if rc == N.IG_OK:
        return
    msg = err.value.decode(errors="replace")
    if rc == N.IG_ECONFIG:
        raise ConfigError(msg)
    if rc == N.IG_EIO:
        raise IoError(msg)
    if rc == N.IG_EINVALID:
        raise ValueError(msg)  # std::invalid_argument (a std::logic_error)
    raise InternalError(msg)


@dataclass
class GramCount:
    """counting.hpp:27-33."""
    gram: bytes
    count: int

    def __iter__(self):
        return iter((self.gram, self.count))


@dataclass
class PassResult:
    """intergrams.hpp:35-47."""
    label: str
    gram_len: int = 0
    seconds: float = 0.0
    bytes_processed: int = 0
    candidate_space: int = 0
    retained: int = 0
    retained_short: bool = False

    def throughput_bps(self) -> float:
        return self.bytes_processed / self.seconds if self.seconds > 0 else 0.0


@dataclass
class IntergramsResult:
    """intergrams.hpp:49-53 (keys/counts also kept as numpy arrays)."""
    topk: List[GramCount]
    passes: List[PassResult]
    diagnostics: List[str]
    keys: np.ndarray = field(default=None, repr=False)  # packed u64 (n <= 8; None above)
    counts: np.ndarray = field(default=None, repr=False)
    grams: np.ndarray = field(default=None, repr=False)  # (len, n) uint8, every n


@dataclass
class IntergramConfig:
    """intergrams.hpp:19-33 (same defaults)."""
    n: int = 6
    k: int = 10000
    z: float = 1.5
    mode: CountMode = CountMode.kOnce
    merge: MergeStrategy = MergeStrategy.kBatchedFlush
    workers: int = 1
    flush_batch_size: int = 8
    frequency_ordered_trie: bool = True
    device: int = -1

    def k_prime(self) -> int:
        return int(math.ceil(self.z * float(self.k)))

    def validate(self) -> None:
        """IntergramConfig::validate, intergrams.cpp:37-42."""
        if self.n < 1:
            raise ConfigError("gram length n must be >= 1")
        if self.k < 1:
            raise ConfigError("k must be >= 1")
        if not (self.z >= 1.0):
            raise ConfigError("oversample factor z must be >= 1")
        if self.flush_batch_size < 1:
            raise ConfigError("flush batch size must be >= 1")

    def _params(self) -> N.ig_params:
        return N.ig_params(n=int(self.n), k=int(self.k), z=float(self.z), mode=int(self.mode),
                           flush_batch_size=int(self.flush_batch_size), device=int(self.device))


# ----------------------------------------------------------------- corpus

class Corpus:
    """A CSR byte corpus: data (u8) and offsets (u64, m+1).  Sequence order is
    the reference's enumeration order (Corpus::for_each, corpus.hpp:46-64)."""

    def __init__(self, data: np.ndarray, offsets: np.ndarray):
        self.data = np.ascontiguousarray(data, dtype=np.uint8)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        if self.offsets.size < 1 or int(self.offsets[0]) != 0:
            raise ConfigError("corpus offsets must start at 0")
        if int(self.offsets[-1]) != self.data.size:
            raise ConfigError("corpus offsets must end at len(data)")

    @property
    def num_seqs(self) -> int:
        return int(self.offsets.size - 1)

    @property
    def bytes_total(self) -> int:
        return int(self.offsets[-1])

    def sequences(self) -> List[bytes]:
        o = self.offsets
        return [self.data[o[i]:o[i + 1]].tobytes() for i in range(self.num_seqs)]

    def _view(self) -> N.ig_corpus:
        return N.ig_corpus(data=self.data.ctypes.data, offsets=self.offsets.ctypes.data,
                           num_seqs=self.num_seqs, location=N.IG_HOST)


@dataclass
class CorpusSpec:
    """corpus.hpp:30-36: files / directories read by the library straight into
    HBM (ig_*_files), with the reference's enumeration and record rules."""
    roots: Sequence[str]
    recurse: bool = False
    line_mode: bool = False
    chunk_size: int = 0

    def _native(self):
        arr = (C.c_char_p * max(len(self.roots), 1))(*[os.fsencode(r) for r in self.roots])
        spec = N.ig_file_corpus(roots=arr, num_roots=len(self.roots), recurse=int(self.recurse),
                                line_mode=int(self.line_mode), chunk_size=int(self.chunk_size))
        return spec, arr  # keep arr alive with the struct

    def files(self) -> Tuple[int, int]:
        """(number of files, total bytes) the spec enumerates (host only)."""
        spec, _keep = self._native()
        n, b = C.c_uint64(0), C.c_uint64(0)
        err = C.create_string_buffer(1024)
        _raise(N.lib().ig_file_corpus_files(C.byref(spec), C.byref(n), C.byref(b), err,
                                            len(err)), err)
        return int(n.value), int(b.value)


def make_memory_corpus(sequences: Iterable[bytes]) -> Corpus:
    """corpus.hpp:67 — in-memory corpus from a list of byte strings."""
    seqs = [bytes(s) for s in sequences]
    lens = np.fromiter((len(s) for s in seqs), dtype=np.uint64, count=len(seqs))
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    np.cumsum(lens, out=off[1:])
    data = np.frombuffer(b"".join(seqs), dtype=np.uint8).copy()
    return Corpus(data, off)


def as_corpus(c) -> Corpus:
    if isinstance(c, Corpus):
        return c
    return make_memory_corpus(c)


# ----------------------------------------------------------------- grams

def key_to_gram(key: int, n: int) -> bytes:
    return int(key).to_bytes(8, "big")[8 - n:]


def gram_to_key(gram: bytes) -> int:
    return int.from_bytes(gram, "big")


def candidate_id(prefix_ordinal: int, last_byte: int) -> int:
    """intergrams.hpp:56-59."""
    assert 0 <= last_byte <= 255
    return prefix_ordinal * 256 + last_byte


def candidate_gram(prefixes: Sequence[GramCount], cid: int) -> bytes:
    """intergrams.hpp:62-66."""
    return prefixes[cid >> 8].gram + bytes([cid & 0xFF])


def dense_capacity(n: int) -> int:
    """dense_pass.cpp:5-10."""
    if n < 1 or n > 3:
        raise ConfigError("dense pass supports gram lengths 1..3")
    return 1 << (8 * n)


def dense_gram(gid: int, n: int) -> bytes:
    """dense_pass.cpp:12-19."""
    return key_to_gram(gid, n)


# ----------------------------------------------------------------- results

def _result(r: N.ig_result, materialize: bool = True) -> IntergramsResult:
    """materialize=False keeps the list as numpy keys/counts only (topk = [])."""
    n = int(r.len)
    gl = int(r.gram_len)
    counts = np.ctypeslib.as_array(r.counts, shape=(max(n, 1),))[:n].copy() if n else \
        np.zeros(0, np.uint64)
    grams = None
    if r.grams and n:
        grams = np.ctypeslib.as_array(r.grams, shape=(n * gl,)).copy().reshape(n, gl)
    elif r.grams or gl > 8:
        grams = np.zeros((0, gl), np.uint8)
    if r.keys:
        keys = np.ctypeslib.as_array(r.keys, shape=(max(n, 1),))[:n].copy() if n else \
            np.zeros(0, np.uint64)
        topk = [GramCount(key_to_gram(int(k), gl), int(c)) for k, c in zip(keys, counts)] \
            if materialize else []
    else:  # n > 8: grams only
        keys = None
        topk = [GramCount(bytes(g), int(c)) for g, c in zip(grams, counts)] \
            if materialize else []
    passes = []
    for i in range(int(r.num_passes)):
        p = r.passes[i]
        passes.append(PassResult(p.label.decode(), int(p.gram_len), float(p.seconds),
                                 int(p.bytes_processed), int(p.candidate_space),
                                 int(p.retained), bool(p.retained_short)))
    diag = (r.diagnostics or b"").decode()
    return IntergramsResult(topk, passes, [d for d in diag.split("\n") if d], keys, counts,
                            grams)


def run_intergrams(corpus, cfg: IntergramConfig, materialize: bool = True) -> IntergramsResult:
    """run_intergrams (intergrams.hpp:74-75) on the GPU.  A CorpusSpec is read
    from disk by the library (pinned slabs -> HBM, ig_topk_ngrams_files).
    materialize=False: the list as numpy keys/grams/counts only."""
    cfg.validate()
    if isinstance(corpus, CorpusSpec):
        spec, _keep = corpus._native()
        err = C.create_string_buffer(1024)
        out = N.ig_result()
        params = cfg._params()
        rc = N.lib().ig_topk_ngrams_files(C.byref(spec), C.byref(params), C.byref(out), err,
                                          len(err))
        _raise(rc, err)
        try:
            return _result(out, materialize)
        finally:
            N.lib().ig_result_free(C.byref(out))
    lib = N.lib()
    err = C.create_string_buffer(1024)
    out = N.ig_result()
    params = cfg._params()
    if isinstance(corpus, (list, tuple)) and all(isinstance(q, (bytes, bytearray, str))
                                                 for q in corpus):
        # the reference's in-memory corpus (make_memory_corpus): sequences
        # gathered in place by the library (ig_topk_ngrams_seqs), no packing
        seqs = [q.encode("latin-1") if isinstance(q, str) else bytes(q) for q in corpus]
        m = len(seqs)
        ptrs = (C.c_void_p * max(m, 1))(*[C.cast(C.c_char_p(q), C.c_void_p) for q in seqs])
        lens = (C.c_uint64 * max(m, 1))(*[len(q) for q in seqs])
        rc = lib.ig_topk_ngrams_seqs(ptrs, lens, m, C.byref(params), C.byref(out), err, len(err))
        _raise(rc, err)
        try:
            return _result(out, materialize)
        finally:
            lib.ig_result_free(C.byref(out))
    c = as_corpus(corpus)
    view = c._view()
    rc = lib.ig_topk_ngrams(C.byref(view), C.byref(params), C.byref(out), err, len(err))
    _raise(rc, err)
    try:
        return _result(out, materialize)
    finally:
        lib.ig_result_free(C.byref(out))


def nccl_unique_id() -> bytes:
    """ig_nccl_unique_id: the 128-byte id rank 0 hands to every rank."""
    buf = C.create_string_buffer(128)
    err = C.create_string_buffer(1024)
    _raise(N.lib().ig_nccl_unique_id(buf, err, len(err)), err)
    return buf.raw


def run_intergrams_multi(corpus, cfg: IntergramConfig, devices) -> IntergramsResult:
    """run_intergrams over several GPUs of this process (ig_topk_ngrams_multi):
    whole-sequence shards balanced by bytes, one NCCL all-reduce per pass."""
    cfg.validate()
    c = as_corpus(corpus)
    devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
    err = C.create_string_buffer(1024)
    out = N.ig_result()
    view = c._view()
    params = cfg._params()
    rc = N.lib().ig_topk_ngrams_multi(C.byref(view), devs, len(devices), C.byref(params),
                                      C.byref(out), err, len(err))
    _raise(rc, err)
    try:
        return _result(out)
    finally:
        N.lib().ig_result_free(C.byref(out))


def count_dense(corpus, n: int, mode: CountMode, device: int = -1) -> np.ndarray:
    """count_dense (dense_pass.hpp:25-28): the 256^n u64 table."""
    c = as_corpus(corpus)
    cap = 1 << (8 * n) if 1 <= n <= 3 else 1
    table = np.zeros(cap, dtype=np.uint64)
    err = C.create_string_buffer(1024)
    view = c._view()
    rc = N.lib().ig_count_dense(C.byref(view), n, int(mode), device, table.ctypes.data, err,
                                len(err))
    _raise(rc, err)
    return table


def count_trigrams(corpus, mode: CountMode, device: int = -1) -> np.ndarray:
    """dense_pass.hpp:31-34."""
    return count_dense(corpus, 3, mode, device)


def extend_pass(corpus, prefixes: Sequence[bytes], j: int, mode: CountMode,
                device: int = -1) -> Tuple[np.ndarray, int]:
    """extend_pass (intergrams.hpp:70-72) with the trie built from `prefixes`
    (rank order).  Returns (table[256*len(prefixes)], bytes_processed)."""
    c = as_corpus(corpus)
    plen = len(prefixes[0]) if prefixes else 0
    for p in prefixes:
        if len(p) != plen:
            raise ValueError("trie prefixes must share one length")
    keys = np.array([gram_to_key(p) for p in prefixes], dtype=np.uint64)
    table = np.zeros(max(256 * len(prefixes), 1), dtype=np.uint64)
    bp = C.c_uint64(0)
    err = C.create_string_buffer(1024)
    view = c._view()
    rc = N.lib().ig_extend_pass(C.byref(view), keys.ctypes.data if keys.size else None,
                                len(prefixes), plen, j, int(mode), device,
                                table.ctypes.data, C.byref(bp), err, len(err))
    _raise(rc, err)
    return table[:256 * len(prefixes)], int(bp.value)


def top_k(table: np.ndarray, k: int, prefix_keys: Optional[np.ndarray] = None,
          device: int = -1) -> Tuple[np.ndarray, np.ndarray]:
    """top_k (counting.cpp:52-98) of a u64 table on the GPU.  Keys are the ids
    (prefix_keys None) or (prefix_keys[id>>8] << 8) | (id & 255)."""
    t = np.ascontiguousarray(table, dtype=np.uint64)
    cap = int(t.size)
    kk = min(int(k), max(cap, 1)) if k >= 1 else 1
    keys = np.zeros(kk, np.uint64)
    counts = np.zeros(kk, np.uint64)
    ln = C.c_uint64(0)
    err = C.create_string_buffer(1024)
    pk = None
    if prefix_keys is not None:
        pk = np.ascontiguousarray(prefix_keys, dtype=np.uint64)
    rc = N.lib().ig_top_k(t.ctypes.data, cap, int(k), pk.ctypes.data if pk is not None else None,
                          device, keys.ctypes.data, counts.ctypes.data, C.byref(ln), err,
                          len(err))
    _raise(rc, err)
    n = int(ln.value)
    return keys[:n], counts[:n]


def shard_range(offsets: np.ndarray, rank: int, world: int) -> Tuple[int, int]:
    """Byte-balanced whole-sequence shard of `rank` (host-only)."""
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    a, b = C.c_uint64(0), C.c_uint64(0)
    N.lib().ig_shard_range(off.ctypes.data, off.size - 1, rank, world, C.byref(a), C.byref(b))
    return int(a.value), int(b.value)


def run_result_topk(r: IntergramsResult, n: int) -> List[GramCount]:
    """The GramCount list of a result (materialised from keys/counts if needed)."""
    if r.topk:
        return r.topk
    if r.keys is None:
        return [GramCount(bytes(g), int(c)) for g, c in zip(r.grams, r.counts)] \
            if r.grams is not None else r.topk
    return [GramCount(key_to_gram(int(k), n), int(c)) for k, c in zip(r.keys, r.counts)]


def topk_to_tsv(topk: Sequence[GramCount]) -> str:
    """metrics.cpp:202-211: lowercase hex, TAB, decimal count, LF."""
    return "".join(f"{g.gram.hex()}\t{g.count}\n" for g in topk)


# ------------------------------------------------- exact / hashgram / featurize

kOracleCorpusGuard = N.IG_ORACLE_GUARD  # oracle.hpp:17


def naive_topk(corpus, n: int, mode: CountMode, k: int,
               max_corpus_bytes: int = kOracleCorpusGuard, device: int = -1) -> List[GramCount]:
    """naive_topk(naive_count(corpus, n, mode, guard), k) (oracle.cpp:7-47),
    counted exactly on the GPU (sort + run-length reduction)."""
    c = as_corpus(corpus)
    err = C.create_string_buffer(1024)
    out = N.ig_result()
    view = c._view()
    rc = N.lib().ig_naive_topk(C.byref(view), int(n), int(k), int(mode), int(max_corpus_bytes),
                               device, C.byref(out), err, len(err))
    _raise(rc, err)
    try:
        return _result(out).topk
    finally:
        N.lib().ig_result_free(C.byref(out))


@dataclass
class HashgramConfig:
    """hashgram.hpp:19-31 (same defaults)."""
    buckets: int = 1 << 31
    n: int = 6
    k: int = 10000
    mode: CountMode = CountMode.kOnce
    seed: int = 0
    merge: MergeStrategy = MergeStrategy.kBatchedFlush
    workers: int = 1
    flush_batch_size: int = 8
    trie_second_pass: bool = False
    device: int = -1


@dataclass
class HashgramResult:
    """hashgram.hpp:69-72."""
    topk: List[GramCount]
    passes: List[PassResult]


def run_hashgram(corpus, cfg: HashgramConfig) -> HashgramResult:
    """run_hashgram (hashgram.cpp:325-383) on the GPU."""
    c = as_corpus(corpus)
    p = N.ig_hashgram_params(buckets=int(cfg.buckets), n=int(cfg.n), k=int(cfg.k),
                             mode=int(cfg.mode), seed=int(cfg.seed),
                             flush_batch_size=int(cfg.flush_batch_size),
                             trie_second_pass=int(bool(cfg.trie_second_pass)),
                             device=int(cfg.device))
    err = C.create_string_buffer(1024)
    out = N.ig_result()
    view = c._view()
    rc = N.lib().ig_hashgram_topk(C.byref(view), C.byref(p), C.byref(out), err, len(err))
    _raise(rc, err)
    try:
        r = _result(out)
        return HashgramResult(r.topk, r.passes)
    finally:
        N.lib().ig_result_free(C.byref(out))


def mix64(gram: bytes, seed: int) -> int:
    """mix64 (hashgram.cpp:22-59), host-side."""
    buf = (C.c_uint8 * max(len(gram), 1)).from_buffer_copy(gram or b"\0")
    return int(N.lib().ig_mix64(C.addressof(buf), len(gram), seed))


def hash_ngram(gram: bytes, seed: int, buckets: int) -> int:
    """hashgram.hpp:36-39."""
    return mix64(gram, seed) % buckets


class FeatureMatrix:
    """metrics.hpp:39-46: (row, col) entries sorted by row then col, held as
    numpy arrays (``row``, ``col``); ``entries`` materialises the pair list."""

    def __init__(self, rows: int, cols: int, row: np.ndarray, col: np.ndarray):
        self.rows = rows
        self.cols = cols
        self.row = row
        self.col = col

    @property
    def entries(self) -> List[Tuple[int, int]]:
        return list(zip(self.row.tolist(), self.col.tolist()))

    def column_popcounts(self) -> List[int]:
        """metrics.cpp:77-81."""
        return np.bincount(self.col.astype(np.int64), minlength=self.cols).tolist()


def featurize(corpus, vocab: Sequence[GramCount], workers: int = 1,
              device: int = -1) -> FeatureMatrix:
    """featurize (metrics.cpp:83-132) on the GPU.  `workers` has no GPU meaning."""
    c = as_corpus(corpus)
    grams = [g.gram if isinstance(g, GramCount) else bytes(g) for g in vocab]
    n = len(grams[0]) if grams else 0
    for g in grams:
        if len(g) != n:
            raise ValueError("featurize: vocab grams must share one length")
    if grams and n > N.IG_MAX_N:
        raise ConfigError("featurize: gram length above 8 is not supported by the GPU path")
    keys = np.array([gram_to_key(g) for g in grams], dtype=np.uint64)
    err = C.create_string_buffer(1024)
    out = N.ig_matrix()
    view = c._view()
    rc = N.lib().ig_featurize(C.byref(view), keys.ctypes.data if keys.size else None,
                              len(grams), n, device, C.byref(out), err, len(err))
    _raise(rc, err)
    try:
        nnz = int(out.nnz)
        rows = np.ctypeslib.as_array(out.row, shape=(nnz,)).copy() if nnz else np.zeros(0, np.uint64)
        cols = np.ctypeslib.as_array(out.col, shape=(nnz,)).copy() if nnz else np.zeros(0, np.uint32)
        return FeatureMatrix(int(out.rows), int(out.cols), rows, cols)
    finally:
        N.lib().ig_matrix_free(C.byref(out))


# ----------------------------------------------------------------- session

class Session:
    """A device session with the corpus resident in HBM (ig_session_*)."""

    def __init__(self, device: int = 0, stream: int = 0,
                 collective: Optional[N.ig_collective] = None,
                 nccl: Optional[dict] = None):
        """nccl: {"rank", "world", "id" (128 bytes from nccl_unique_id() on
        rank 0), "bytes_total", "seqs_total"} — the session's table all-reduces
        go through the library's own NCCL communicator (ig_session_create_nccl)."""
        self._lib = N.lib()
        self._h = C.c_void_p()
        self._coll = collective  # keep the callback alive
        err = C.create_string_buffer(1024)
        st = C.c_void_p(stream) if stream else None
        if nccl is not None:
            uid = bytes(nccl["id"])
            assert len(uid) == 128
            rc = self._lib.ig_session_create_nccl(
                device, st, int(nccl["rank"]), int(nccl["world"]), uid,
                int(nccl["bytes_total"]), int(nccl["seqs_total"]), C.byref(self._h), err, len(err))
        else:
            rc = self._lib.ig_session_create(device, st,
                                             C.byref(collective) if collective else None,
                                             C.byref(self._h), err, len(err))
        _raise(rc, err)

    def load(self, corpus=None, *, data_ptr: int = 0, offsets_ptr: int = 0, num_seqs: int = 0,
             device_ptrs: bool = False) -> None:
        err = C.create_string_buffer(1024)
        if corpus is not None:
            c = as_corpus(corpus)
            self._corpus = c
            view = c._view()
        else:
            view = N.ig_corpus(data=data_ptr, offsets=offsets_ptr, num_seqs=num_seqs,
                               location=N.IG_DEVICE if device_ptrs else N.IG_HOST)
        rc = self._lib.ig_session_load(self._h, C.byref(view), err, len(err))
        _raise(rc, err)

    def run(self, cfg: IntergramConfig, materialize: bool = True) -> IntergramsResult:
        """run_intergrams on the resident corpus.  materialize=False returns the
        list as numpy `keys`/`counts` (big-endian packed grams) without building
        per-gram Python objects."""
        cfg.validate()
        err = C.create_string_buffer(1024)
        out = N.ig_result()
        params = cfg._params()
        rc = self._lib.ig_session_run(self._h, C.byref(params), C.byref(out), err, len(err))
        _raise(rc, err)
        try:
            return _result(out, materialize)
        finally:
            self._lib.ig_result_free(C.byref(out))

    def load_and_run(self, corpus, cfg: IntergramConfig,
                     materialize: bool = True) -> IntergramsResult:
        """Host corpus -> result, with the H2D copy pipelined under the dense
        pass (ig_session_run_host).  The corpus stays resident afterwards."""
        cfg.validate()
        c = as_corpus(corpus)
        self._corpus = c
        view = c._view()
        err = C.create_string_buffer(1024)
        out = N.ig_result()
        params = cfg._params()
        rc = self._lib.ig_session_run_host(self._h, C.byref(view), C.byref(params), C.byref(out),
                                           err, len(err))
        _raise(rc, err)
        try:
            return _result(out, materialize)
        finally:
            self._lib.ig_result_free(C.byref(out))

    def load_files(self, spec: CorpusSpec) -> None:
        """Reads a file corpus straight into this session's HBM."""
        s, _keep = spec._native()
        err = C.create_string_buffer(1024)
        _raise(self._lib.ig_session_load_files(self._h, C.byref(s), err, len(err)), err)

    def run_files(self, spec: CorpusSpec, cfg: IntergramConfig,
                  materialize: bool = True) -> IntergramsResult:
        """Reads a file corpus into HBM and runs on it; the dense pass consumes
        the corpus while later files are still being read (whole-file and
        chunk records)."""
        cfg.validate()
        s, _keep = spec._native()
        err = C.create_string_buffer(1024)
        out = N.ig_result()
        params = cfg._params()
        rc = self._lib.ig_session_run_files(self._h, C.byref(s), C.byref(params), C.byref(out),
                                            err, len(err))
        _raise(rc, err)
        try:
            return _result(out, materialize)
        finally:
            self._lib.ig_result_free(C.byref(out))

    def corpus(self) -> Tuple[np.ndarray, np.ndarray]:
        """The resident corpus copied back: (data u8, offsets u64)."""
        m, tot = C.c_uint64(0), C.c_uint64(0)
        err = C.create_string_buffer(1024)
        _raise(self._lib.ig_session_corpus(self._h, None, 0, None, 0, C.byref(m), C.byref(tot),
                                           err, len(err)), err)
        data = np.zeros(max(tot.value, 1), np.uint8)
        off = np.zeros(m.value + 1, np.uint64)
        _raise(self._lib.ig_session_corpus(self._h, data.ctypes.data, tot.value,
                                           off.ctypes.data, off.size, C.byref(m), C.byref(tot),
                                           err, len(err)), err)
        return data[:tot.value], off

    @property
    def launches(self) -> int:
        return int(self._lib.ig_session_launches(self._h))

    def set_profiling(self, on: bool) -> None:
        """Per-kernel-family device timing (CUDA events on the session stream)."""
        self._lib.ig_session_set_profiling(self._h, 1 if on else 0)

    def kernel_stats(self, reset: bool = False) -> dict:
        """{family: (total_ms, launches)} accumulated since the last reset."""
        n = len(N.KERNEL_FAMILIES)
        ms = np.zeros(n, np.float64)
        cnt = np.zeros(n, np.uint64)
        self._lib.ig_session_kernel_stats(self._h, ms.ctypes.data, cnt.ctypes.data, n,
                                          1 if reset else 0)
        return {f: (float(ms[i]), int(cnt[i])) for i, f in enumerate(N.KERNEL_FAMILIES)}

    def close(self) -> None:
        if self._h:
            self._lib.ig_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
