"""Seeded synthetic corpora with BASELINE.json's config shapes (csrc/synth.c).

The paper's corpora (EMBER, C4, 1000gp) are not available; these seeded
generators reproduce the BASELINE configs' shapes, sizes and value
distributions.  The generator itself is pinned in csrc/synth.c's header.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, replace
from typing import Tuple

import numpy as np

from ._native import LIB_DIR

K_ZIPF, K_LOGNORMAL, K_MARKOV, K_MIXED = 1, 3, 4, 5
VOCAB_SEED = 0x1B200


class igs_spec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("num_seqs", C.c_uint64), ("seq_len", C.c_uint64),
                ("total", C.c_uint64), ("seed", C.c_uint64), ("vocab_seed", C.c_uint64)]


@dataclass(frozen=True)
class Config:
    name: str
    kind: int
    num_seqs: int
    seq_len: int
    total: int
    seed: int
    n: int
    k: int
    mode: int  # 0 once, 1 all
    z: float = 1.5
    gpus: str = "1"

    def spec(self) -> igs_spec:
        return igs_spec(self.kind, self.num_seqs, self.seq_len, self.total, self.seed, VOCAB_SEED)

    def describe(self) -> str:
        return DESCRIPTIONS[self.name]


MiB = 1 << 20
GiB = 1 << 30
CONFIGS = {
    "c1": Config("c1", K_ZIPF, 256, 256 * 1024, 256 * 256 * 1024, 1, 4, 1024, 1),
    "c2": Config("c2", K_ZIPF, 4096, MiB, 4 * GiB, 2, 6, 10000, 0),
    "c3": Config("c3", K_LOGNORMAL, 0, 0, 16 * GiB, 3, 8, 100000, 1, gpus="1/2/4/8"),
    "c4": Config("c4", K_MARKOV, 8192, 4 * MiB, 32 * GiB, 4, 8, 65536, 0),
    "c5": Config("c5", K_MIXED, 65536, MiB, 64 * GiB, 5, 8, 1000000, 1, gpus="8"),
}
DESCRIPTIONS = {
    "c1": "256 x 256 KiB Zipf(1.1) 65536-token corpus, n=4 k=1024 count-all",
    "c2": "4096 x 1 MiB Zipf(1.1) token corpus, n=6 k=10000 count-once",
    "c3": "16 GiB lognormal(12,1.5)-length Zipf token corpus, n=8 k=100000 count-all",
    "c4": "8192 x 4 MiB ACGT order-5 Markov Dirichlet(0.3), n=8 k=65536 count-once",
    "c5": "65536 x 1 MiB 90% uniform + 10% Zipf runs, n=8 k=1000000 count-all",
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        path = os.path.join(LIB_DIR, "libigsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C paper_2511_14955_b200`")
        L = C.CDLL(path)
        L.igs_offsets.argtypes = [C.POINTER(igs_spec), C.c_void_p]
        L.igs_offsets.restype = C.c_uint64
        L.igs_fill.argtypes = [C.POINTER(igs_spec), C.c_void_p, C.c_uint64, C.c_uint64,
                               C.c_void_p, C.c_int]
        L.igs_fill.restype = C.c_int
        _lib = L
    return _lib


def offsets(cfg: Config) -> np.ndarray:
    sp = cfg.spec()
    m = lib().igs_offsets(C.byref(sp), None)
    off = np.zeros(m + 1, np.uint64)
    lib().igs_offsets(C.byref(sp), off.ctypes.data)
    return off


def generate(cfg: Config, first: int = 0, count: int = -1, threads: int = 0,
             out: np.ndarray = None) -> Tuple[np.ndarray, np.ndarray]:
    """Sequences [first, first+count) of cfg as (data u8, offsets u64 rebased to 0).
    `out` may supply the (e.g. pinned) destination buffer."""
    off_all = offsets(cfg)
    m = off_all.size - 1
    if count < 0:
        count = m - first
    count = max(0, min(count, m - first))
    off = off_all[first:first + count + 1] - off_all[first]
    total = int(off[-1]) if off.size else 0
    data = out[:total] if out is not None else np.empty(total, np.uint8)
    if threads <= 0:
        threads = os.cpu_count() or 1
    sp = cfg.spec()
    if count:
        lib().igs_fill(C.byref(sp), off_all.ctypes.data, first, count, data.ctypes.data, threads)
    return data, off.astype(np.uint64)


def scaled(cfg: Config, num_seqs: int = None, seq_len: int = None, total: int = None) -> Config:
    """Same generator at a different size (test corpora)."""
    kw = {}
    if num_seqs is not None:
        kw["num_seqs"] = num_seqs
    if seq_len is not None:
        kw["seq_len"] = seq_len
    if total is not None:
        kw["total"] = total
    return replace(cfg, **kw)


def fingerprint(data: np.ndarray, off: np.ndarray) -> str:
    """Cheap corpus fingerprint (sha256 over the offsets and the first 64 bytes
    of every 1 MiB block) pinning the generator output behind a golden."""
    import hashlib
    h = hashlib.sha256(np.ascontiguousarray(off, np.uint64).tobytes())
    n = int(data.size)
    if n:
        idx = (np.arange(0, n, 1 << 20, dtype=np.int64)[:, None] + np.arange(64)[None, :])
        h.update(np.asarray(data)[np.minimum(idx, n - 1)].tobytes())
    return h.hexdigest()[:16]
