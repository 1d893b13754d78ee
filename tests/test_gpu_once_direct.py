"""Count-once small-alphabet passes against the C oracle.

With <= 16 distinct bytes in the corpus, an extension pass whose K' * A
candidates fit a shared-memory bitmap counts each long sequence with one CTA
and no routing.  Results must equal the reference algorithm's
(proj/src/intergrams.cpp:44-66 with counting.hpp:48-74), with and without the
direct path (IG_NO_DIRECT=1 forces the route path)."""
import functools
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from paper_2511_14955_b200 import synth as S

pytestmark = pytest.mark.gpu

ONCE = ig.CountMode.kOnce


@functools.lru_cache(maxsize=None)
def corpus(name):
    if name == "acgt":  # c4's order-5 Markov generator: 4 bytes
        return S.generate(S.scaled(S.CONFIGS["c4"], num_seqs=24, seq_len=40_000))
    rng = np.random.default_rng(3)
    if name == "mixed":  # 13 bytes, sequences of 1 .. 30000 bytes (short and long paths)
        lens = rng.integers(1, 30_000, 60)
        data = rng.choice(np.frombuffer(b"ACGTNacgtn-.x", np.uint8), int(lens.sum()))
    else:  # 16 bytes exactly: the largest alphabet the direct path takes
        lens = rng.integers(9_000, 20_000, 30)
        data = rng.integers(0, 16, int(lens.sum()), dtype=np.uint8) * 7
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    return data.astype(np.uint8), off


@functools.lru_cache(maxsize=None)
def oracle(name, n, k):
    data, off = corpus(name)
    return O.oracle_run(data, off, n, k, 1.5, int(ONCE))


@pytest.mark.parametrize("name", ["acgt", "mixed", "hex16"])
@pytest.mark.parametrize("n,k", [(8, 65536), (6, 300), (5, 20), (3, 50)])
@pytest.mark.parametrize("path", ["direct", "direct-chd", "route", "resident"])
def test_once_small_alphabet_equals_oracle(gpu_lib, name, n, k, path):
    # direct: the one-shot call (pipelined load: extension passes direct, dense
    # pass routed); direct-chd: the CHD lookup instead of the rank table;
    # route: no direct path; resident: Session.load + run, where the dense
    # pass is direct too (the corpus alphabet is known)
    data, off = corpus(name)
    rc, keys, counts, rows, diag = oracle(name, n, k)
    assert rc == 0
    env = {"direct-chd": {"IG_NO_DIRECT_LUT": "1"}, "route": {"IG_NO_DIRECT": "1"}}.get(path, {})
    old = {v: os.environ.get(v) for v in ("IG_NO_DIRECT", "IG_NO_DIRECT_LUT")}
    try:
        for v in old:
            os.environ.pop(v, None)
        os.environ.update(env)
        icfg = ig.IntergramConfig(n=n, k=k, z=1.5, mode=ONCE)
        if path == "resident":
            sess = ig.Session(device=0)
            sess.load(ig.Corpus(data, off))
            r = sess.run(icfg)
            r2 = sess.run(icfg)  # the corpus alphabet is measured once per load
            sess.close()
            assert np.array_equal(r2.keys, keys) and np.array_equal(r2.counts, counts)
        else:
            r = ig.run_intergrams(ig.Corpus(data, off), icfg)
    finally:
        for v, x in old.items():
            os.environ.pop(v, None)
            if x is not None:
                os.environ[v] = x
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    assert r.diagnostics == diag
    assert [p.retained for p in r.passes] == [q["retained"] for q in rows]


@functools.lru_cache(maxsize=None)
def few_long(nseq):
    """nseq long sequences (a genome read one chromosome per sequence):
    the direct path splits each into parts counted by different CTAs, whose
    bitmaps are OR-ed per sequence before counting (DirectItem)."""
    return S.generate(S.scaled(S.CONFIGS["c4"], num_seqs=nseq, seq_len=3 << 20))


@pytest.mark.parametrize("nseq", [1, 3])
@pytest.mark.parametrize("split", [None, "65536", "1000"])
def test_once_direct_few_long_sequences_split(gpu_lib, nseq, split):
    # split None: the default plan (>= 1 MiB parts of the 3 MiB sequences);
    # 65536 / 1000: forced small parts (many parts per sequence, part ends
    # inside a 16-byte segment)
    data, off = few_long(nseq)
    rc, keys, counts, rows, diag = O.oracle_run(data, off, 8, 4096, 1.5, int(ONCE))
    assert rc == 0
    old = os.environ.get("IG_DIRECT_SPLIT_BYTES")
    try:
        if split:
            os.environ["IG_DIRECT_SPLIT_BYTES"] = split
        for resident in (False, True):
            icfg = ig.IntergramConfig(n=8, k=4096, z=1.5, mode=ONCE)
            if resident:
                sess = ig.Session(device=0)
                sess.load(ig.Corpus(data, off))
                r = sess.run(icfg)
                sess.close()
            else:
                r = ig.run_intergrams(ig.Corpus(data, off), icfg)
            assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
            assert [p.retained for p in r.passes] == [q["retained"] for q in rows]
    finally:
        os.environ.pop("IG_DIRECT_SPLIT_BYTES", None)
        if old is not None:
            os.environ["IG_DIRECT_SPLIT_BYTES"] = old
