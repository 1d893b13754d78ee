"""Grams longer than 8 bytes (n > 8) against the reference itself.

The reference takes any n (intergrams.cpp:37-42; its PrefixTrie has any
depth, trie.cpp:20-137).  Here passes j <= 8 run on packed u64 keys; a pass
j >= 9 walks each position's prefix rank up from its first 8 bytes through
per-level id -> rank tables and counts by sorting (exact.cu kEmitChain).
Lists come back as gram bytes (ig_result.grams).  Checked against
oracle/_ref (the reference compiled from its own sources): same grams,
counts, order, pass rows and diagnostics, both count modes, through the
one-shot call, a resident session, the seqs entry point and the C++ API."""
import functools

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from paper_2511_14955_b200 import synth as S

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def corpus(name):
    if name == "zipf":  # c2's token generator: repeated long grams
        return S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=48, seq_len=60_000))
    if name == "acgt":  # c4's small alphabet: weak pruning
        return S.generate(S.scaled(S.CONFIGS["c4"], num_seqs=20, seq_len=50_000))
    rng = np.random.default_rng(11)  # ragged: empty / short / long sequences, few bytes
    lens = rng.integers(0, 3000, 70)
    lens[[3, 9, 40]] = 0
    lens[[5, 6]] = [9, 11]
    data = rng.choice(np.frombuffer(b"abcab", np.uint8), int(lens.sum()))
    return data.astype(np.uint8), np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)


@functools.lru_cache(maxsize=None)
def reference(name, n, k, mode):
    data, off = corpus(name)
    return O.ref_run_grams(data, off, n, k, 1.5, mode, 0)


def check(r, ref):
    rc, grams, counts, rows, diag, err = ref
    assert rc == 0, err
    assert r.keys is None and r.grams.shape == grams.shape
    assert np.array_equal(r.grams, grams) and np.array_equal(r.counts, counts)
    assert [p.retained for p in r.passes] == [q["retained"] for q in rows]
    assert [p.candidate_space for p in r.passes] == [q["candidate_space"] for q in rows]
    assert [p.label for p in r.passes] == [q["label"] for q in rows]
    assert r.diagnostics == diag
    assert [g.gram for g in r.topk] == [bytes(g) for g in grams]


@pytest.mark.parametrize("name", ["zipf", "acgt", "ragged"])
@pytest.mark.parametrize("n,k", [(9, 300), (12, 1000), (16, 50)])
@pytest.mark.parametrize("mode", [0, 1])
def test_long_grams_equal_reference(gpu_lib, name, n, k, mode):
    data, off = corpus(name)
    cfg = ig.IntergramConfig(n=n, k=k, z=1.5, mode=ig.CountMode(mode))
    check(ig.run_intergrams(ig.Corpus(data, off), cfg), reference(name, n, k, mode))


@pytest.mark.parametrize("mode", [0, 1])
def test_long_grams_session_and_seqs(gpu_lib, mode):
    data, off = corpus("zipf")
    cfg = ig.IntergramConfig(n=11, k=400, z=2.0, mode=ig.CountMode(mode))
    ref = O.ref_run_grams(data, off, 11, 400, 2.0, mode, 0)
    sess = ig.Session(device=0)
    sess.load(ig.Corpus(data, off))
    check(sess.run(cfg), ref)
    check(sess.run(cfg), ref)  # level tables reused across runs
    sess.close()
    seqs = [bytes(data[off[q]:off[q + 1]]) for q in range(off.size - 1)]
    check(ig.run_intergrams(seqs, cfg), ref)


def test_long_grams_u64_tables(gpu_lib, monkeypatch):
    # the u64 count tables (a > 4 GiB corpus's) through the chain passes
    monkeypatch.setenv("IG_FORCE_U64", "1")
    data, off = corpus("acgt")
    cfg = ig.IntergramConfig(n=10, k=500, z=1.5, mode=ig.CountMode.kAll)
    check(ig.run_intergrams(ig.Corpus(data, off), cfg), reference("acgt", 10, 500, 1))


def test_long_grams_empty_passes(gpu_lib):
    # 8-byte sequences only: pass 9 counts nothing and returns an empty list;
    # at n = 10 pass 10 then has a depth-0 trie (intergrams.cpp:46-48) and
    # the reference raises ConfigError, as the GPU path must
    data = np.frombuffer(b"abcdefgh" * 3, np.uint8).copy()
    off = np.array([0, 8, 16, 24], np.uint64)
    ref = O.ref_run_grams(data, off, 9, 10, 1.5, 1, 0)
    check(ig.run_intergrams(ig.Corpus(data, off),
                            ig.IntergramConfig(n=9, k=10, mode=ig.CountMode.kAll)), ref)
    assert O.ref_run_grams(data, off, 10, 10, 1.5, 1, 0)[0] == 2  # ConfigError
    with pytest.raises(ig.ConfigError):
        ig.run_intergrams(ig.Corpus(data, off),
                          ig.IntergramConfig(n=10, k=10, mode=ig.CountMode.kAll))
