"""GPU parity of the sort-based exact paths (paper_2511_14955_b200/csrc/exact.cu)
through the C-ABI: naive_topk (oracle.cpp:7-47), run_hashgram
(hashgram.cpp:325-383) and featurize (metrics.cpp:83-132), against the
reference's golden vectors (tests/golden/golden_extra.json) and the C oracle
on seeded random corpora.  Bit-exact: same grams, counts, order, pass rows."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from tests import util

pytestmark = pytest.mark.gpu

GX = json.load(open(os.path.join(util.HERE, "golden", "golden_extra.json")))
ONCE, ALL = ig.CountMode.kOnce, ig.CountMode.kAll


def as_tsv(topk):
    return "".join(f"{g.gram.hex()}\t{g.count}\n" for g in topk)


def corpus_of(data, off):
    return ig.Corpus(data, off)


def oracle_naive_tsv(data, off, n, mode, k):
    keys, counts = O.oracle_naive(data, off, n, mode, k)
    return util.tsv(keys, counts, n)


# ------------------------------------------------------------------ naive

@pytest.mark.parametrize("n", range(1, 9))
@pytest.mark.parametrize("mode", [ONCE, ALL])
def test_naive_matches_oracle(gpu_lib, n, mode):
    rng = O.Mt64(4000 + n)
    for alphabet, max_len in ((3, 300), (16, 500), (256, 200)):
        seqs = O.random_corpus(rng, 20, max_len, alphabet)
        d, off = O.csr(seqs)
        for k in (1, 7, 100, 100000):
            got = ig.naive_topk(corpus_of(d, off), n, mode, k)
            assert as_tsv(got) == oracle_naive_tsv(d, off, n, int(mode), k), (alphabet, k)


def test_naive_golden_cases(gpu_lib):
    # the reference's own run_intergrams goldens with full retention equal
    # the naive top-k (tests/test_intergrams.cpp:149-161); check the naive
    # path on the golden corpora against the oracle restatement
    for c in util.golden()["cases"][:40]:
        data, off = util.corpus_from(c["corpus"])
        if c["n"] > 8:
            continue
        got = ig.naive_topk(corpus_of(data, off), c["n"], ig.CountMode(c["mode"]), c["k"])
        assert as_tsv(got) == oracle_naive_tsv(data, off, c["n"], c["mode"], c["k"])


def test_naive_edges(gpu_lib):
    assert ig.naive_topk([], 3, ONCE, 5) == []
    assert ig.naive_topk([b"", b"ab"], 3, ALL, 5) == []
    r = ig.naive_topk([b"aaaa", b"aaab"], 3, ONCE, 2)  # SPEC.md:693 golden
    assert as_tsv(r) == "616161\t2\n616162\t1\n"
    r = ig.naive_topk([b"\xff" * 20], 8, ALL, 3)  # all-ones 8-gram key
    assert [(g.gram, g.count) for g in r] == [(b"\xff" * 8, 13)]
    with pytest.raises(ig.ConfigError, match="guard"):
        ig.naive_topk([b"x" * 100], 3, ALL, 1, max_corpus_bytes=99)
    assert len(ig.naive_topk([b"x" * 100], 3, ALL, 1, max_corpus_bytes=100)) == 1


def test_naive_batch_merge(gpu_lib, monkeypatch):
    # many small batches force the merge (second sort + reduce-by-key) path
    monkeypatch.setenv("IG_EXACT_BATCH_BYTES", "700")
    rng = O.Mt64(77)
    seqs = O.random_corpus(rng, 40, 600, 4) + O.random_corpus(rng, 40, 2000, 4)
    d, off = O.csr(seqs)
    for n in (2, 5, 8):
        for mode in (ONCE, ALL):
            got = ig.naive_topk(corpus_of(d, off), n, mode, 300)
            assert as_tsv(got) == oracle_naive_tsv(d, off, n, int(mode), 300)


# --------------------------------------------------------------- hashgram

def hg_id(c):
    return f"n{c['n']}-m{c['mode']}-B{c['buckets']}-k{c['k']}"


@pytest.mark.parametrize("case", GX["hashgram"], ids=[hg_id(c) for c in GX["hashgram"]])
def test_hashgram_matches_reference_golden(gpu_lib, case):
    data, off = util.corpus_from(case["corpus"])
    cfg = ig.HashgramConfig(buckets=case["buckets"], n=case["n"], k=case["k"],
                            mode=ig.CountMode(case["mode"]), seed=case["seed"])
    r = ig.run_hashgram(corpus_of(data, off), cfg)
    assert as_tsv(r.topk) == case["tsv"]
    rows = [{"label": p.label, "gram_len": p.gram_len, "bytes_processed": p.bytes_processed,
             "candidate_space": p.candidate_space, "retained": p.retained,
             "retained_short": p.retained_short} for p in r.passes]
    assert rows == case["passes"]


@pytest.mark.parametrize("buckets", [1, 3, 1000, 1 << 31, (1 << 33) + 7, 1 << 50])
def test_hashgram_matches_oracle(gpu_lib, buckets):
    rng = O.Mt64(31 + buckets % 1000)
    for _ in range(4):
        seqs = O.random_corpus(rng, 16, 400, 6)
        d, off = O.csr(seqs)
        for n in (2, 4, 7, 8):
            for mode in (ONCE, ALL):
                for k, seed in ((5, 0), (60, 2 ** 64 - 1)):
                    r = ig.run_hashgram(corpus_of(d, off), ig.HashgramConfig(
                        buckets=buckets, n=n, k=k, mode=mode, seed=seed))
                    rc, keys, counts, kept, ex = O.oracle_hashgram(d, off, n, k, int(mode),
                                                                   buckets, seed)
                    assert rc == 0
                    assert as_tsv(r.topk) == util.tsv(keys, counts, n)
                    assert r.passes[1].retained == kept and r.passes[2].retained == ex


# -------------------------------------------------------------- featurize

@pytest.mark.parametrize("case", GX["featurize"], ids=lambda c: f"n{c['n']}-v{len(c['vocab'])}")
def test_featurize_matches_reference_golden(gpu_lib, case):
    data, off = util.corpus_from(case["corpus"])
    vocab = [ig.GramCount(bytes.fromhex(v), 1) for v in case["vocab"]]
    m = ig.featurize(corpus_of(data, off), vocab)
    assert m.rows == case["rows"] and m.cols == len(vocab)
    assert [(r << 32) | c for r, c in m.entries] == case["entries"]


def test_featurize_matches_oracle(gpu_lib, monkeypatch):
    rng = O.Mt64(555)
    for t in range(6):
        if t >= 3:
            monkeypatch.setenv("IG_EXACT_BATCH_BYTES", "1000")
        seqs = O.random_corpus(rng, 60, 900, 4)
        d, off = O.csr(seqs)
        for n in (1, 3, 6, 8):
            grams = sorted({s[i:i + n] for s in seqs for i in range(0, max(len(s) - n + 1, 0), 3)})
            vocab = grams[::max(1, len(grams) // 50)] + grams[:5]
            m = ig.featurize(corpus_of(d, off), vocab)
            want = O.oracle_featurize(d, off, np.array([int.from_bytes(g, "big") for g in vocab],
                                                       np.uint64), n)
            assert [(r << 32) | c for r, c in m.entries] == want.tolist()
            assert m.rows == len(seqs)


def test_featurize_edges(gpu_lib):
    m = ig.featurize([b"abc", b"", b"zzz"], [])
    assert (m.rows, m.cols, m.entries) == (3, 0, [])
    m = ig.featurize([b"abc", b"", b"zzz"], [ig.GramCount(b"", 1)])  # empty gram
    assert m.entries == [(0, 0), (1, 0), (2, 0)]
    m = ig.featurize([], [ig.GramCount(b"ab", 1)])
    assert (m.rows, m.entries) == (0, [])


# ------------------------------------------- full-size cross-path property

@pytest.mark.slow
def test_c2_once_counts_equal_featurize_popcounts(gpu_lib):
    """At BASELINE config 2 (4096 x 1 MiB, n=6, k=10000, ONCE) every count the
    Intergrams path reports is the number of sequences containing the gram,
    which featurize (an independent kernel path) measures exactly."""
    from paper_2511_14955_b200 import synth as S
    data, off = S.generate(S.CONFIGS["c2"], 0, -1)
    c = ig.Corpus(data, off)
    r = ig.run_intergrams(c, ig.IntergramConfig(n=6, k=10000, z=1.5, mode=ONCE))
    m = ig.featurize(c, r.topk)
    pops = m.column_popcounts()
    assert pops == [g.count for g in r.topk]


def test_hashgram_large_b_equals_oracle(gpu_lib):
    # the corpora of the reference's own test_hashgram.cpp:86-101 (B = 2^40,
    # n = 4, k = 8, count-once, seed 7): the GPU path equals the reference
    # algorithm (oracle) there; the reference binary itself cannot allocate
    # CountTable(2^40) (tests/test_ref_unit_tests.py)
    rng = O.Mt64(1234)
    for _ in range(10):
        d, off = O.csr(O.random_corpus(rng, 10, 100, 4))
        r = ig.run_hashgram(corpus_of(d, off), ig.HashgramConfig(
            buckets=1 << 40, n=4, k=8, mode=ONCE, seed=7))
        rc, keys, counts, kept, ex = O.oracle_hashgram(d, off, 4, 8, 0, 1 << 40, 7)
        assert rc == 0
        assert as_tsv(r.topk) == util.tsv(keys, counts, 4)
        assert r.passes[1].retained == kept and r.passes[2].retained == ex
