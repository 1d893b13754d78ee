"""GPU parity: the CUDA path (through the C-ABI) against the C oracle and the
reference's own known-answer tests (proj/tests/test_intergrams.cpp,
test_dense_pass.cpp).  Bit-exact: same grams, same counts, same order."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig

pytestmark = pytest.mark.gpu

ONCE, ALL = ig.CountMode.kOnce, ig.CountMode.kAll


def cfg(n, k, z, mode):
    return ig.IntergramConfig(n=n, k=k, z=z, mode=mode)


def oracle_topk(seqs, n, mode, k):
    d, off = O.csr(seqs)
    keys, counts = O.oracle_naive(d, off, n, int(mode), k)
    return [ig.GramCount(ig.key_to_gram(int(a), n), int(b)) for a, b in zip(keys, counts)]


def test_four_way_tie_resolves_canonically(gpu_lib):
    # tests/test_intergrams.cpp:119-125
    r = ig.run_intergrams([b"abab", b"abba"], cfg(4, 1, 100.0, ONCE))
    assert [tuple(g) for g in r.topk] == [(b"abab", 1)]


def test_dense_once_all_kat(gpu_lib):
    # tests/test_dense_pass.cpp:50-62
    t = ig.count_trigrams([b"aaaa"], ONCE)
    assert t[0x616161] == 1 and t.sum() == 1
    t = ig.count_trigrams([b"aaaa"], ALL)
    assert t[0x616161] == 2 and t.sum() == 2


@pytest.mark.parametrize("seed", [2024, 31, 77])
def test_dense_table_equals_oracle(gpu_lib, seed):
    # tests/test_dense_pass.cpp:64-86
    rng = O.Mt64(seed)
    for _ in range(5):
        seqs = O.random_corpus(rng, 20, 100, 8)
        d, off = O.csr(seqs)
        for n in (1, 2, 3):
            for mode in (ONCE, ALL):
                got = ig.count_dense(seqs, n, mode)
                want = O.oracle_count_dense(d, off, n, int(mode))
                assert np.array_equal(got, want), (n, mode)


def test_full_retention_reproduces_oracle(gpu_lib):
    # tests/test_intergrams.cpp:149-161
    rng = O.Mt64(909)
    for _ in range(10):
        seqs = O.random_corpus(rng, 8, 200, 4)
        k = 16
        total = sum(len(s) for s in seqs)
        z = max(1.0, (total + 1) / k)
        for mode in (ONCE, ALL):
            r = ig.run_intergrams(seqs, cfg(5, k, z, mode))
            assert r.topk == oracle_topk(seqs, 5, mode, k)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("mode", [ONCE, ALL])
def test_run_equals_c_oracle(gpu_lib, n, mode):
    rng = O.Mt64(1000 + n)
    for _ in range(4):
        seqs = O.random_corpus(rng, 12, 400, 6)
        d, off = O.csr(seqs)
        rc, keys, counts, rows, diag = O.oracle_run(d, off, n, 9, 1.5, int(mode))
        if rc != 0:
            with pytest.raises(ig.ConfigError):
                ig.run_intergrams(seqs, cfg(n, 9, 1.5, mode))
            continue
        r = ig.run_intergrams(seqs, cfg(n, 9, 1.5, mode))
        assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
        assert r.diagnostics == diag
        assert [(p.label, p.gram_len, p.bytes_processed, p.candidate_space, p.retained,
                 p.retained_short) for p in r.passes] == \
               [(q["label"], q["gram_len"], q["bytes_processed"], q["candidate_space"],
                 q["retained"], q["retained_short"]) for q in rows]


@pytest.mark.parametrize("seed", range(6))
def test_extend_pass_table_equals_oracle(gpu_lib, seed):
    # tests/test_intergrams.cpp:69-110: random prefix subsets, both modes
    rng = O.Mt64(606 + seed)
    seqs = O.random_corpus(rng, 10, 120, 6)
    d, off = O.csr(seqs)
    j = 4 + seed % 2
    allp, _ = O.oracle_naive(d, off, j - 1, int(ONCE), 1 << 20)
    kept = [int(x) for x in allp if rng() % 2 == 0] or [int(allp[0])]
    pre = [ig.key_to_gram(x, j - 1) for x in kept]
    for mode in (ONCE, ALL):
        t, bp = ig.extend_pass(seqs, pre, j, mode)
        rc, t2, b2 = O.oracle_extend(d, off, np.array(kept, np.uint64), j - 1, j, int(mode))
        assert rc == 0 and np.array_equal(t, t2) and bp == b2


def test_extend_pass_rejects_wrong_depth(gpu_lib):
    # tests/test_intergrams.cpp:112-117
    with pytest.raises(ig.ConfigError):
        ig.extend_pass([b"abcd"], [b"ab"], 4, ONCE)
    with pytest.raises(ig.ConfigError):
        ig.extend_pass([b"abcd"], [], 4, ONCE)


def test_extend_pass_kat(gpu_lib):
    # tests/test_intergrams.cpp:48-67
    t, _ = ig.extend_pass([b"abab"], [b"aba"], 4, ONCE)
    assert t.size == 256 and t[ig.candidate_id(0, ord("b"))] == 1 and t.sum() == 1
    t, _ = ig.extend_pass([b"abab"], [b"bab"], 4, ONCE)
    assert t.sum() == 0


@pytest.mark.parametrize("seed", [99, 123, 7])
def test_top_k_api_equals_oracle(gpu_lib, seed):
    # tests/test_counting.cpp:149-171 (k beyond capacity included)
    rng = O.Mt64(seed)
    t = np.array([rng() % 16 for _ in range(1000)], np.uint64)
    for k in (1, 10, 999, 5000):
        keys, counts = ig.top_k(t, k)
        k2, c2 = O.oracle_top_k(t, k)
        assert np.array_equal(keys, k2) and np.array_equal(counts, c2)
    with pytest.raises(ig.ConfigError):
        ig.top_k(t, 0)
    assert ig.top_k(np.zeros(100, np.uint64), 5)[0].size == 0  # test_counting.cpp:144-147


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_once_mixed_short_and_long_sequences(gpu_lib, seed):
    # count-once splits sequences by length: <= 512 B (a warp each), <= 8 KiB
    # (a CTA each, both in k_once_short) and longer (route path); all three
    # classes count into one table and must match the oracle together
    rng = O.Mt64(4400 + seed)
    seqs = []
    for i in range(60):
        cls = rng() % 3
        n = (rng() % 513) if cls == 0 else (513 + rng() % 7680) if cls == 1 else (8193 + rng() % 40000)
        seqs.append(O.random_bytes(rng, n, 3 + seed))
    d, off = O.csr(seqs)
    for n, k, z in ((3, 50, 1.5), (5, 200, 1.5), (8, 300, 2.0)):
        got = ig.run_intergrams(seqs, cfg(n, k, z, ONCE))
        rc, keys, counts, rows, diag = O.oracle_run(d, off, n, k, z, int(ONCE))
        assert rc == 0
        assert [(g.gram, g.count) for g in got.topk] == \
            [(ig.key_to_gram(int(a), n), int(b)) for a, b in zip(keys, counts)]
