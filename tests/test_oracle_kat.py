"""Known-answer tests of the reference suite (proj/tests/*.cpp), restated on the
C oracle.  Each test cites the reference test it restates."""
import numpy as np
import pytest

from oracle import oracle as O

ONCE, ALL = O.ONCE, O.ALL


def key(g: bytes) -> int:
    return int.from_bytes(g, "big")


def run(seqs, n, k, z, mode):
    d, off = O.csr(seqs)
    return O.oracle_run(d, off, n, k, z, mode)


def test_count_once_dedups_within_a_sequence():  # test_dense_pass.cpp:50-55
    d, off = O.csr([b"aaaa"])
    t = O.oracle_count_dense(d, off, 3, ONCE)
    assert t[key(b"aaa")] == 1 and t.sum() == 1


def test_count_all_counts_every_occurrence():  # test_dense_pass.cpp:57-62
    d, off = O.csr([b"aaaa"])
    t = O.oracle_count_dense(d, off, 3, ALL)
    assert t[key(b"aaa")] == 2 and t.sum() == 2


def test_topk_trigrams_ranked():  # test_dense_pass.cpp:88-101
    d, off = O.csr([b"aaaa", b"aaab"])
    t = O.oracle_count_dense(d, off, 3, ONCE)
    keys, counts = O.oracle_top_k(t, 2)
    assert list(zip(keys, counts)) == [(key(b"aaa"), 2), (key(b"aab"), 1)]
    assert len(O.oracle_top_k(t, 10)[0]) == 2


def test_tied_trigrams_byte_ascending():  # test_dense_pass.cpp:103-118
    d, off = O.csr([b"abcxbcd"])
    t = O.oracle_count_dense(d, off, 3, ONCE)
    keys, counts = O.oracle_top_k(t, 5)
    assert len(keys) == 5 and list(keys) == sorted(keys) and set(counts) == {1}


def test_once_le_all_le_m():  # test_dense_pass.cpp:120-131
    rng = O.Mt64(77)
    seqs = O.random_corpus(rng, 12, 60, 4)
    d, off = O.csr(seqs)
    once = O.oracle_count_dense(d, off, 3, ONCE)
    allc = O.oracle_count_dense(d, off, 3, ALL)
    assert (once <= allc).all() and (once <= len(seqs)).all()


def test_count_all_conservation():  # test_dense_pass.cpp:133-139
    rng = O.Mt64(88)
    seqs = O.random_corpus(rng, 15, 120, 32)
    d, off = O.csr(seqs)
    allc = O.oracle_count_dense(d, off, 3, ALL)
    assert allc.sum() == sum(max(0, len(s) - 2) for s in seqs)


def test_top_k_tie_break():  # test_counting.cpp:129-142
    t = np.array([3, 3, 1, 0], np.uint64)
    keys, counts = O.oracle_top_k(t, 2)
    assert list(keys) == [0, 1] and list(counts) == [3, 3]


def test_top_k_all_zero_is_empty():  # test_counting.cpp:144-147
    assert len(O.oracle_top_k(np.zeros(100, np.uint64), 5)[0]) == 0


def test_top_k_equals_full_sort():  # test_counting.cpp:149-171
    rng = O.Mt64(99)
    for _ in range(8):
        t = np.array([rng() % 16 for _ in range(1000)], np.uint64)
        for k in (1, 10, 999, 5000):
            keys, counts = O.oracle_top_k(t, k)
            ref = sorted(((int(c), i) for i, c in enumerate(t) if c), key=lambda e: (-e[0], e[1]))
            ref = ref[:k]
            assert [(int(c), int(i)) for i, c in zip(keys, counts)] == ref


def test_candidate_id_arithmetic():  # test_intergrams.cpp:41-46
    # the oracle's extension table is indexed rank*256 + last byte
    d, off = O.csr([b"abab"])
    rc, t, b = O.oracle_extend(d, off, np.array([key(b"aba")], np.uint64), 3, 4, ONCE)
    assert rc == 0 and t.size == 256 and t[ord("b")] == 1 and t.sum() == 1
    rc, t, b = O.oracle_extend(d, off, np.array([key(b"bab")], np.uint64), 3, 4, ONCE)
    assert rc == 0 and t.sum() == 0  # test_intergrams.cpp:62-66


def test_extend_requires_depth():  # test_intergrams.cpp:112-117
    d, off = O.csr([b"abcd"])
    rc, _, _ = O.oracle_extend(d, off, np.array([key(b"ab")], np.uint64), 2, 4, ONCE)
    assert rc == 2


def test_four_way_tie():  # test_intergrams.cpp:119-125
    rc, keys, counts, _, _ = run([b"abab", b"abba"], 4, 1, 100.0, ONCE)
    assert rc == 0 and list(keys) == [key(b"abab")] and list(counts) == [1]


def test_degenerate_corpora_diagnostics():  # test_intergrams.cpp:210-217
    rc, keys, counts, rows, diag = run([b"aaaa", b"aaab"], 4, 5, 10.0, ONCE)
    assert rc == 0 and diag and list(counts) == [1, 1]


def test_pass_rows_structure():  # test_intergrams.cpp:219-237
    rng = O.Mt64(5)
    seqs = O.random_corpus(rng, 6, 300, 30)
    rc, keys, counts, rows, diag = run(seqs, 6, 4, 2.0, ONCE)
    counting = [r for r in rows if r["bytes_processed"] > 0]
    assert len(counting) == 4
    assert all(r["bytes_processed"] == sum(len(s) for s in seqs) for r in counting)
    assert len(rows) == 2 * 6 - 4


def test_invalid_configs():  # test_intergrams.cpp:239-243
    d, off = O.csr([b"abc"])
    assert O.oracle_run(d, off, 0, 1, 1.0, ONCE)[0] == 2
    assert O.oracle_run(d, off, 4, 0, 1.0, ONCE)[0] == 2
    assert O.oracle_run(d, off, 4, 1, 0.5, ONCE)[0] == 2
    assert O.oracle_run(d, off, 4, 1, float("nan"), ONCE)[0] == 2


def test_naive_kats():  # test_oracle.cpp:8-59
    d, off = O.csr([b"abcab"])
    keys, counts = O.oracle_naive(d, off, 3, ONCE, 10)
    assert sorted(zip(keys, counts)) == sorted([(key(b"abc"), 1), (key(b"bca"), 1),
                                               (key(b"cab"), 1)])
    d, off = O.csr([b"abcab", b"abc"])
    keys, counts = O.oracle_naive(d, off, 3, ONCE, 10)
    assert dict(zip(keys, counts))[key(b"abc")] == 2
    d, off = O.csr([b"ab"])
    assert len(O.oracle_naive(d, off, 3, ALL, 10)[0]) == 0


def test_full_retention_equals_naive():  # test_intergrams.cpp:149-161
    rng = O.Mt64(909)
    for _ in range(10):
        seqs = O.random_corpus(rng, 8, 200, 4)
        d, off = O.csr(seqs)
        z = max(1.0, (int(off[-1]) + 1) / 16)
        for mode in (ONCE, ALL):
            rc, keys, counts, _, _ = O.oracle_run(d, off, 5, 16, z, mode)
            nk, nc = O.oracle_naive(d, off, 5, mode, 16)
            assert rc == 0 and list(keys) == list(nk) and list(counts) == list(nc)


def test_mt19937_64_known_value():
    # std::mt19937_64 default seed 5489: the 10000th output is 9981545732273789042
    rng = O.Mt64(5489)
    v = None
    for _ in range(10000):
        v = rng()
    assert v == 9981545732273789042
