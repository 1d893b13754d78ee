"""Differential test: the C oracle against the reference compiled from its own
sources (oracle/_ref), on fresh seeded corpora.  Skipped where the reference
build is unavailable (the golden fixtures still pin the oracle there)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference build unavailable")


@pytest.mark.parametrize("seed", range(20))
def test_random_configs(seed):
    rng = O.Mt64(31337 + seed)
    seqs = O.random_corpus(rng, 16, 500, [2, 5, 17, 256][seed % 4])
    d, off = O.csr(seqs)
    for n in (1, 2, 3, 4, 6, 8):
        for mode in (O.ONCE, O.ALL):
            k = 1 + rng() % 30
            z = 1.0 + (rng() % 5) / 2
            a = O.oracle_run(d, off, n, k, z, mode)
            b = O.ref_run(d, off, n, k, z, mode, 1 + seed % 3)
            assert a[0] == b[0]
            if a[0]:
                continue
            assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
            assert a[4] == b[4]


@pytest.mark.parametrize("seed", range(6))
def test_extend_tables(seed):
    rng = O.Mt64(606 + seed)
    seqs = O.random_corpus(rng, 10, 120, 6)
    d, off = O.csr(seqs)
    j = 4 + seed % 2
    allp, _ = O.oracle_naive(d, off, j - 1, O.ONCE, 1 << 20)
    kept = [int(x) for x in allp if rng() % 2 == 0] or [int(allp[0])]
    pre = [x.to_bytes(8, "big")[8 - (j - 1):] for x in kept]
    for mode in (O.ONCE, O.ALL):
        rc, t, b = O.oracle_extend(d, off, np.array(kept, np.uint64), j - 1, j, mode)
        rc2, t2, b2, err = O.ref_extend(d, off, pre, j, mode)
        assert rc == rc2 == 0 and np.array_equal(t, t2) and b == b2
