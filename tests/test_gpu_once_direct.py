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
@pytest.mark.parametrize("n,k", [(8, 65536), (6, 300), (5, 20)])
@pytest.mark.parametrize("direct", [True, False])
def test_once_small_alphabet_equals_oracle(gpu_lib, name, n, k, direct):
    data, off = corpus(name)
    rc, keys, counts, rows, diag = oracle(name, n, k)
    assert rc == 0
    old = os.environ.pop("IG_NO_DIRECT", None)
    try:
        if not direct:
            os.environ["IG_NO_DIRECT"] = "1"
        r = ig.run_intergrams(ig.Corpus(data, off), ig.IntergramConfig(n=n, k=k, z=1.5, mode=ONCE))
    finally:
        os.environ.pop("IG_NO_DIRECT", None)
        if old is not None:
            os.environ["IG_NO_DIRECT"] = old
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    assert r.diagnostics == diag
    assert [p.retained for p in r.passes] == [q["retained"] for q in rows]
