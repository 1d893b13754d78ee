"""Count-all extension-pass lookup paths against the C oracle (bit-exact).

The count-all extension pass (proj/src/intergrams.cpp:44-66, one count per
occurrence whose (j-1)-byte prefix is a survivor) has several GPU lookup
structures, chosen by survivor count and prefix length:
shared-memory packed set (small K), the 3-byte-prefix rank bitmap (first
extension pass, K > 4096), packed 8-byte or {key, p} 16-byte global slots,
and hit chaining (each pass probes only positions whose prefix the previous
pass counted).  Every combination must give the reference's list."""
import functools
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from paper_2511_14955_b200 import synth as S

pytestmark = pytest.mark.gpu

ALL = ig.CountMode.kAll


def _corpora():
    # c5-like (90 % uniform bytes + Zipf runs: most windows miss the prefix
    # set) and c3-like (lognormal lengths: short sequences, boundaries at any
    # byte offset, Zipf tokens: most windows hit)
    d5, o5 = S.generate(S.scaled(S.CONFIGS["c5"], num_seqs=6, seq_len=300_001))
    d3, o3 = S.generate(S.scaled(S.CONFIGS["c3"], total=3 << 20))
    # the c5 bytes cut into sequences of 1..6000 bytes: many boundaries, and
    # sequences shorter than the gram length
    rng = np.random.default_rng(11)
    cuts = np.cumsum(rng.integers(1, 6000, d5.size // 1000))
    cuts = cuts[cuts < d5.size]
    om = np.concatenate([[0], cuts, [d5.size]]).astype(np.uint64)
    return {"c5": (d5, o5), "c3": (d3, o3), "mixed": (d5, om)}


CORPORA = None


def corpus(name):
    global CORPORA
    if CORPORA is None:
        CORPORA = _corpora()
    return CORPORA[name]


@functools.lru_cache(maxsize=None)
def oracle(name, k):
    data, off = corpus(name)
    return O.oracle_run(data, off, 8, k, 1.5, int(ALL))


# hot-gram sweeps engage from 32 MiB corpora; these force
# them on the small test corpora, with tiny bucket tables (collisions,
# empty-slot keys), several slices (hit masks OR-ed across sweeps), and u64
# tables counted per segment into a u32 scratch (IG_SEG_TILES: many segments)
HOT = {"IG_HOT_MIN_TILES": "0"}
HOT_SMALL = {**HOT, "IG_HOT_LGNB": "6", "IG_HOT_SLICES": "4"}
HOT_U64 = {**HOT, "IG_HOT_SLICES": "2", "IG_FORCE_U64": "1", "IG_SEG_TILES": "1000"}
TOGGLES = [{}, {"IG_NO_HIT_CHAIN": "1"}, {"IG_NO_RANK_BITMAP": "1"},
           {"IG_NO_HIT_CHAIN": "1", "IG_NO_RANK_BITMAP": "1"},
           HOT, HOT_SMALL, HOT_U64, {**HOT_SMALL, "IG_NO_HIT_CHAIN": "1"},
           {**HOT, "IG_NO_RANK_BITMAP": "1", "IG_HOT_SLICES": "3"},
           {"IG_FORCE_U64": "1", "IG_SEG_TILES": "777", "IG_NO_HOT": "1"},
           # queued sweep: never / always walk a tile live position by live
           # position (the default does for tiles with <= 10 per lane)
           {**HOT, "IG_SPARSE_ITERS": "0"}, {**HOT, "IG_SPARSE_ITERS": "16"},
           {**HOT_SMALL, "IG_SPARSE_ITERS": "16"},
           # the sparse switch forced on (every chained pass) / off
           {**HOT, "IG_SPARSE": "1"}, {**HOT, "IG_SPARSE": "0"},
           # direct hot tables: every candidate that loses its slot counts as
           # important, so every pass falls back to the two-way build
           {**HOT, "IG_HOT_IMPORTANT": "1"}, {**HOT, "IG_HOT_IMPORTANT": "1", "IG_SPARSE": "1"}]


def run_with_env(env, fn):
    saved = {t: os.environ.get(t) for t in env}
    try:
        os.environ.update(env)
        return fn()
    finally:
        for t, v in saved.items():
            if v is None:
                os.environ.pop(t, None)
            else:
                os.environ[t] = v


def _id(d):
    return "-".join(f"{k}={v}" for k, v in d.items()) or "default"


@pytest.mark.parametrize("name", ["c5", "c3", "mixed"])
@pytest.mark.parametrize("k", [40, 5000])  # K' = 60 (shared memory) / 7500 (global, rank bitmap)
@pytest.mark.parametrize("toggles", TOGGLES, ids=_id)
def test_count_all_paths_equal_oracle(gpu_lib, name, k, toggles):
    data, off = corpus(name)
    rc, keys, counts, rows, diag = oracle(name, k)
    assert rc == 0
    r = run_with_env(toggles, lambda: ig.run_intergrams(
        ig.Corpus(data, off), ig.IntergramConfig(n=8, k=k, z=1.5, mode=ALL)))
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    assert r.diagnostics == diag
    assert [p.retained for p in r.passes] == [q["retained"] for q in rows]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("toggles", [HOT, HOT_SMALL, HOT_U64], ids=_id)
def test_hot_sweeps_short_grams_equal_oracle(gpu_lib, n, toggles):
    # the dense pass alone (n <= 3) and one extension pass (n = 4, 5)
    data, off = corpus("mixed")
    rc, keys, counts, rows, diag = O.oracle_run(data, off, n, 3000, 1.5, int(ALL))
    assert rc == 0
    r = run_with_env(toggles, lambda: ig.run_intergrams(
        ig.Corpus(data, off), ig.IntergramConfig(n=n, k=3000, z=1.5, mode=ALL)))
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)


def test_extend_pass_rank_bitmap_layout(gpu_lib):
    # extend_pass with > 4096 three-byte prefixes takes the rank-bitmap path;
    # the table must come back in the reference layout (candidate_id =
    # survivor ordinal * 256 + last byte, intergrams.hpp:56-66)
    data, off = corpus("c5")
    data, off = data[:int(off[2])], off[:3]
    allp, _ = O.oracle_naive(data, off, 3, int(ALL), 1 << 20)
    rng = np.random.default_rng(5)
    kept = np.array(sorted(rng.choice(allp, 6000, replace=False), key=lambda x: rng.random()),
                    np.uint64)
    pre = [ig.key_to_gram(int(x), 3) for x in kept]
    seqs = [bytes(data[int(off[i]):int(off[i + 1])]) for i in range(off.size - 1)]
    t, bp = ig.extend_pass(seqs, pre, 4, ALL)
    rc, t2, b2 = O.oracle_extend(data, off, kept, 3, 4, int(ALL))
    assert rc == 0 and np.array_equal(t, t2) and bp == b2
