"""BASELINE config shapes on the GPU.  Reduced-size samples of every config are
compared with the C oracle bit for bit; at full size (c1 entirely; c2 at 4 GiB)
the run is checked through size-independent properties: canonical order,
count bounds (count-once <= m; extension counts <= prefix counts), prefix
consistency with the previous pass, and determinism across runs."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from paper_2511_14955_b200 import synth as S

pytestmark = pytest.mark.gpu


def run_both(cfg, n, k, mode, z=1.5):
    data, off = S.generate(cfg)
    r = ig.run_intergrams(ig.Corpus(data, off), ig.IntergramConfig(n=n, k=k, z=z,
                                                                   mode=ig.CountMode(mode)))
    rc, keys, counts, rows, diag = O.oracle_run(data, off, n, k, z, mode)
    assert rc == 0
    return r, keys, counts, diag


@pytest.mark.parametrize("name,extra", [
    ("c1", {}),  # full size: 256 x 256 KiB
    ("c2", {"num_seqs": 96}),
    ("c3", {"total": 96 << 20}),
    ("c4", {"num_seqs": 24}),
    ("c5", {"num_seqs": 64}),
])
def test_config_sample_equals_oracle(gpu_lib, name, extra):
    base = S.CONFIGS[name]
    cfg = S.scaled(base, **extra)
    k = base.k if name in ("c1", "c2") else min(base.k, 2000)
    r, keys, counts, diag = run_both(cfg, base.n, k, base.mode)
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    assert r.diagnostics == diag


def check_canonical(r):
    c = r.counts.astype(np.int64)
    k = r.keys
    assert (np.diff(c) <= 0).all()
    same = np.diff(c) == 0
    assert (k[1:][same] > k[:-1][same]).all()


@pytest.mark.slow
def test_c2_full_size_properties(gpu_lib):
    cfg = S.CONFIGS["c2"]
    data, off = S.generate(cfg)
    corpus = ig.Corpus(data, off)
    sess = ig.Session(device=0)
    sess.load(corpus)
    c6 = ig.IntergramConfig(n=6, k=10000, z=1.5, mode=ig.CountMode.kOnce)
    r1 = sess.run(c6)
    r2 = sess.run(c6)
    assert r1.topk == r2.topk  # determinism
    assert len(r1.topk) == 10000
    check_canonical(r1)
    assert int(r1.counts.max()) <= cfg.num_seqs  # count-once bound
    # prefix consistency: every 6-gram's 5-prefix is a 5-gram survivor, and its
    # count never exceeds the prefix count (test_intergrams.cpp:163-208)
    r5 = sess.run(ig.IntergramConfig(n=5, k=15000, z=1.5, mode=ig.CountMode.kOnce))
    pc = {g.gram: g.count for g in r5.topk}
    for g in r1.topk:
        assert g.gram[:5] in pc and g.count <= pc[g.gram[:5]]
    passes = [p for p in r1.passes if p.bytes_processed]
    assert len(passes) == 4 and all(p.bytes_processed == 4 << 30 for p in passes)
    sess.close()


@pytest.mark.slow
def test_more_than_2_32_routed_positions_doubling(gpu_lib):
    # A count-once corpus of two identical halves has every count exactly
    # doubled and the same list: a size-independent check past 2^32 routed
    # positions (the route offsets and scans must be 64-bit).
    cfg = S.scaled(S.CONFIGS["c2"], num_seqs=2200)
    data, off = S.generate(cfg)
    half = ig.Corpus(data, off)
    off2 = np.concatenate([off, off[1:] + off[-1]]).astype(np.uint64)
    doubled = ig.Corpus(np.concatenate([data, data]), off2)
    assert int(off2[-1]) > (1 << 32)
    icfg = ig.IntergramConfig(n=6, k=3000, z=1.5, mode=ig.CountMode.kOnce)
    sess = ig.Session(device=0)
    sess.load(half)
    r1 = sess.run(icfg)
    sess.load(doubled)
    r2 = sess.run(icfg)
    assert [g.gram for g in r2.topk] == [g.gram for g in r1.topk]
    assert [g.count for g in r2.topk] == [2 * g.count for g in r1.topk]
    sess.close()


@pytest.mark.slow
def test_count_all_past_2_32_positions_doubling(gpu_lib):
    # Count-all over two identical halves totalling > 2^32 bytes: u64 tables,
    # several < 4 GiB count launches per pass, hit masks across launch
    # boundaries, the rank bitmap.  Every count doubles and the list stays.
    cfg = S.scaled(S.CONFIGS["c5"], num_seqs=2100)
    data, off = S.generate(cfg)
    half = ig.Corpus(data, off)
    off2 = np.concatenate([off, off[1:] + off[-1]]).astype(np.uint64)
    doubled = ig.Corpus(np.concatenate([data, data]), off2)
    assert int(off2[-1]) > (1 << 32)
    icfg = ig.IntergramConfig(n=8, k=20000, z=1.5, mode=ig.CountMode.kAll)
    sess = ig.Session(device=0)
    sess.load(half)
    r1 = sess.run(icfg, materialize=False)
    sess.load(doubled)
    r2 = sess.run(icfg, materialize=False)
    sess.close()
    assert np.array_equal(r2.keys, r1.keys)
    assert np.array_equal(r2.counts, 2 * r1.counts)


@pytest.mark.parametrize("name,extra,k", [("c2", {"num_seqs": 600, "seq_len": 1 << 20}, 1000),
                                          ("c1", {}, 1024),
                                          ("c3", {"total": 700 << 20}, 2000),
                                          ("c4", {"num_seqs": 48}, 65536)])
def test_pipelined_host_load_equals_resident(gpu_lib, name, extra, k):
    # ig_session_run_host (batched H2D under the dense pass) == load + run.
    # c4 (4 bytes): the resident run counts its dense pass with the
    # small-alphabet kernel, the pipelined one routes it
    base = S.CONFIGS[name]
    cfg = S.scaled(base, **extra)
    data, off = S.generate(cfg)
    corpus = ig.Corpus(data, off)
    icfg = ig.IntergramConfig(n=base.n, k=k, z=1.5, mode=ig.CountMode(base.mode))
    s1 = ig.Session(device=0)
    r1 = s1.load_and_run(corpus, icfg)
    r1b = s1.run(icfg)  # resident afterwards
    s1.close()
    s2 = ig.Session(device=0)
    s2.load(corpus)
    r2 = s2.run(icfg)
    s2.close()
    assert r1.topk == r2.topk == r1b.topk
    assert [p.bytes_processed for p in r1.passes] == [p.bytes_processed for p in r2.passes]


@pytest.mark.parametrize("name,extra,k", [
    ("c1", {}, None),                       # full size, the reference's own k
    ("c2", {"num_seqs": 192}, None),        # 192 MiB, k = 10000
    ("c3", {"total": 192 << 20}, 20000),
    ("c4", {"num_seqs": 48}, None),         # 192 MiB, k = 65536
    ("c5", {"num_seqs": 128}, 100000),
    pytest.param("c2", {"num_seqs": 1024}, None, marks=pytest.mark.slow),   # 1 GiB
    pytest.param("c3", {"total": 1 << 30}, None, marks=pytest.mark.slow),   # k = 100000
    pytest.param("c4", {"num_seqs": 256}, None, marks=pytest.mark.slow),    # 1 GiB
    pytest.param("c5", {"num_seqs": 1024}, None, marks=pytest.mark.slow),   # k = 1000000
])
def test_config_sample_equals_reference(gpu_lib, name, extra, k):
    """The reference itself (oracle/_ref: proj/src compiled unmodified, all host
    threads) on the same seeded sample: identical list, counts, order, pass rows
    and diagnostics."""
    if not O.ref_available():
        pytest.skip("reference build unavailable")
    base = S.CONFIGS[name]
    cfg = S.scaled(base, **extra)
    k = k or base.k
    data, off = S.generate(cfg)
    r = ig.run_intergrams(ig.Corpus(data, off), ig.IntergramConfig(
        n=base.n, k=k, z=base.z, mode=ig.CountMode(base.mode)))
    rc, keys, counts, rows, diag, secs, err = O.ref_run(data, off, base.n, k, base.z, base.mode, 0)
    assert rc == 0, err
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    assert r.diagnostics == diag
    got_rows = [{"label": p.label, "gram_len": p.gram_len, "bytes_processed": p.bytes_processed,
                 "candidate_space": p.candidate_space, "retained": p.retained,
                 "retained_short": p.retained_short} for p in r.passes]
    assert got_rows == [{kk: x[kk] for kk in got_rows[0]} for x in rows]
