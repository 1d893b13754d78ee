"""The seeded corpus generator (csrc/synth.c) reproduces BASELINE.json's shapes
and is deterministic: any subset of sequences regenerates byte-identically."""
import numpy as np

from paper_2511_14955_b200 import synth as S


def test_shapes():
    off = S.offsets(S.CONFIGS["c1"])
    assert off.size - 1 == 256 and int(off[-1]) == 64 << 20
    off = S.offsets(S.CONFIGS["c2"])
    assert off.size - 1 == 4096 and int(off[-1]) == 4 << 30
    off = S.offsets(S.CONFIGS["c3"])
    lens = np.diff(off)
    assert int(off[-1]) == 16 << 30
    assert lens[:-1].min() >= 256 and lens.max() <= 64 << 20
    assert 25000 < lens.size < 45000  # lognormal(12, 1.5): mean ~ e^13.125
    assert int(S.offsets(S.CONFIGS["c4"])[-1]) == 32 << 30
    assert int(S.offsets(S.CONFIGS["c5"])[-1]) == 64 << 30


def test_subset_determinism():
    cfg = S.scaled(S.CONFIGS["c2"], num_seqs=12, seq_len=5000)
    d, off = S.generate(cfg, threads=3)
    d2, off2 = S.generate(cfg, first=4, count=5, threads=1)
    assert np.array_equal(d2, d[off[4]:off[9]])
    d3, _ = S.generate(cfg, threads=8)
    assert np.array_equal(d, d3)


def test_value_distributions():
    d, off = S.generate(S.scaled(S.CONFIGS["c4"], num_seqs=3, seq_len=20000))
    assert set(np.unique(d).tolist()) <= {0x41, 0x43, 0x47, 0x54}
    d, off = S.generate(S.scaled(S.CONFIGS["c5"], num_seqs=2, seq_len=1 << 16))
    assert len(np.unique(d)) == 256
    d, off = S.generate(S.scaled(S.CONFIGS["c1"], num_seqs=2, seq_len=1 << 16))
    # Zipf tokens: heavy repetition of the hottest token
    _, counts = np.unique(d, return_counts=True)
    assert counts.max() > 3 * counts.mean()
