"""Randomised parity: hypothesis draws corpora (sequence counts and lengths,
alphabets, runs of repeated bytes, empty and short sequences) and configs (n,
k, z, mode); the GPU result must equal the C oracle bit for bit, including the
error class.  Seeds are derived by hypothesis, so failures shrink and replay."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig

pytestmark = pytest.mark.gpu


@st.composite
def corpora(draw):
    m = draw(st.integers(0, 24))
    alphabet = draw(st.sampled_from([1, 2, 3, 4, 7, 16, 256]))
    seed = draw(st.integers(0, 2**32 - 1))
    rng = np.random.default_rng(seed)
    seqs = []
    for _ in range(m):
        kind = draw(st.sampled_from(["rand", "run", "short", "empty", "long"]))
        if kind == "empty":
            seqs.append(b"")
        elif kind == "short":
            seqs.append(bytes(rng.integers(0, alphabet, draw(st.integers(1, 9)), dtype=np.uint8)))
        elif kind == "run":
            b = int(rng.integers(0, 256))
            seqs.append(bytes([b]) * draw(st.integers(1, 300)))
        elif kind == "long":
            seqs.append(bytes(rng.integers(0, alphabet, draw(st.integers(600, 5000)), dtype=np.uint8)))
        else:
            seqs.append(bytes(rng.integers(0, alphabet, draw(st.integers(0, 400)), dtype=np.uint8)))
    return seqs


@settings(max_examples=400, deadline=None, suppress_health_check=list(HealthCheck))
@given(seqs=corpora(), n=st.integers(1, 8), k=st.integers(1, 60),
       z=st.sampled_from([1.0, 1.5, 2.0, 7.5]), mode=st.sampled_from([0, 1]))
def test_fuzz_gpu_equals_oracle(gpu_lib, seqs, n, k, z, mode):
    d, off = O.csr(seqs)
    rc, keys, counts, rows, diag = O.oracle_run(d, off, n, k, z, mode)
    cfg = ig.IntergramConfig(n=n, k=k, z=z, mode=ig.CountMode(mode))
    if rc != 0:
        with pytest.raises(ig.ConfigError):
            ig.run_intergrams(seqs, cfg)
        return
    r = ig.run_intergrams(seqs, cfg)
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    assert r.diagnostics == diag
    assert [(p.label, p.retained, p.retained_short, p.candidate_space) for p in r.passes] == \
           [(q["label"], q["retained"], q["retained_short"], q["candidate_space"]) for q in rows]
