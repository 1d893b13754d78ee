"""GPU parity against the golden vectors produced by the reference itself
(tests/golden/golden.json): every case through the C-ABI run_intergrams, and
the dense tables through ig_count_dense.  Bit-exact lists, counts, order, pass
rows, diagnostics and error classes."""
import hashlib

import pytest

from paper_2511_14955_b200 import intergrams as ig
from tests import util

pytestmark = pytest.mark.gpu
G = util.golden()


@pytest.mark.parametrize("case", G["cases"], ids=[util.case_id(c) for c in G["cases"]])
def test_gpu_matches_reference_golden(gpu_lib, case):
    data, off = util.corpus_from(case["corpus"])
    cfg = ig.IntergramConfig(n=case["n"], k=case["k"], z=case["z"],
                             mode=ig.CountMode(case["mode"]))
    corpus = ig.Corpus(data, off)
    if case["rc"] == 2:
        with pytest.raises(ig.ConfigError):
            ig.run_intergrams(corpus, cfg)
        return
    r = ig.run_intergrams(corpus, cfg)
    assert ig.topk_to_tsv(r.topk) == case["tsv"]
    assert [{"label": p.label, "gram_len": p.gram_len, "bytes_processed": p.bytes_processed,
             "candidate_space": p.candidate_space, "retained": p.retained,
             "retained_short": p.retained_short} for p in r.passes] == case["passes"]
    assert r.diagnostics == case["diagnostics"]


@pytest.mark.parametrize("t", G["dense_tables"], ids=lambda t: f"n{t['n']}-m{t['mode']}")
def test_gpu_dense_table_digest(gpu_lib, t):
    data, off = util.corpus_from(t["corpus"])
    tab = ig.count_dense(ig.Corpus(data, off), t["n"], ig.CountMode(t["mode"]))
    assert hashlib.sha256(tab.astype("<u8").tobytes()).hexdigest() == t["sha256"]
