"""The C oracle restatement (oracle/ig_oracle.c) against golden vectors produced
by the reference itself (tests/golden/golden.json, see make_golden.py).  This is
what pins the oracle: same list, same counts, same order, same pass rows and
diagnostics, same error behaviour."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from tests import util

G = util.golden()


@pytest.mark.parametrize("case", G["cases"], ids=[util.case_id(c) for c in G["cases"]])
def test_oracle_matches_reference_golden(case):
    data, off = util.corpus_from(case["corpus"])
    rc, keys, counts, rows, diag = O.oracle_run(data, off, case["n"], case["k"], case["z"],
                                                case["mode"])
    assert rc == case["rc"]
    if rc != 0:
        return
    assert util.tsv(keys, counts, case["n"]) == case["tsv"]
    assert rows == case["passes"]
    assert diag == case["diagnostics"]


@pytest.mark.parametrize("t", G["dense_tables"], ids=lambda t: f"n{t['n']}-m{t['mode']}")
def test_oracle_dense_table_digest(t):
    data, off = util.corpus_from(t["corpus"])
    tab = O.oracle_count_dense(data, off, t["n"], t["mode"])
    assert hashlib.sha256(tab.astype("<u8").tobytes()).hexdigest() == t["sha256"]
    assert int(tab.sum()) == t["total"]
