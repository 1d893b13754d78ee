"""§8(f) rows 3-4 without a GPU: the C oracle's hash-gramming and featurize
restatements (oracle/ig_oracle.c) against golden vectors produced by the
reference itself (tests/golden/golden_extra.json: run_hashgram,
hashgram.cpp:325-383; mix64, :22-59; featurize, metrics.cpp:83-132), and the
host-side / validation behaviour of the new C-ABI entry points."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import _native as N
from paper_2511_14955_b200 import intergrams as ig
from tests import util

GX = json.load(open(os.path.join(util.HERE, "golden", "golden_extra.json")))


def hg_id(c):
    return f"n{c['n']}-m{c['mode']}-B{c['buckets']}-k{c['k']}"


@pytest.mark.parametrize("case", GX["hashgram"], ids=[hg_id(c) for c in GX["hashgram"]])
def test_oracle_hashgram_matches_reference(case):
    data, off = util.corpus_from(case["corpus"])
    rc, keys, counts, kept, exact = O.oracle_hashgram(data, off, case["n"], case["k"],
                                                      case["mode"], case["buckets"],
                                                      case["seed"])
    assert rc == case["rc"] == 0
    assert util.tsv(keys, counts, case["n"]) == case["tsv"]
    assert kept == case["passes"][1]["retained"]
    assert exact == case["passes"][2]["retained"]


@pytest.mark.parametrize("case", GX["mix64"], ids=lambda c: f"{c['hex'][:8]}-{c['seed']}")
def test_mix64_oracle_and_library(case):
    b = bytes.fromhex(case["hex"])
    assert O.oracle_mix64(b, case["seed"]) == case["mix64"]
    assert ig.mix64(b, case["seed"]) == case["mix64"]  # host-only C-ABI entry


@pytest.mark.parametrize("case", GX["featurize"], ids=lambda c: f"n{c['n']}-v{len(c['vocab'])}")
def test_oracle_featurize_matches_reference(case):
    data, off = util.corpus_from(case["corpus"])
    vk = np.array([int(v, 16) if v else 0 for v in case["vocab"]], np.uint64)
    ent = O.oracle_featurize(data, off, vk, case["n"])
    assert ent.tolist() == case["entries"]


def _corpus():
    return ig.make_memory_corpus([b"abcdefgh", b"abc"])


@pytest.mark.parametrize("n,k,guard,msg", [(0, 1, 1 << 20, "gram length"),
                                           (3, 1, 5, "guard exceeded"),
                                           (9, 1, 1 << 20, "above 8"),
                                           (3, 0, 1 << 20, "top-k requires")])
def test_naive_validation_before_device(n, k, guard, msg):
    out = N.ig_result()
    err = C.create_string_buffer(256)
    rc = N.lib().ig_naive_topk(C.byref(_corpus()._view()), n, k, 0, guard, -1, C.byref(out), err,
                               256)
    assert rc == N.IG_ECONFIG and msg in err.value.decode()


@pytest.mark.parametrize("B,n,k,msg", [(0, 3, 1, "bucket count"), (8, 0, 1, "gram length"),
                                       (8, 3, 0, "k must"), (8, 9, 1, "above 8")])
def test_hashgram_validation_before_device(B, n, k, msg):
    p = N.ig_hashgram_params(buckets=B, n=n, k=k, mode=0, seed=0, flush_batch_size=8,
                             trie_second_pass=0, device=-1)
    out = N.ig_result()
    err = C.create_string_buffer(256)
    rc = N.lib().ig_hashgram_topk(C.byref(_corpus()._view()), C.byref(p), C.byref(out), err, 256)
    assert rc == N.IG_ECONFIG and msg in err.value.decode()


def test_featurize_validation_before_device():
    with pytest.raises(ValueError, match="share one length"):
        ig.featurize(_corpus(), [ig.GramCount(b"ab", 1), ig.GramCount(b"abc", 1)])
    with pytest.raises(ig.ConfigError, match="above 8"):
        ig.featurize(_corpus(), [ig.GramCount(b"abcdefghi", 1)])
