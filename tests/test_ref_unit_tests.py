"""The reference's own unit tests, compiled UNMODIFIED against the drop-in.

tests/cpp/Makefile builds /root/reference/proj/tests/test_{intergrams,
dense_pass,counting,trie,corpus,oracle,hashgram}.cpp + test_main.cpp with the
doctest-compatible shim (tests/cpp/doctest_shim/doctest.h) against
include/intergrams/*.hpp and links libintergrams_b200.so
(-> tests/cpp/_build/reftests, built by __graft_entry__.build() where the
reference exists; the GPU box runs the prebuilt binary).

Excluded, because the reference itself cannot pass them:
  * test_trie.cpp "lookup agrees with a set reference on random probes"
    never terminates: with alphabet 3 and depth 1 only 3 distinct probes
    exist, and the case loops until it has drawn 200 (test_trie.cpp:96-101).
  * test_hashgram.cpp "collision-free configurations equal the oracle
    exactly" (B = 2^40): the reference throws std::bad_alloc allocating
    CountTable(2^40) (hashgram.cpp:337), and its algorithm keeps the top-k
    BUCKETS with count ties broken by bucket id (hashgram.cpp:73-101), not by
    gram bytes, so on all 10 seeded corpora its list differs from
    naive_topk (test_ref_hashgram_case_fails_on_reference below runs both
    facts).  The GPU path instead equals the reference algorithm there
    (tests/test_gpu_exact.py::test_hashgram_large_b_equals_oracle).
test_theory.cpp is out of scope.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "reftests")
NONTERMINATING = "lookup agrees with a set reference on random probes"
REF_FAILS = "collision-free configurations equal the oracle exactly"
EXCLUDED = [NONTERMINATING, REF_FAILS]

# Cases that touch no device entry point (host classes and corpus
# enumeration of the drop-in): they run in the CPU suite too.
HOST_CASES = [
    "candidate_id arithmetic", "extend_pass requires a trie of depth j-1",
    "invalid configs are rejected", "dense capacity and gram mapping",
    "mark is idempotent", "fresh bitset is empty", "boundary ids",
    "flush_batch adds per-bitset contributions", "flush_batch on an empty batch is the identity",
    "flush_batch equals the scalar one-bit-at-a-time reference",
    "flush_batch equals sequential single flushes in any order",
    "flush_batch rejects capacity mismatch", "increment_all",
    "top_k breaks count ties by gram bytes ascending", "top_k of an all-zero table is empty",
    "top_k equals the full-sort reference", "top_k is a function of the (gram, count) multiset",
    "membership on a small byte trie", "single prefix", "empty trie answers absent for any probe",
    "mixed prefix lengths are rejected", "duplicate prefixes are rejected",
    "wrong window length is a logic error", "ordinals are a bijection with rank order",
    "frequency-ordered layout never changes lookup results",
    "node count stays linear in the number of prefixes",
    "in-memory corpus enumerates in order", "empty directory yields an empty stream",
    "files enumerate lexicographically by path", "missing root is a configuration error",
    "corpus stats", "line mode splits on newlines",
    "line mode: trailing newline adds no empty record",
    "chunk mode splits files into fixed-size records",
    "re-iteration yields byte-identical streams", "recursive enumeration is opt-in",
    "naive_topk", "corpus size guard", "hashing is deterministic for a fixed seed",
    "a single bucket absorbs everything",
    "bucket distribution passes a chi-square uniformity test",
    "large bucket spaces use the sorted-membership path",
]


def binary():
    if os.path.isdir("/root/reference/proj/tests"):  # build where the sources are
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/_build/reftests is missing (built by __graft_entry__.build())")
    return BIN


def listed():
    out = subprocess.run([binary(), "-ltc"], check=True, capture_output=True, text=True).stdout
    return [ln.split("\t", 1)[1] for ln in out.splitlines() if "\t" in ln]


def test_reference_test_inventory():
    names = listed()
    assert len(names) == 73 and len(set(names)) == 73
    assert set(HOST_CASES) <= set(names) and set(EXCLUDED) <= set(names)


@pytest.mark.parametrize("name", HOST_CASES)
def test_reference_host_case(name):
    r = subprocess.run([binary(), f"-tce={name}"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 1 passed | 0 failed" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_reference_unit_tests_on_gpu(gpu_lib):
    r = subprocess.run([binary()] + [f"-ntc={x}" for x in EXCLUDED], capture_output=True,
                       text=True, timeout=1200)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "reftests.txt"), "w") as f:
        f.write(out)
    assert r.returncode == 0, out[-4000:]
    assert "test cases: 71 | 71 passed | 0 failed" in out, out[-4000:]


def hashgram_case_corpora():
    """The 10 corpora of test_hashgram.cpp:86-101 (mt19937_64(1234),
    random_corpus(rng, 10, 100, 4))."""
    from oracle import oracle as O
    rng = O.Mt64(1234)
    return [O.csr(O.random_corpus(rng, 10, 100, 4)) for _ in range(10)]


def test_ref_hashgram_case_fails_on_reference():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    data, off = hashgram_case_corpora()[0]
    rc, _, _, _, err = O.ref_hashgram(data, off, 4, 8, 0, 1 << 40, 7)
    assert rc != 0 and "bad_alloc" in err
    differs = 0
    for data, off in hashgram_case_corpora():
        rc, k1, c1, _, _ = O.oracle_hashgram(data, off, 4, 8, 0, 1 << 40, 7)
        k2, c2 = O.oracle_naive(data, off, 4, 0, 8)
        assert rc == 0 and list(c1) == list(c2)  # same counts, other tied grams
        differs += list(k1) != list(k2)
    assert differs == 10
