"""Run with IG_ONCE_EXACT_MIN_K=1 (every count-once extension pass through the
sort fallback): the golden count-once cases and random corpora against the
oracle.  Exit status 0 = all equal.  Driven by tests/test_gpu_once_exact.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2511_14955_b200 import intergrams as ig  # noqa: E402
from tests import util  # noqa: E402

assert os.environ.get("IG_ONCE_EXACT_MIN_K") == "1"
bad = 0
n_cases = 0
for c in util.golden()["cases"]:
    if c["mode"] != 0 or c["rc"] != 0:
        continue
    data, off = util.corpus_from(c["corpus"])
    r = ig.run_intergrams(ig.Corpus(data, off), ig.IntergramConfig(n=c["n"], k=c["k"], z=c["z"]))
    n_cases += 1
    if ig.topk_to_tsv(r.topk) != c["tsv"]:
        bad += 1
        print("golden mismatch", util.case_id(c))
rng = O.Mt64(2718)
for t in range(12):
    seqs = O.random_corpus(rng, 30, 5000, 4 + t % 3)
    d, off = O.csr(seqs)
    for n, k in ((4, 30), (6, 100), (8, 500)):
        r = ig.run_intergrams(seqs, ig.IntergramConfig(n=n, k=k, z=1.5))
        rc, keys, counts, rows, diag = O.oracle_run(d, off, n, k, 1.5, 0)
        n_cases += 1
        if rc != 0 or ig.topk_to_tsv(r.topk) != util.tsv(keys, counts, n):
            bad += 1
            print("random mismatch", t, n, k)
print(f"{n_cases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
