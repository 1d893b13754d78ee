"""The `intergrams` CLI end to end on a B200: `count` / `bench` / `featurize`
over files on disk (corpus enumeration of src/corpus.cpp:40-152: file, line
and chunk records, lexicographic file order, recursion) against the C oracle,
and the SPEC.md:693 golden (`count --algorithm naive --n 3 --k 2` over
["aaaa", "aaab"] prints "616161\\t2\\n616162\\t1\\n")."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from tests import util

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2511_14955_b200", "_lib", "intergrams")


def run(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, env=e)


def write_corpus(d, seqs, mode="files"):
    """Lays seqs out on disk; returns (inputs, flags) that enumerate them in order."""
    d.mkdir(parents=True, exist_ok=True)
    if mode == "files":
        for i, s in enumerate(seqs):
            (d / f"s{i:05d}.bin").write_bytes(s)
        return [d], []
    if mode == "lines":
        (d / "corpus.txt").write_bytes(b"\n".join(seqs) + b"\n")
        return [d / "corpus.txt"], ["--line-mode"]
    raise ValueError(mode)


def test_spec_golden_naive(gpu_lib, tmp_path):
    (tmp_path / "a").write_bytes(b"aaaa")
    (tmp_path / "b").write_bytes(b"aaab")
    r = run("count", "--algorithm", "naive", "--n", "3", "--k", "2", tmp_path / "a", tmp_path / "b")
    assert r.returncode == 0, r.stderr
    assert r.stdout == "616161\t2\n616162\t1\n"


@pytest.mark.parametrize("mode", ["once", "all"])
@pytest.mark.parametrize("layout", ["files", "lines"])
def test_count_intergrams_matches_oracle(gpu_lib, tmp_path, mode, layout):
    rng = O.Mt64(808 if mode == "once" else 909)
    for t in range(3):
        seqs = [s.replace(b"\n", b"x") for s in O.random_corpus(rng, 30, 400, 5)]
        if layout == "lines":
            seqs = [s for s in seqs]  # empty lines are sequences too
        inputs, flags = write_corpus(tmp_path / f"{layout}{t}", seqs, layout)
        d, off = O.csr(seqs)
        for n, k, z in ((3, 20, 1.5), (5, 40, 1.5), (8, 10, 3.0)):
            r = run("count", *inputs, *flags, "-n", n, "-k", k, "-z", z, "--mode", mode)
            rc, keys, counts, rows, diag = O.oracle_run(d, off, n, k, z, 0 if mode == "once" else 1)
            if rc != 0:
                assert r.returncode == 2, r.stderr
                continue
            assert r.returncode == 0, r.stderr
            assert r.stdout == util.tsv(keys, counts, n)


def test_count_chunks_recursion_and_algorithms(gpu_lib, tmp_path):
    rng = O.Mt64(4242)
    blob = O.random_bytes(rng, 5000, 4)
    sub = tmp_path / "root" / "deeper"
    sub.mkdir(parents=True)
    (tmp_path / "root" / "b.bin").write_bytes(blob[:3000])
    (sub / "a.bin").write_bytes(blob[3000:])
    # recursion + chunk records: files sorted by path, then 700-byte records
    files = sorted([str(tmp_path / "root" / "b.bin"), str(sub / "a.bin")])
    seqs = []
    for f in files:
        data = open(f, "rb").read()
        seqs += [data[i:i + 700] for i in range(0, len(data), 700)]
    d, off = O.csr(seqs)
    base = ["-r", "--chunk-size", "700", tmp_path / "root"]
    r = run("count", *base, "-n", "6", "-k", "30", "--mode", "all")
    rc, keys, counts, _, _ = O.oracle_run(d, off, 6, 30, 1.5, 1)
    assert r.returncode == 0 and r.stdout == util.tsv(keys, counts, 6)
    r = run("count", *base, "-a", "naive", "-n", "7", "-k", "25", "--mode", "once")
    keys, counts = O.oracle_naive(d, off, 7, 0, 25)
    assert r.returncode == 0 and r.stdout == util.tsv(keys, counts, 7)
    r = run("count", *base, "-a", "hashgram", "-n", "5", "-k", "15", "-B", "4096", "--seed", "9")
    rc, keys, counts, kept, ex = O.oracle_hashgram(d, off, 5, 15, 0, 4096, 9)
    assert r.returncode == 0 and r.stdout == util.tsv(keys, counts, 5)
    # non-recursive: the nested file is skipped
    r = run("count", tmp_path / "root", "-a", "naive", "-n", "3", "-k", "5")
    d2, off2 = O.csr([blob[:3000]])
    keys, counts = O.oracle_naive(d2, off2, 3, 0, 5)
    assert r.stdout == util.tsv(keys, counts, 3)


def test_bench_reports(gpu_lib, tmp_path):
    rng = O.Mt64(5150)
    seqs = O.random_corpus(rng, 20, 2000, 4)
    inputs, _ = write_corpus(tmp_path / "c", seqs)
    out = tmp_path / "top.tsv"
    env = {"INTERGRAMS_WORKERS": "3"}
    r = run("bench", *inputs, "-n", "5", "-k", "50", "-o", out, env=env)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "step\truntime_s\tthroughput"
    labels = [ln.split("\t")[0] for ln in lines[1:]]
    assert labels == ["3-gram pass", "top-zk 3-grams/trie building", "4-gram pass",
                      "top-zk 4-grams/trie building", "5-gram pass", "top-k 5-grams", "total"]
    assert lines[1].split("\t")[2].endswith("MB/s") and lines[2].split("\t")[2] == "-"
    d, off = O.csr(seqs)
    rc, keys, counts, rows, _ = O.oracle_run(d, off, 5, 50, 1.5, 0)
    assert out.read_text() == util.tsv(keys, counts, 5)
    # JSON report, Jaccard against the result file itself
    rep = tmp_path / "rep.json"
    r = run("bench", *inputs, "-n", "5", "-k", "50", "--report", "json", "--report-file", rep,
            "--reference", out, env=env)
    assert r.returncode == 0, r.stderr
    j = json.loads(rep.read_text())
    assert j["schema_version"] == 1 and j["algorithm"] == "intergrams"
    assert j["config"] == ("algorithm=intergrams n=5 k=50 z=1.5 mode=once workers=3 "
                           "flush-batch=8 merge=flush")
    assert j["jaccard_vs_reference"] == 1.0
    got = [{k: s[k] for k in ("label", "gram_len", "bytes_processed", "candidate_space",
                              "retained", "retained_short")} for s in j["steps"]]
    assert got == rows
    assert abs(j["total_seconds"] - sum(s["seconds"] for s in j["steps"])) < 1e-9
    # hashgram rows
    r = run("bench", *inputs, "-a", "hashgram", "-n", "4", "-k", "9", "-B", "100", "--report",
            "json", env=env)
    j = json.loads(r.stdout)
    assert [s["label"] for s in j["steps"]] == ["hash pass", "top-k buckets", "exact pass",
                                                "top-k grams"]
    assert j["config"].startswith("algorithm=hashgram n=4 k=9 B=100 seed=0 mode=once workers=3")
    # naive has no pass rows
    r = run("bench", *inputs, "-a", "naive", "-n", "4", "-k", "9")
    assert r.stdout == "step\truntime_s\tthroughput\ntotal\t0.0000\t-\n"


def test_featurize_cli(gpu_lib, tmp_path):
    rng = O.Mt64(61)
    seqs = O.random_corpus(rng, 25, 300, 4)
    inputs, _ = write_corpus(tmp_path / "c", seqs)
    vocab = tmp_path / "vocab.tsv"
    r = run("count", *inputs, "-n", "4", "-k", "12", "-a", "naive", "-o", vocab)
    assert r.returncode == 0
    mat = tmp_path / "m.coo"
    r = run("featurize", *inputs, "--vocab", vocab, "--matrix-out", mat)
    assert r.returncode == 0, r.stderr
    grams = [bytes.fromhex(ln.split("\t")[0]) for ln in vocab.read_text().splitlines()]
    d, off = O.csr(seqs)
    want = O.oracle_featurize(d, off, np.array([int.from_bytes(g, "big") for g in grams],
                                               np.uint64), 4)
    assert mat.read_text() == "".join(f"{int(e) >> 32}\t{int(e) & 0xffffffff}\n" for e in want)
    assert (tmp_path / "m.coo.vocab").read_text() == "".join(g.hex() + "\n" for g in grams)
    assert r.stderr == f"rows={len(seqs)} cols={len(grams)} nnz={len(want)}\n"


def test_io_error_on_unwritable_output(gpu_lib, tmp_path):
    (tmp_path / "a").write_bytes(b"abcdefgh")
    r = run("count", tmp_path / "a", "-n", "3", "-k", "2", "-o", tmp_path / "no" / "such" / "f")
    assert r.returncode == 3 and r.stderr.startswith("io error: cannot open output file")
