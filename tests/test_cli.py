"""The `intergrams` CLI (paper_2511_14955_b200/tools/cli.cpp, built into
paper_2511_14955_b200/_lib/intergrams) against the reference's CLI surface
(proj/src/cli.cpp): flag parsing, exit codes 0/2/3/4 (:423-440), the host-only
`compare` subcommand (:382-396) and the RunReport TSV/JSON rendering
(metrics.cpp:134-200, pinned by golden strings the reference printed).  The
GPU-backed subcommands are exercised in tests/test_gpu_cli.py."""
import json
import os
import subprocess

import pytest

from tests import util

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2511_14955_b200", "_lib")
CLI = os.path.join(LIBDIR, "intergrams")
GX = json.load(open(os.path.join(util.HERE, "golden", "golden_extra.json")))


def run(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([CLI, *args], capture_output=True, text=True, env=e)


@pytest.fixture(scope="module")
def report_fmt(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cli") / "report_fmt")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "report_fmt.cpp"), "-L", LIBDIR,
                    "-lintergrams_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


@pytest.mark.parametrize("i", range(len(GX["reports"])))
def test_run_report_matches_reference(report_fmt, i):
    rep = GX["reports"][i]
    lines = "".join(
        f"{r['label']}\t{r['gram_len']}\t{r['seconds']}\t{r['bytes_processed']}\t"
        f"{r['candidate_space']}\t{r['retained']}\t{int(r['retained_short'])}\n"
        for r in rep["rows"])
    args = [report_fmt, rep["algorithm"], rep["echo"], "1" if rep["json"] else "0"]
    if rep["jaccard"] is not None:
        args.append(rep["jaccard"])
    r = subprocess.run(args, input=lines, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout == rep["text"]


def test_help_and_usage_errors():
    assert run("--help").returncode == 0
    r = run("count", "--help")
    assert r.returncode == 0 and "--oversample" in r.stdout
    assert run().returncode == 2                                   # require_subcommand(1)
    assert run("frobnicate").returncode == 2
    assert run("count").returncode == 2                            # inputs required
    assert run("count", "--bogus", "x").returncode == 2
    assert run("count", "--mode", "sometimes", "x").returncode == 2   # IsMember
    assert run("count", "-a", "fast", "x").returncode == 2
    assert run("count", "-n", "three", "x").returncode == 2
    assert run("count", "-n", "-3", "x").returncode == 2
    assert run("count", "-k").returncode == 2
    assert run("bench", "--report", "xml", "x").returncode == 2
    assert run("featurize", "x").returncode == 2                   # --vocab/--matrix-out required
    assert run("compare", "a").returncode == 2                     # expected(2)
    r = run("theory", "--a", "1.1")
    assert r.returncode == 2 and "configuration error" in r.stderr


def test_config_errors_before_the_device(tmp_path):
    f = tmp_path / "a.txt"
    f.write_bytes(b"abcdef")
    r = run("count", str(tmp_path / "missing"))
    assert r.returncode == 2 and "corpus root does not exist" in r.stderr
    for args in (["-n", "0"], ["-k", "0"], ["-z", "0.5"], ["--flush-batch", "0"]):
        r = run("count", *args, str(f))
        assert r.returncode == 2 and r.stderr.startswith("configuration error:"), (args, r.stderr)
    r = run("count", "-a", "hashgram", "-B", "0", str(f))
    assert r.returncode == 2 and "bucket count" in r.stderr
    r = run("count", "-a", "naive", "-n", "0", str(f))
    assert r.returncode == 2


def test_compare_is_jaccard(tmp_path):
    a = tmp_path / "a.tsv"
    b = tmp_path / "b.tsv"
    a.write_text("616161\t5\n626262\t3\n636363\t1\n")
    b.write_text("626262\t9\n636363\t1\n646464\t1\n656565\t1\n")
    r = run("compare", str(a), str(b))
    assert r.returncode == 0 and r.stdout == "0.400000\n"
    e = tmp_path / "empty.tsv"
    e.write_text("")
    assert run("compare", str(e), str(e)).stdout == "1.000000\n"
    r = run("compare", str(a), str(tmp_path / "nope.tsv"))
    assert r.returncode == 3 and r.stderr.startswith("io error: cannot open result file")
    bad = tmp_path / "bad.tsv"
    bad.write_text("zz\t1\n")
    assert run("compare", str(a), str(bad)).returncode == 2       # from_hex ConfigError


def test_featurize_io_errors_before_the_device(tmp_path):
    f = tmp_path / "a.txt"
    f.write_bytes(b"abcdef")
    r = run("featurize", str(f), "--vocab", str(tmp_path / "nope"), "--matrix-out",
            str(tmp_path / "m"))
    assert r.returncode == 3 and "cannot open vocab file" in r.stderr
