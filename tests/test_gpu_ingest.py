"""Corpus ingestion straight into HBM (csrc/ingest.cu) on a
B200: the resident corpus a file spec produces equals the reference's own
Corpus(CorpusSpec) materialisation (proj/src/corpus.cpp:13-152, oracle/_ref)
byte for byte and offset for offset, in whole-file, line and chunk modes, with
and without recursion; multi-slab files exercise the pinned-slab pipeline;
run_intergrams over a file spec equals the in-memory run."""
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from tests import ingest_util as U

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sess(gpu_lib):
    s = ig.Session(device=0)
    yield s
    s.close()


MODES = [dict(), dict(line_mode=True), dict(chunk_size=1), dict(chunk_size=7),
         dict(chunk_size=4096), dict(line_mode=True, chunk_size=5)]


@pytest.mark.parametrize("seed", [11, 12, 13])
@pytest.mark.parametrize("recurse", [False, True])
@pytest.mark.parametrize("mode", range(len(MODES)))
def test_resident_corpus_equals_reference(sess, tmp_path, seed, recurse, mode):
    root = U.random_tree(str(tmp_path / "c"), seed, newline_rate=0.02 + 0.05 * (seed % 2))
    kw = MODES[mode]
    spec = ig.CorpusSpec([root], recurse=recurse, **kw)
    sess.load_files(spec)
    data, off = sess.corpus()
    rc, rdata, roff, nf, err = O.ref_corpus_files([root], recurse=recurse, **kw)
    assert rc == 0, err
    assert np.array_equal(off, roff)
    assert data.tobytes() == rdata.tobytes()


def test_empty_and_newline_only_files(sess, tmp_path):
    d = tmp_path / "e"
    d.mkdir()
    (d / "a").write_bytes(b"")
    (d / "b").write_bytes(b"\n\n\n")
    (d / "c").write_bytes(b"x\n\ny")
    for kw in (dict(), dict(line_mode=True), dict(chunk_size=2)):
        sess.load_files(ig.CorpusSpec([str(d)], **kw))
        data, off = sess.corpus()
        rc, rdata, roff, nf, err = O.ref_corpus_files([str(d)], **kw)
        assert np.array_equal(off, roff) and data.tobytes() == rdata.tobytes(), kw


def test_multi_slab_files(sess, tmp_path):
    # > 8 slabs of 32 MiB: slabs are reused, files straddle slab boundaries
    rng = np.random.default_rng(5)
    d = tmp_path / "big"
    d.mkdir()
    parts = []
    for i, n in enumerate((100 << 20, 1, 0, 170 << 20, 33 << 20)):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        b[rng.integers(0, max(n, 1), n // 500)] = 10 if n else 0
        (d / f"p{i}").write_bytes(b.tobytes())
        parts.append(b.tobytes())
    whole = b"".join(parts)
    sess.load_files(ig.CorpusSpec([str(d)]))
    data, off = sess.corpus()
    assert hashlib.sha256(data.tobytes()).digest() == hashlib.sha256(whole).digest()
    assert off.tolist() == np.cumsum([0] + [len(p) for p in parts]).tolist()
    sess.load_files(ig.CorpusSpec([str(d)], line_mode=True))
    data, off = sess.corpus()
    lines = [ln for p in parts for ln in (p.split(b"\n")[:-1] + ([p.split(b"\n")[-1]] if p.split(b"\n")[-1] else []))]
    assert int(off[-1]) == sum(len(x) for x in lines) and off.size == len(lines) + 1
    assert hashlib.sha256(data.tobytes()).digest() == hashlib.sha256(b"".join(lines)).digest()


@pytest.mark.parametrize("mode", [ig.CountMode.kOnce, ig.CountMode.kAll])
def test_run_over_files_equals_in_memory(gpu_lib, tmp_path, mode):
    root = U.random_tree(str(tmp_path / "r"), 77, nfiles=30, newline_rate=0.01)
    for kw in (dict(recurse=True), dict(recurse=True, line_mode=True)):
        rc, rdata, roff, nf, err = O.ref_corpus_files([root], **kw)
        for n, k, z in ((3, 20, 1.5), (6, 50, 2.0)):
            cfg = ig.IntergramConfig(n=n, k=k, z=z, mode=mode)
            a = ig.run_intergrams(ig.CorpusSpec([root], **kw), cfg)
            b = ig.run_intergrams(ig.Corpus(rdata, roff), cfg)
            assert [tuple(g) for g in a.topk] == [tuple(g) for g in b.topk]
            assert [p.retained for p in a.passes] == [p.retained for p in b.passes]


def test_missing_root_is_config_error(gpu_lib, tmp_path):
    with pytest.raises(ig.ConfigError):
        ig.run_intergrams(ig.CorpusSpec([str(tmp_path / "missing")]), ig.IntergramConfig(n=3, k=1))


@pytest.mark.parametrize("mode", [ig.CountMode.kOnce, ig.CountMode.kAll])
def test_pipelined_run_files_multi_slab(sess, tmp_path, mode):
    # run_files overlaps the dense pass with the readers: batches of >= 256 MiB
    from paper_2511_14955_b200 import synth as S
    data, off = S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=700), 0, -1)
    d = tmp_path / "p"
    d.mkdir()
    per = (len(data) // 5) // (1 << 20) * (1 << 20)
    cuts = [0, per, 2 * per, 3 * per, 4 * per, len(data)]
    for i in range(5):
        (d / f"x{i}").write_bytes(data[cuts[i]:cuts[i + 1]].tobytes())
    cfg = ig.IntergramConfig(n=5, k=500, z=1.5, mode=mode)
    a = sess.run_files(ig.CorpusSpec([str(d)], chunk_size=1 << 20), cfg, materialize=False)
    b = ig.run_intergrams(ig.Corpus(data, np.ascontiguousarray(off, np.uint64)), cfg)
    assert np.array_equal(a.keys, b.keys) and np.array_equal(a.counts, b.counts)
