"""Host-corpus entry points against the reference itself (oracle/_ref).

A host corpus reaches HBM three ways, and every one must give the reference's
list (proj/src/intergrams.cpp:68-166):
  * page-locked buffer: DMA batches on a copy stream (ig_session_run_host);
  * ordinary (pageable) contiguous buffer: host threads stream it through
    pinned slabs (ig_topk_ngrams -> run_host_streamed);
  * the reference's in-memory Corpus, one buffer per sequence: gathered in
    place, no packed copy (ig_topk_ngrams_seqs, the C++ run_intergrams).
The corpus spans several 32 MiB slabs and dense-pass batches, and holds empty
and short sequences at slab boundaries."""
import functools

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from paper_2511_14955_b200 import synth as S

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def corpus():
    data, off = S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=150, seq_len=300_000))
    seqs = [bytes(data[off[q]:off[q + 1]]) for q in range(off.size - 1)]
    # empty and short sequences, some around the 32 MiB slab boundary
    for at in (0, 7, 111, 112, 149):
        seqs.insert(at, b"")
    seqs.insert(60, b"abc")
    seqs.append(b"xy")
    lens = np.array([len(q) for q in seqs], np.uint64)
    off2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    flat = np.frombuffer(b"".join(seqs), np.uint8).copy()
    return seqs, flat, off2


@functools.lru_cache(maxsize=None)
def reference(n, k, mode):
    _, flat, off = corpus()
    rc, keys, counts, rows, diag, _, err = O.ref_run(flat, off, n, k, 1.5, mode, 0)
    assert rc == 0, err
    return keys, counts, [r["retained"] for r in rows]


@pytest.mark.parametrize("n,k,mode", [(5, 3000, 0), (6, 5000, 1), (3, 100, 1)])
@pytest.mark.parametrize("path", ["pageable", "seqs", "pinned", "pinned-session"])
def test_host_corpus_paths_equal_reference(gpu_lib, n, k, mode, path):
    import torch
    seqs, flat, off = corpus()
    keys, counts, retained = reference(n, k, mode)
    cfg = ig.IntergramConfig(n=n, k=k, z=1.5, mode=ig.CountMode(mode))
    if path == "pageable":
        r = ig.run_intergrams(ig.Corpus(flat, off), cfg)
    elif path == "seqs":
        r = ig.run_intergrams(seqs, cfg)
    else:
        pinned = torch.empty(flat.size, dtype=torch.uint8, pin_memory=True).numpy()
        pinned[:] = flat
        if path == "pinned":
            r = ig.run_intergrams(ig.Corpus(pinned, off), cfg)
        else:
            sess = ig.Session(device=0)
            r = sess.load_and_run(ig.Corpus(pinned, off), cfg)
            r2 = sess.run(cfg)  # resident afterwards
            sess.close()
            assert np.array_equal(r2.keys, keys) and np.array_equal(r2.counts, counts)
    assert np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    assert [p.retained for p in r.passes] == retained


def test_seqs_entry_point_edge_cases(gpu_lib):
    cfg = ig.IntergramConfig(n=4, k=10, z=1.5, mode=ig.CountMode.kAll)
    # no bytes: the dense pass keeps nothing and the 4-gram pass has a
    # depth-0 trie, a ConfigError on the reference too (intergrams.cpp:46-48)
    for empty in ([], [b"", b""]):
        rc = O.ref_run_grams(np.zeros(0, np.uint8), np.zeros(len(empty) + 1, np.uint64),
                             4, 10, 1.5, 1, 0)[0]
        assert rc == 2
        with pytest.raises(ig.ConfigError):
            ig.run_intergrams(empty, cfg)
    cfg3 = ig.IntergramConfig(n=3, k=10, z=1.5, mode=ig.CountMode.kAll)
    assert len(ig.run_intergrams([], cfg3).counts) == 0
    assert len(ig.run_intergrams([b"", b""], cfg3).counts) == 0
    r = ig.run_intergrams([b"abcdabcd", b"", b"cdab"], cfg)
    rc, keys, counts, _, _ = O.oracle_run(np.frombuffer(b"abcdabcdcdab", np.uint8),
                                          np.array([0, 8, 8, 12], np.uint64), 4, 10, 1.5, 1)
    assert rc == 0 and np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
