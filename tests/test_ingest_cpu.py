"""File enumeration of the library's corpus loader (ig_file_corpus_files,
csrc/ingest.cu) against the reference's own Corpus(CorpusSpec)
(proj/src/corpus.cpp:13-53, compiled in oracle/_ref): same files (count and
bytes) in recursive and flat modes, and the same error classes."""
import os

import pytest

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig
from tests import ingest_util as U

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference build unavailable")


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("recurse", [False, True])
def test_enumeration_matches_reference(tmp_path, seed, recurse):
    root = U.random_tree(str(tmp_path / "c"), seed)
    extra = os.path.join(root, "d0")
    for roots in ([root], [root, extra], [extra, root, os.path.join(extra, os.listdir(extra)[0])]):
        n, b = ig.CorpusSpec(roots, recurse=recurse).files()
        rc, data, off, nf, err = O.ref_corpus_files(roots, recurse=recurse)
        assert rc == 0, err
        assert (n, b) == (nf, int(off[-1]))   # whole-file records: bytes of all files


def test_missing_root_and_empty_spec(tmp_path):
    with pytest.raises(ig.ConfigError, match="does not exist"):
        ig.CorpusSpec([str(tmp_path / "nope")]).files()
    rc, *_ = O.ref_corpus_files([str(tmp_path / "nope")])
    assert rc == 2
    with pytest.raises(ig.ConfigError, match="no roots"):
        ig.CorpusSpec([]).files()
