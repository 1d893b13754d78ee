"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/intergrams_b200.h declares, validates configurations like
IntergramConfig::validate (intergrams.cpp:37-42) before touching a device, and
computes byte-balanced whole-sequence shards on the host."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2511_14955_b200 import _native as N
from paper_2511_14955_b200 import intergrams as ig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "intergrams_b200.h")).read()
    return re.findall(r"IG_API\s+[\w\s\*]+?\b(ig_\w+)\s*\(", src)


def test_header_and_binding_agree():
    decl = set(declared_symbols())
    bound = {name for name, _, _ in N.SYMBOLS}
    assert decl and decl == bound


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    nm = os.popen(f"nm -D --defined-only {N.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (ig_\w+)", nm))
    assert set(declared_symbols()) <= exported


def test_version():
    assert b"sm_100a" in N.lib().ig_version()


@pytest.mark.parametrize("n,k,z,msg", [(0, 1, 1.0, "gram length"), (4, 0, 1.0, "k must"),
                                       (4, 1, 0.5, "oversample"), (4, 1, float("nan"), "oversample")])
def test_invalid_config_rejected_before_device(n, k, z, msg):
    corpus = ig.make_memory_corpus([b"abcdefgh"])
    params = N.ig_params(n=n, k=k, z=z, mode=0, flush_batch_size=8, device=-1)
    out = N.ig_result()
    err = C.create_string_buffer(256)
    rc = N.lib().ig_topk_ngrams(C.byref(corpus._view()), C.byref(params), C.byref(out), err, 256)
    assert rc == N.IG_ECONFIG and msg in err.value.decode()


def test_python_mirror_validate():
    with pytest.raises(ig.ConfigError):
        ig.IntergramConfig(n=0).validate()
    with pytest.raises(ig.ConfigError):
        ig.IntergramConfig(k=0).validate()
    with pytest.raises(ig.ConfigError):
        ig.IntergramConfig(z=0.5).validate()
    assert ig.IntergramConfig(k=10000, z=1.5).k_prime() == 15000  # intergrams.hpp:29-31


def brute_shards(off, world):
    total = int(off[-1])
    cuts = [0]
    for r in range(1, world):
        t = total * r // world
        i = int(np.searchsorted(off, t, side="left"))
        i = min(i, off.size - 1)
        if i > 0 and (int(off[i]) - t) > (t - int(off[i - 1])):
            i -= 1
        cuts.append(i)
    cuts.append(off.size - 1)
    return [(cuts[r], max(cuts[r], cuts[r + 1])) for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_partitions_whole_sequences(world):
    rng = np.random.default_rng(world)
    lens = rng.integers(0, 5000, size=777)
    off = np.zeros(lens.size + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    got = [ig.shard_range(off, r, world) for r in range(world)]
    assert got == brute_shards(off, world)
    assert got[0][0] == 0 and got[-1][1] == lens.size
    for (a, b), (c, d) in zip(got, got[1:]):
        assert b == c  # contiguous, disjoint, complete
    total = int(off[-1])
    for a, b in got:  # byte balance within one sequence of the ideal cut
        assert abs(int(off[b] - off[a]) - total / world) <= 2 * lens.max() + 1


@pytest.mark.parametrize("n", [9, 16, 64])
def test_long_grams_pass_validation(n):
    # the reference takes any n (intergrams.cpp:37-42): no ConfigError (on a
    # box without a GPU the call then fails at the device, not in validation)
    corpus = ig.make_memory_corpus([b"abcdefghijklmnop"])
    params = N.ig_params(n=n, k=3, z=1.5, mode=0, flush_batch_size=8, device=-1)
    out = N.ig_result()
    err = C.create_string_buffer(256)
    rc = N.lib().ig_topk_ngrams(C.byref(corpus._view()), C.byref(params), C.byref(out), err, 256)
    assert rc != N.IG_ECONFIG, err.value
    if rc == N.IG_OK:
        N.lib().ig_result_free(C.byref(out))
