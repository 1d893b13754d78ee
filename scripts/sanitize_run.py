"""Small runs of every kernel family for compute-sanitizer (memcheck /
synccheck / racecheck / initcheck): each result is checked against the C
oracle, so a sanitizer run also proves the paths ran to a correct end.

  compute-sanitizer --tool memcheck python scripts/sanitize_run.py [quick|once-exact]

once-exact runs only the count-once sort fallback (its switch
IG_ONCE_EXACT_MIN_K is read once per process, so it gets its own process).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2511_14955_b200 import intergrams as ig  # noqa: E402
from paper_2511_14955_b200 import synth as S  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"


def check(name, data, off, n, k, mode, runner=None):
    cfg = ig.IntergramConfig(n=n, k=k, z=1.5, mode=ig.CountMode(mode))
    r = runner(cfg) if runner else ig.run_intergrams(ig.Corpus(data, off), cfg)
    if n <= 8:
        rc, keys, counts, _, _ = O.oracle_run(data, off, n, k, 1.5, mode)
        ok = rc == 0 and np.array_equal(r.keys, keys) and np.array_equal(r.counts, counts)
    else:
        rc, grams, counts, *_ = O.ref_run_grams(data, off, n, k, 1.5, mode, 0)
        ok = rc == 0 and np.array_equal(r.grams, grams) and np.array_equal(r.counts, counts)
    print(f"{name}: n={n} k={k} mode={mode} len={len(r.counts)} {'OK' if ok else 'MISMATCH'}",
          flush=True)
    return ok


ok = True
if len(sys.argv) > 1 and sys.argv[1] == "once-exact":
    os.environ["IG_ONCE_EXACT_MIN_K"] = "1"
    d, o = S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=8, seq_len=100000))
    ok = check("once-exact", d, o, 5, 500, 0)
    print("ALL OK" if ok else "FAILURES", flush=True)
    sys.exit(0 if ok else 1)
# c1 shape (count-all dense + extension, small tables staged in smem)
d, o = S.generate(S.scaled(S.CONFIGS["c1"], num_seqs=32, seq_len=65536))
ok &= check("c1-sample", d, o, 4, 1024, 1)
# c2 shape: count-once route path (count / scatter / consume), short seqs too
d, o = S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=24, seq_len=1 << 20))
ok &= check("c2-sample", d, o, 6, 2000, 0)
# c3 shape above the hot-sweep threshold (>= 32 MiB): sample, hot set, queued sweep
if not quick:
    d, o = S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=40, seq_len=1 << 20))
    ok &= check("hot-sweep", d, o, 8, 4000, 1)
# c4 shape: small-alphabet direct kernels (split parts forced)
os.environ["IG_DIRECT_SPLIT_BYTES"] = "200000"
d, o = S.generate(S.scaled(S.CONFIGS["c4"], num_seqs=3, seq_len=1 << 20))
ok &= check("c4-direct", d, o, 8, 4096, 0)
d2, o2 = d, o


def resident(cfg):
    s = ig.Session(device=0)
    s.load(ig.Corpus(d2, o2))
    r = s.run(cfg)
    s.close()
    return r


ok &= check("c4-direct-resident", d, o, 8, 4096, 0, resident)
del os.environ["IG_DIRECT_SPLIT_BYTES"]
# long grams (chain emit + sort), both modes
d, o = S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=8, seq_len=60000))
ok &= check("long-grams", d, o, 11, 300, 1)
ok &= check("long-grams-once", d, o, 10, 300, 0)
print("ALL OK" if ok else "FAILURES", flush=True)
sys.exit(0 if ok else 1)
