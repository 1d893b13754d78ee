"""Count-once with a survivor set beyond the route path (exact sort fallback)."""
import time

import numpy as np

from paper_2511_14955_b200 import intergrams as ig

rng = np.random.default_rng(1)
m, ln = 64, 1 << 20
data = rng.integers(0, 256, m * ln, dtype=np.uint8)
off = np.arange(0, m * ln + 1, ln, dtype=np.uint64)
s = ig.Session(device=0)
s.load(ig.Corpus(data, off))
cfg = ig.IntergramConfig(n=4, k=3_000_000, z=1.0, mode=ig.CountMode.kOnce)
t0 = time.perf_counter()
r = s.run(cfg, materialize=False)
t1 = time.perf_counter()
print("passes", [(p.label, p.retained, round(p.seconds * 1e3, 1)) for p in r.passes])
print("len", len(r.keys), "max count", int(r.counts.max()), "min", int(r.counts.min()),
      f"{(t1 - t0) * 1e3:.0f} ms")
assert int(r.counts.max()) <= m
