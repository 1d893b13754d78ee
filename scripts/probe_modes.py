"""Timing probe: one config's corpus counted in a chosen mode (experiments).
usage: python scripts/probe_modes.py CONFIG MODE(all|once) [SEQS|TOTAL_GIB] [N] [K]"""
import hashlib
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2511_14955_b200 import intergrams as ig  # noqa: E402
from paper_2511_14955_b200 import synth as S  # noqa: E402

name, mode = sys.argv[1], sys.argv[2]
cfg = S.CONFIGS[name]
if len(sys.argv) > 3:
    v = float(sys.argv[3])
    cfg = S.scaled(cfg, total=int(v * 2**30)) if cfg.kind == S.K_LOGNORMAL else S.scaled(cfg, num_seqs=int(v))
n = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.n
k = int(sys.argv[5]) if len(sys.argv) > 5 else cfg.k
t0 = time.time()
data, off = S.generate(cfg)
print("generated", data.size, "B in", round(time.time() - t0, 1), "s", flush=True)
s = ig.Session(device=0)
s.load(ig.Corpus(data, off))
icfg = ig.IntergramConfig(n=n, k=k, z=1.5,
                          mode=ig.CountMode.kAll if mode == "all" else ig.CountMode.kOnce, device=0)
r = s.run(icfg, materialize=False)
s.set_profiling(True)
s.kernel_stats(reset=True)
reps = 2
t0 = time.time()
for _ in range(reps):
    r = s.run(icfg, materialize=False)
dt = (time.time() - t0) / reps
ks = s.kernel_stats(reset=True)
print(json.dumps({"config": name, "mode": mode, "bytes": int(data.size), "n": n, "k": k,
                  "ms_wall": dt * 1e3, "GBps": data.size / dt / 1e9,
                  "digest": hashlib.sha256(r.keys.tobytes() + r.counts.tobytes()).hexdigest()[:12],
                  "passes": {p.label: round(p.seconds * 1e3, 2) for p in r.passes},
                  "kernels": {f: round(v[0] / reps, 2) for f, v in ks.items() if v[1]}}), flush=True)
