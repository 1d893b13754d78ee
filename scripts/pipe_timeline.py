"""Timeline of two sessions pipelining load_and_run on one GPU (host clocks)."""
import threading
import time

import numpy as np
import torch

from paper_2511_14955_b200 import intergrams as ig, synth as S

cfg = S.CONFIGS["c2"]
off = S.offsets(cfg)
host = torch.empty(int(off[-1]), dtype=torch.uint8, pin_memory=True)
data, off = S.generate(cfg, 0, -1, out=host.numpy())
corpus = ig.Corpus(data, np.ascontiguousarray(off, np.uint64))
icfg = ig.IntergramConfig(n=6, k=10000, z=1.5, mode=ig.CountMode.kOnce)
sess = [ig.Session(device=0, stream=torch.cuda.Stream().cuda_stream) for _ in range(2)]
for s in sess:
    s.load_and_run(corpus, icfg, materialize=False)
torch.cuda.synchronize()
T0 = time.perf_counter()
log = []


import sys
DELAY = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0


def worker(i):
    if i:
        time.sleep(DELAY)
    for r in range(4):
        a = time.perf_counter()
        sess[i].load_and_run(corpus, icfg, materialize=False)
        b = time.perf_counter()
        log.append((i, r, (a - T0) * 1e3, (b - T0) * 1e3))


th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
for e in sorted(log, key=lambda x: x[2]):
    print(f"session {e[0]} run {e[1]}: {e[2]:7.1f} -> {e[3]:7.1f} ms ({e[3] - e[2]:.1f})")
print("total", round((time.perf_counter() - T0) * 1e3, 1), "ms for 8 runs")
a = time.perf_counter()
for r in range(4):
    sess[0].load_and_run(corpus, icfg, materialize=False)
print("serial 4 runs", round((time.perf_counter() - a) * 1e3, 1), "ms")
