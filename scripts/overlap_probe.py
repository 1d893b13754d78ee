"""Does a 4 GiB pinned H2D copy on another stream slow a resident run?"""
import threading
import time

import numpy as np
import torch

from paper_2511_14955_b200 import intergrams as ig, synth as S

cfg = S.CONFIGS["c2"]
off = S.offsets(cfg)
host = torch.empty(int(off[-1]), dtype=torch.uint8, pin_memory=True)
data, off = S.generate(cfg, 0, -1, out=host.numpy())
s = ig.Session(device=0)
s.load(ig.Corpus(data, np.ascontiguousarray(off, np.uint64)))
icfg = ig.IntergramConfig(n=6, k=10000, z=1.5, mode=ig.CountMode.kOnce)
s.run(icfg, materialize=False)
dev = torch.empty(int(off[-1]), dtype=torch.uint8, device="cuda")
cs = torch.cuda.Stream()


def t_run():
    torch.cuda.synchronize()
    a = time.perf_counter()
    s.run(icfg, materialize=False)
    return (time.perf_counter() - a) * 1e3


def t_copy():
    torch.cuda.synchronize()
    a = time.perf_counter()
    with torch.cuda.stream(cs):
        dev.copy_(host, non_blocking=True)
    cs.synchronize()
    return (time.perf_counter() - a) * 1e3


print("run alone", [round(t_run(), 1) for _ in range(3)])
print("copy alone", [round(t_copy(), 1) for _ in range(3)])
for _ in range(3):
    torch.cuda.synchronize()
    a = time.perf_counter()
    with torch.cuda.stream(cs):
        dev.copy_(host, non_blocking=True)
    r = s.run(icfg, materialize=False)
    b = time.perf_counter()
    cs.synchronize()
    c = time.perf_counter()
    print(f"run with copy in flight: run returned {1e3 * (b - a):.1f} ms, copy done {1e3 * (c - a):.1f} ms")
