"""Count-once on many short sequences: time and peak memory of one run."""
import sys
import time

import numpy as np
import torch

from paper_2511_14955_b200 import intergrams as ig, synth as S

for nseq, slen in ((1 << 16, 4096), (1 << 18, 1024), (1 << 20, 1024), (1 << 18, 16384), (1 << 16, 65536)):
    cfg = S.scaled(S.CONFIGS["c2"], num_seqs=nseq, seq_len=slen)
    data, off = S.generate(cfg, 0, -1)
    s = ig.Session(device=0)
    s.load(ig.Corpus(data, np.ascontiguousarray(off, np.uint64)))
    icfg = ig.IntergramConfig(n=6, k=10000, z=1.5, mode=ig.CountMode.kOnce)
    torch.cuda.reset_peak_memory_stats()
    try:
        r = s.run(icfg, materialize=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = s.run(icfg, materialize=False)
        t1 = time.perf_counter()
        free, tot = torch.cuda.mem_get_info()
        print(f"{nseq} x {slen}: {len(data) / (t1 - t0) / 1e9:.2f} GB/s, {(t1 - t0) * 1e3:.0f} ms, "
              f"device used {(tot - free) / 2**30:.1f} GiB", flush=True)
        print("   ", [(p.label, round(p.seconds * 1e3, 1)) for p in r.passes])
    except Exception as e:
        print(nseq, slen, "failed:", e, flush=True)
    s.close()
    del s
