import numpy as np
from paper_2511_14955_b200 import synth as S, intergrams as ig
cfg = S.CONFIGS["c4"]
data, off = S.generate(cfg, 0, 256)
s = ig.Session(device=0)
s.load(ig.Corpus(data, np.ascontiguousarray(off, np.uint64)))
r = s.run(ig.IntergramConfig(n=8, k=65536, z=1.5, mode=ig.CountMode.kOnce), materialize=False)
for p in r.passes: print(p.label, p.retained, p.candidate_space, round(p.seconds*1e3,2))
