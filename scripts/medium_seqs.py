"""Count-once kernel breakdown on medium-length sequences (route path)."""
import numpy as np

from paper_2511_14955_b200 import intergrams as ig, synth as S

for nseq, slen in ((1 << 18, 16384), (1 << 16, 65536)):
    cfg = S.scaled(S.CONFIGS["c2"], num_seqs=nseq, seq_len=slen)
    data, off = S.generate(cfg, 0, -1)
    s = ig.Session(device=0)
    s.load(ig.Corpus(data, np.ascontiguousarray(off, np.uint64)))
    icfg = ig.IntergramConfig(n=6, k=10000, z=1.5, mode=ig.CountMode.kOnce)
    s.run(icfg, materialize=False)
    s.set_profiling(True)
    s.kernel_stats(reset=True)
    r = s.run(icfg, materialize=False)
    st = s.kernel_stats(reset=True)
    print(nseq, slen, {k: (round(v[0], 1), v[1]) for k, v in st.items() if v[1]})
    s.close()
