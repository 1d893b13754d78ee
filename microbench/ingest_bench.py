"""File ingestion throughput (csrc/ingest.cu): the c2 corpus written as 16
files of 256 MiB and read back as 1 MiB chunk records (the same 4096
sequences), page-cache resident.  Prints load-only and load+run GB/s and
checks the list against the in-memory run."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14955_b200 import intergrams as ig, synth as S  # noqa: E402

cfg = S.CONFIGS["c2"]
data, off = S.generate(cfg, 0, -1)
d = "/tmp/ig_c2_files"
os.makedirs(d, exist_ok=True)
per = len(data) // 16
for i in range(16):
    with open(f"{d}/part{i:02d}.bin", "wb") as f:
        f.write(data[i * per:(i + 1) * per].tobytes())
spec = ig.CorpusSpec([d], chunk_size=1 << 20)
icfg = ig.IntergramConfig(n=6, k=10000, z=1.5, mode=ig.CountMode.kOnce)
s = ig.Session(device=0)
s.load_files(spec)  # warm: pinned slabs, buffers
for rep in range(3):
    t0 = time.perf_counter()
    s.load_files(spec)
    t1 = time.perf_counter()
    r = s.run(icfg, materialize=False)
    t2 = time.perf_counter()
    print(f"load {len(data) / (t1 - t0) / 1e9:.1f} GB/s ({(t1 - t0) * 1e3:.0f} ms), "
          f"load+run {len(data) / (t2 - t0) / 1e9:.1f} GB/s ({(t2 - t0) * 1e3:.0f} ms)")
for rep in range(3):
    t0 = time.perf_counter()
    r = s.run_files(spec, icfg, materialize=False)
    t1 = time.perf_counter()
    print(f"run_files (dense pass overlapped with the load) {len(data) / (t1 - t0) / 1e9:.1f} GB/s "
          f"({(t1 - t0) * 1e3:.0f} ms)")
ref = ig.Session(device=0)
ref.load(ig.Corpus(data, np.ascontiguousarray(off, np.uint64)))
r2 = ref.run(icfg, materialize=False)
assert np.array_equal(r.keys, r2.keys) and np.array_equal(r.counts, r2.counts)
print("identical list:", len(r.keys), "grams; host cores", os.cpu_count())
