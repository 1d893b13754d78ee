"""Full-size goldens (TEST INFRASTRUCTURE): runs the REFERENCE itself
(oracle/_ref/libigref.so = /root/reference/proj/src compiled unmodified) on a
BASELINE config's complete synthetic corpus and records the result's digest,
pass rows and diagnostics in tests/golden/fullsize.json.

  python tests/golden/make_fullsize.py c2 [c3 ...] [--file-dir DIR]

c2/c3 run on an in-memory corpus (make_memory_corpus).  Equal-length configs
larger than RAM allows twice (c4, c5) are written once as a flat file and read
by the reference through CorpusSpec{roots={file}, chunk_size=seq_len}
(proj/src/corpus.cpp:89-103), which reproduces the sequence boundaries exactly.
tests/test_gpu_fullsize.py runs the GPU path on the same corpus and compares.
"""
import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2511_14955_b200 import synth as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize.json")


def tsv_digest(keys, counts, n):
    """sha256 of the reference TSV (metrics.cpp:202-211) of the list."""
    h = hashlib.sha256()
    fmt = "%0" + str(2 * n) + "x\t%d\n"
    for i in range(0, len(keys), 65536):
        h.update("".join(fmt % (int(k), int(c)) for k, c in
                         zip(keys[i:i + 65536], counts[i:i + 65536])).encode())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--file-dir", default=os.path.join(ROOT, ".scratch"))
    ap.add_argument("--force-file", action="store_true")
    args = ap.parse_args()
    gold = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in args.configs:
        cfg = S.CONFIGS[name]
        off = S.offsets(cfg)
        total = int(off[-1])
        use_file = args.force_file or (cfg.num_seqs and total > (24 << 30))
        t0 = time.time()
        if use_file:
            os.makedirs(args.file_dir, exist_ok=True)
            path = os.path.join(args.file_dir, f"{name}.bin")
            if not (os.path.exists(path) and os.path.getsize(path) == total):
                mm = np.memmap(path, dtype=np.uint8, mode="w+", shape=(total,))
                for q in range(0, cfg.num_seqs, 1024):  # bounded resident set
                    cnt = min(1024, cfg.num_seqs - q)
                    b0, b1 = int(off[q]), int(off[q + cnt])
                    S.generate(cfg, q, cnt, out=mm[b0:b1])
                    mm.flush()
                del mm
            data = np.memmap(path, dtype=np.uint8, mode="r", shape=(total,))
            fp = S.fingerprint(data, off)
            del data
            print(f"{name}: corpus file {path} ready in {time.time() - t0:.0f}s", flush=True)
            rc, keys, counts, rows, diag, secs, err = O.ref_run_file(
                path, cfg.seq_len, cfg.n, cfg.k, cfg.z, cfg.mode, 0)
        else:
            data, off = S.generate(cfg)
            fp = S.fingerprint(data, off)
            print(f"{name}: corpus generated in {time.time() - t0:.0f}s", flush=True)
            rc, keys, counts, rows, diag, secs, err = O.ref_run(data, off, cfg.n, cfg.k, cfg.z,
                                                                cfg.mode, 0)
            del data
        assert rc == 0, err
        g = {
            "config": name, "n": cfg.n, "k": cfg.k, "z": cfg.z, "mode": cfg.mode,
            "corpus_bytes": total, "num_seqs": int(off.size - 1), "corpus_fingerprint": fp,
            "tsv_sha256": tsv_digest(keys, counts, cfg.n), "len": int(len(keys)),
            "head": [[int(k), int(c)] for k, c in zip(keys[:20], counts[:20])],
            "tail": [[int(k), int(c)] for k, c in zip(keys[-5:], counts[-5:])],
            "counts_sum": int(np.asarray(counts, np.uint64).sum()),
            "passes": [{k: r[k] for k in ("label", "gram_len", "bytes_processed",
                                          "candidate_space", "retained", "retained_short")}
                       for r in rows],
            "diagnostics": diag,
            "reference": {"seconds": secs, "workers": int(O.ref().igref_hardware_concurrency()),
                          "corpus": "file+chunk_size" if use_file else "in-memory",
                          "host": platform.node(), "cpu": platform.processor() or "",
                          "pass_seconds": [round(r["seconds"], 3) for r in rows]},
        }
        gold[name] = g
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1)
        print(f"{name}: reference {secs:.1f}s, len {len(keys)}, sha {g['tsv_sha256'][:16]}",
              flush=True)


if __name__ == "__main__":
    main()
