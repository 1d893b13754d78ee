#!/usr/bin/env python
"""Generates tests/golden/golden.json from the REFERENCE implementation.

The reference CPU path is compiled from its own sources under
/root/reference/proj/src into oracle/_ref/libigref.so (oracle/Makefile; nothing
is copied) and run here through ig_ref::run_intergrams / count_dense /
naive_topk.  The fixtures then travel with the repo and pin both the C oracle
restatement (tests/test_oracle_golden.py, CPU) and the CUDA path
(tests/test_gpu_golden.py, GPU).

Corpora are stored as generator recipes (std::mt19937_64 random corpora exactly
as tests/helpers.hpp:55-65 builds them, the seeded synthetic generator, or
literal byte strings) so the fixture stays small.

    python tests/golden/make_golden.py      # rewrites tests/golden/golden.json
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

ONCE, ALL = 0, 1


def corpus_from(recipe):
    kind = recipe["kind"]
    if kind == "literal":
        seqs = [bytes.fromhex(h) for h in recipe["hex"]]
        return O.csr(seqs)
    if kind == "random":
        rng = O.Mt64(recipe["seed"])
        for _ in range(recipe.get("skip", 0)):
            O.random_corpus(rng, recipe["max_m"], recipe["max_len"], recipe["alphabet"])
        seqs = O.random_corpus(rng, recipe["max_m"], recipe["max_len"], recipe["alphabet"])
        return O.csr(seqs)
    if kind == "synth":
        from paper_2511_14955_b200 import synth as S
        cfg = S.scaled(S.CONFIGS[recipe["config"]], num_seqs=recipe.get("num_seqs"),
                       seq_len=recipe.get("seq_len"), total=recipe.get("total"))
        data, off = S.generate(cfg, 0, recipe.get("count", -1))
        return data, off
    raise ValueError(kind)


def tsv(keys, counts, n):
    return "".join(f"{int(k):0{2 * n}x}\t{int(c)}\n" for k, c in zip(keys, counts))


def run_case(recipe, n, k, z, mode):
    data, off = corpus_from(recipe)
    rc, keys, counts, rows, diag, secs, err = O.ref_run(data, off, n, k, z, mode, 1)
    case = {"corpus": recipe, "n": n, "k": k, "z": z, "mode": mode, "rc": rc}
    if rc == 0:
        case["tsv"] = tsv(keys, counts, n)
        case["passes"] = [{kk: r[kk] for kk in ("label", "gram_len", "bytes_processed",
                                                  "candidate_space", "retained",
                                                  "retained_short")} for r in rows]
        case["diagnostics"] = diag
    else:
        case["error"] = err
    return case


def main():
    cases = []
    lit = lambda *ss: {"kind": "literal", "hex": [s.hex() for s in ss]}  # noqa: E731
    # known-answer corpora from the reference tests and the survey probes
    cases.append(run_case(lit(b"abab", b"abba"), 4, 1, 100.0, ONCE))  # test_intergrams.cpp:119
    cases.append(run_case(lit(b"aaaa", b"aaab"), 4, 5, 10.0, ONCE))  # test_intergrams.cpp:210
    cases.append(run_case(lit(b"aaaa", b"aaab"), 3, 2, 1.0, ONCE))   # SPEC.md:693 golden
    cases.append(run_case(lit(b"aaaa", b"aaab"), 3, 2, 1.0, ALL))
    cases.append(run_case(lit(b"abcxbcd"), 3, 5, 1.0, ONCE))        # test_dense_pass.cpp:103
    cases.append(run_case(lit(b"ab"), 4, 3, 1.5, ALL))              # probe P5: ConfigError
    cases.append(run_case(lit(b"abab"), 5, 3, 1.5, ALL))            # probe P5: empty list
    cases.append(run_case(lit(b"abab"), 6, 3, 1.5, ALL))            # probe P5: ConfigError
    cases.append(run_case(lit(bytes([0xff, 0, 1, 2, 0x80]), bytes([0, 1, 2, 3, 0x7f])),
                          4, 10, 1.5, ALL))                         # probe P6: byte order
    cases.append(run_case(lit(), 3, 4, 1.5, ONCE))                  # empty corpus
    cases.append(run_case(lit(b"", b"", b"xyz", b""), 3, 4, 1.5, ONCE))
    cases.append(run_case(lit(b"", b"a", b"ab", b"abc", b"abcd", b"abcde"), 4, 8, 2.0, ALL))
    cases.append(run_case(lit(bytes(range(256)) * 3), 2, 300, 1.0, ALL))
    cases.append(run_case(lit(b"\x00" * 40, b"\xff" * 40), 8, 4, 1.0, ONCE))
    # random corpora (tests/helpers.hpp random_corpus), all n and both modes
    seed = 7000
    for n in range(1, 9):
        for mode in (ONCE, ALL):
            for alphabet, max_len in ((4, 200), (6, 400), (256, 300)):
                seed += 1
                rec = {"kind": "random", "seed": seed, "max_m": 12, "max_len": max_len,
                       "alphabet": alphabet}
                for k, z in ((9, 1.5), (40, 1.0)):
                    cases.append(run_case(rec, n, k, z, mode))
    # full retention (test_intergrams.cpp:149-161 shape)
    for t in range(4):
        rec = {"kind": "random", "seed": 909, "skip": t, "max_m": 8, "max_len": 200,
               "alphabet": 4}
        data, off = corpus_from(rec)
        z = max(1.0, (int(off[-1]) + 1) / 16)
        for mode in (ONCE, ALL):
            cases.append(run_case(rec, 5, 16, z, mode))
    # seeded synthetic corpora with the BASELINE generators (small)
    for cfg, n, k, mode, extra in (("c1", 4, 64, ALL, {"num_seqs": 16, "seq_len": 16384}),
                                   ("c2", 6, 100, ONCE, {"num_seqs": 24, "seq_len": 8192}),
                                   ("c3", 8, 200, ALL, {"total": 300000}),
                                   ("c4", 8, 128, ONCE, {"num_seqs": 12, "seq_len": 4096}),
                                   ("c5", 8, 500, ALL, {"num_seqs": 8, "seq_len": 16384})):
        rec = {"kind": "synth", "config": cfg, **extra}
        cases.append(run_case(rec, n, k, 1.5, mode))
    # dense tables (count_dense) as digests
    tables = []
    for seed in (2024, 31, 3):
        rec = {"kind": "random", "seed": seed, "max_m": 24, "max_len": 400, "alphabet": 64}
        data, off = corpus_from(rec)
        for n in (1, 2, 3):
            for mode in (ONCE, ALL):
                t = O.ref_count_dense(data, off, n, mode, 1)
                tables.append({"corpus": rec, "n": n, "mode": mode,
                               "sha256": hashlib.sha256(t.astype("<u8").tobytes()).hexdigest(),
                               "total": int(t.sum()), "nonzero": int((t != 0).sum())})
    # hash-gramming (run_hashgram, hashgram.cpp:325-383) and featurize
    # (metrics.cpp:83-132), §8(f) rows 3-4
    hashgram = []
    seed = 9100
    for n in (1, 2, 3, 4, 6, 8):
        for mode in (ONCE, ALL):
            for B, k, hseed in ((1, 3, 0), (7, 4, 1), (97, 10, 0), (1 << 20, 25, 12345),
                                (1 << 31, 40, 0), (1 << 40, 30, 99)):
                seed += 1
                if B > (1 << 33):  # the reference's dense CountTable(B) cannot be allocated
                    continue
                rec = {"kind": "random", "seed": seed, "max_m": 10, "max_len": 300,
                       "alphabet": 5 if n > 3 else 64}
                data, off = corpus_from(rec)
                rc, keys, counts, rows, err = O.ref_hashgram(data, off, n, k, mode, B, hseed)
                case = {"corpus": rec, "n": n, "k": k, "mode": mode, "buckets": B,
                        "seed": hseed, "rc": rc}
                if rc == 0:
                    case["tsv"] = tsv(keys, counts, n)
                    case["passes"] = [{kk: r[kk] for kk in ("label", "gram_len",
                                                             "bytes_processed",
                                                             "candidate_space", "retained",
                                                             "retained_short")} for r in rows]
                hashgram.append(case)
    mix = []
    for s in (b"", b"a", b"ab", b"abcdefg", b"abcdefgh", b"abcdefghi", bytes(range(200, 217))):
        for hs in (0, 1, 0xDEADBEEF, (1 << 64) - 1):
            mix.append({"hex": s.hex(), "seed": hs, "mix64": O.ref_mix64(s, hs)})
    feats = []
    seed = 9500
    for n in (1, 2, 3, 4, 5, 8):
        for vocab_kind in ("sampled", "with_dups", "absent"):
            seed += 1
            rec = {"kind": "random", "seed": seed, "max_m": 16, "max_len": 250, "alphabet": 4}
            data, off = corpus_from(rec)
            seqs = [bytes(data[int(off[i]):int(off[i + 1])]) for i in range(off.size - 1)]
            grams = sorted({s[i:i + n] for s in seqs for i in range(0, max(len(s) - n + 1, 0), 5)})
            vocab = grams[: 12]
            if vocab_kind == "with_dups":
                vocab = vocab + vocab[:4][::-1]
            elif vocab_kind == "absent":
                vocab = [bytes([250 + (i % 6)]) * n for i in range(3)] + vocab[:2]
            rc, ent, nrows, err = O.ref_featurize(data, off, vocab)
            feats.append({"corpus": rec, "n": n, "vocab": [v.hex() for v in vocab], "rc": rc,
                          "rows": nrows, "entries": [int(e) for e in ent]})
    rec = {"kind": "literal", "hex": [b"abcabc".hex(), b"".hex(), b"xyz".hex()]}
    data, off = corpus_from(rec)
    rc, ent, nrows, err = O.ref_featurize(data, off, [b"bc", b"ab", b"zz", b"bc"])
    feats.append({"corpus": rec, "n": 2, "vocab": ["6263", "6162", "7a7a", "6263"], "rc": rc,
                  "rows": nrows, "entries": [int(e) for e in ent]})
    rc, ent, nrows, err = O.ref_featurize(data, off, [])
    feats.append({"corpus": rec, "n": 0, "vocab": [], "rc": rc, "rows": nrows,
                  "entries": [int(e) for e in ent]})
    out = {"generator": "tests/golden/make_golden.py (reference compiled from "
                        "/root/reference/proj/src via oracle/Makefile)",
           "cases": cases, "dense_tables": tables}
    # RunReport::to_tsv / to_json (metrics.cpp:134-200) of fixed rows, incl.
    # doubles that exercise every branch of the JSON number formatting
    reports = []
    secs = [0.0, 1.5, 2.0, 0.1 + 0.2, 1e-5, 3.25e-7, 123456.789, 1e15, 1e16, 1.2345678901234567e21,
            0.0001, 0.00012345, 7.0 / 3.0, 1e-300, 5e-324, 9007199254740993.0, 42.0]
    for i in range(0, len(secs), 3):
        rows = [dict(label=f"{3 + j}-gram pass" if j % 2 == 0 else f"top-zk {3 + j}-grams/trie building",
                     gram_len=3 + j, seconds=s, bytes_processed=(j + 1) * 1000003 if j % 2 == 0 else 0,
                     candidate_space=1 << (8 + j), retained=17 * j, retained_short=j % 3 == 1)
                for j, s in enumerate(secs[i:i + 3])]
        for js in (False, True):
            for jac in (None, 0.123456789, 1.0):
                reports.append({"algorithm": "intergrams", "echo": "algorithm=intergrams n=6 k=10 z=1.5",
                                "rows": [dict(r, seconds=r["seconds"].hex()) for r in rows],
                                "json": js, "jaccard": None if jac is None else jac.hex(),
                                "text": O.ref_report("intergrams", "algorithm=intergrams n=6 k=10 z=1.5",
                                                     rows, jac, js)})
    reports.append({"algorithm": "naive", "echo": "algorithm=naive n=3 k=2 mode=once", "rows": [],
                    "json": True, "jaccard": None,
                    "text": O.ref_report("naive", "algorithm=naive n=3 k=2 mode=once", [], None, True)})
    extra = {"generator": out["generator"], "hashgram": hashgram, "mix64": mix,
             "featurize": feats, "reports": reports}
    with open(os.path.join(ROOT, "tests", "golden", "golden_extra.json"), "w") as f:
        json.dump(extra, f, indent=1)
    print(f"wrote {len(hashgram)} hashgram, {len(mix)} mix64, {len(feats)} featurize cases")
    path = os.path.join(ROOT, "tests", "golden", "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {len(cases)} cases, {len(tables)} tables -> {path}")


if __name__ == "__main__":
    main()
