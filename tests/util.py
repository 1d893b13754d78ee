"""Shared helpers for the parity tests (test infrastructure)."""
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden.json")


def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def corpus_from(recipe):
    from tests.golden.make_golden import corpus_from as cf
    return cf(recipe)


def tsv(keys, counts, n):
    return "".join(f"{int(k):0{2 * n}x}\t{int(c)}\n" for k, c in zip(keys, counts))


def case_id(c):
    r = c["corpus"]
    tag = r["kind"] + ("-" + str(r.get("seed", r.get("config", ""))) if r["kind"] != "literal" else "")
    return f"{tag}-n{c['n']}-k{c['k']}-m{c['mode']}"
