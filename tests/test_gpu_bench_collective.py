"""bench.py's multi-GPU plumbing on one GPU: a 1-rank NCCL group launched by
torchrun with the C-ABI collective hook installed (IG_BENCH_FORCE_COLLECTIVE=1).
Every counting pass must go through torch.distributed.all_reduce, and the
result digest must equal the run without a collective."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _bench(config, extra_env, torchrun, collective="torch"):
    args = ["bench.py", "--config", config, "--seqs", "24", "--steps", "1", "--warmup", "3",
            "--no-cpu-baseline", "--no-e2e", "--collective", collective]
    if torchrun:
        args = ["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                "--master-addr", "127.0.0.1", "--master-port", str(_free_port())] + args
    env = dict(os.environ, **extra_env)
    out = subprocess.run([sys.executable] + args, cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


# c2: count-once u32 tables, one all-reduce per pass.  c3 (24 sequences,
# u64 tables forced as for a > 4 GiB corpus): a u64 bound, then the table
# narrowed to u32.
@pytest.mark.parametrize("config,calls_per_pass", [("c2", 1), ("c3", 2)])
def test_bench_collective_hook_equals_single(gpu_lib, config, calls_per_pass):
    env = {"IG_FORCE_U64": "1"} if calls_per_pass == 2 else {}
    plain = _bench(config, env, torchrun=False)
    coll = _bench(config, dict(env, IG_BENCH_FORCE_COLLECTIVE="1"), torchrun=True)
    assert plain["collective"] is None
    assert coll["collective"]["backend"] == "nccl"
    # every counting pass of every run (3 warm-up + 1 timed)
    passes = max(coll["config"]["n"], 3) - 2
    assert coll["collective"]["allreduce_calls"] == 4 * passes * calls_per_pass
    assert coll["result_digest"] == plain["result_digest"]


# The library's own communicator (ig_nccl_unique_id -> broadcast over the
# torch group -> ig_session_create_nccl): every pass table goes through
# ncclAllReduce on the session stream (a 1-rank group here, forced on).
@pytest.mark.parametrize("config", ["c2", "c3"])
def test_bench_library_nccl_equals_single(gpu_lib, config):
    env = {"IG_FORCE_U64": "1"} if config == "c3" else {}
    plain = _bench(config, env, torchrun=False, collective="lib")
    coll = _bench(config, dict(env, IG_BENCH_FORCE_COLLECTIVE="1"), torchrun=True,
                  collective="lib")
    assert plain["collective"] is None
    assert coll["collective"]["owner"].startswith("library")
    assert coll["result_digest"] == plain["result_digest"]


MULTI = r"""
import os, sys, json
import numpy as np
sys.path.insert(0, %r)
from paper_2511_14955_b200 import intergrams as ig, synth as S
data, off = S.generate(S.scaled(S.CONFIGS["c2"], num_seqs=40, seq_len=200_000))
out = {}
for mode in (0, 1):
    cfg = ig.IntergramConfig(n=6, k=2000, z=1.5, mode=ig.CountMode(mode))
    a = ig.run_intergrams(ig.Corpus(data, off), cfg)
    b = ig.run_intergrams_multi(ig.Corpus(data, off), cfg, devices=[0])
    out[mode] = bool(np.array_equal(a.keys, b.keys) and np.array_equal(a.counts, b.counts))
try:
    ig.run_intergrams_multi(ig.Corpus(data, off), cfg, devices=[])
    out["empty"] = "no error"
except ig.ConfigError:
    out["empty"] = "ConfigError"
print(json.dumps(out))
"""


def test_multi_device_entry_point_one_gpu(gpu_lib):
    # ig_topk_ngrams_multi on the one GPU of the box: ncclCommInitAll over
    # [0], one session per device on its own thread, the all-reduce forced at
    # world 1 so every pass table really goes through NCCL
    env = dict(os.environ, IG_COLLECTIVE_AT_WORLD1="1")
    out = subprocess.run([sys.executable, "-c", MULTI % ROOT], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res == {"0": True, "1": True, "empty": "ConfigError"}
