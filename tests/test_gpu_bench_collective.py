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


def _bench(config, extra_env, torchrun):
    args = ["bench.py", "--config", config, "--seqs", "24", "--steps", "1", "--warmup", "3",
            "--no-cpu-baseline", "--no-e2e"]
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
