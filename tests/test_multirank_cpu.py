"""The N>1 host path on CPU: world_size-2 gloo ranks, each holding its
byte-balanced whole-sequence shard (ig_shard_range), sum every pass's count
table with all_reduce and run the same deterministic selection — exactly the
orchestration the CUDA driver runs with its allreduce hook (session.cu
run_t/allreduce).  The per-rank counting uses the C oracle here (no GPU); the
final list must equal the single-process reference result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2511_14955_b200 import intergrams as ig


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce_u64(t: np.ndarray) -> np.ndarray:
    # unsigned counters summed as the same bits in int64 (what bench.py's NCCL hook does)
    x = torch.from_numpy(t.view(np.int64).copy())
    dist.all_reduce(x)
    return x.numpy().view(np.uint64)


def sharded_run(rank, world, data, off, n, k, z, mode):
    a, b = ig.shard_range(off, rank, world)
    ld = data[int(off[a]):int(off[b])].copy()
    loff = (off[a:b + 1] - off[a]).astype(np.uint64)
    kp = int(np.ceil(z * k))
    n0 = min(n, 3)
    table = _allreduce_u64(O.oracle_count_dense(ld, loff, n0, mode))
    if n <= 3:
        return O.oracle_top_k(table, k)
    sk, _ = O.oracle_top_k(table, kp)
    for j in range(4, n + 1):
        if sk.size == 0:
            return None  # ConfigError on every rank
        rc, t, _ = O.oracle_extend(ld, loff, sk, j - 1, j, mode)
        assert rc == 0
        t = _allreduce_u64(t)
        if j < n:
            nk, _ = O.oracle_top_k(t, kp, sk)
            sk = nk
        else:
            return O.oracle_top_k(t, k, sk)


def _worker(rank, world, port, cases, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    for (seed, n, k, z, mode) in cases:
        rng = O.Mt64(seed)
        seqs = O.random_corpus(rng, 40, 600, 5)
        d, off = O.csr(seqs)
        r = sharded_run(rank, world, d, off, n, k, z, mode)
        res.append(None if r is None else (r[0].tolist(), r[1].tolist()))
    # every rank must hold the identical list
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    if rank == 0:
        out.put(gathered)
    dist.destroy_process_group()


CASES = [(11, 3, 8, 1.5, O.ONCE), (12, 4, 10, 1.5, O.ALL), (13, 6, 12, 1.5, O.ONCE),
         (14, 5, 5, 2.0, O.ALL), (15, 8, 20, 1.5, O.ONCE), (16, 2, 30, 1.0, O.ALL)]


def test_two_rank_gloo_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, CASES, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert gathered[0] == gathered[1]
    for (seed, n, k, z, mode), got in zip(CASES, gathered[0]):
        rng = O.Mt64(seed)
        seqs = O.random_corpus(rng, 40, 600, 5)
        d, off = O.csr(seqs)
        if O.ref_available():
            rc, keys, counts = O.ref_run(d, off, n, k, z, mode, 1)[:3]
        else:
            rc, keys, counts = O.oracle_run(d, off, n, k, z, mode)[:3]
        if rc != 0:
            assert got is None
        else:
            assert got == (keys.tolist(), counts.tolist())


def test_u32_sum_as_i32_bits():
    a = np.array([0xFFFFFFF0, 5, 0x80000000], np.uint32)
    b = np.array([0x0000000F, 7, 0x7FFFFFFF], np.uint32)
    s = (a.view(np.int32).astype(np.int64) + b.view(np.int32).astype(np.int64)).astype(np.int32)
    assert np.array_equal(s.view(np.uint32), (a.astype(np.uint64) + b) .astype(np.uint32))
