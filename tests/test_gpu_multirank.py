"""The C-ABI collective hook on one GPU: two sessions (ranks) run concurrently
in two host threads, each on its own whole-sequence shard; the allreduce
callback sums the per-pass tables through host memory with a barrier (the
kernels never wait on each other).  Both ranks must return the single-session
result bit for bit — what NCCL provides across real GPUs."""
import ctypes as C
import threading

import numpy as np
import pytest
import torch

from paper_2511_14955_b200 import _native as N
from paper_2511_14955_b200 import intergrams as ig
from paper_2511_14955_b200 import synth as S

pytestmark = pytest.mark.gpu


class HostAllreduce:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.bufs = {}
        self.calls = 0
        self.dtypes = []

    def make(self, rank):
        def cb(buf, count, dtype, stream, user):
            try:
                typestr = "<u4" if dtype == 0 else "<u8"
                cai = type("CAI", (), {})()
                cai.__cuda_array_interface__ = {"data": (buf, False), "shape": (int(count),),
                                                "typestr": "<i4" if dtype == 0 else "<i8",
                                                "version": 3, "strides": None}
                dev = torch.as_tensor(cai, device="cuda")
                torch.cuda.ExternalStream(stream).synchronize()
                self.bufs[rank] = dev.cpu().numpy().view(typestr[1:].replace("u", "uint")
                                                         .replace("4", "32").replace("8", "64"))
                self.bar.wait()
                dt = np.uint32 if dtype == 0 else np.uint64
                total = sum(self.bufs[r].astype(np.uint64) for r in range(self.world)).astype(dt)
                self.bar.wait()
                dev.copy_(torch.from_numpy(total.view(np.int32 if dtype == 0 else np.int64)))
                torch.cuda.synchronize()
                if rank == 0:
                    self.calls += 1
                    self.dtypes.append((int(dtype), int(count)))
                return 0
            except Exception as e:  # noqa: BLE001
                print("allreduce failed", repr(e))
                return 1
        return N.ALLREDUCE_FN(cb)


@pytest.mark.parametrize("name,n,k,mode", [("c1", 4, 256, 1), ("c2", 6, 500, 0)])
def test_two_ranks_equal_one(gpu_lib, name, n, k, mode):
    cfg = S.scaled(S.CONFIGS[name], num_seqs=24, seq_len=65536)
    data, off = S.generate(cfg)
    icfg = ig.IntergramConfig(n=n, k=k, z=1.5, mode=ig.CountMode(mode))
    single = ig.run_intergrams(ig.Corpus(data, off), icfg)
    ar = HostAllreduce(2)
    results = [None, None]
    cbs = [ar.make(r) for r in range(2)]

    def rank_main(r):
        a, b = ig.shard_range(off, r, 2)
        ld = data[int(off[a]):int(off[b])]
        loff = (off[a:b + 1] - off[a]).astype(np.uint64)
        coll = N.ig_collective(rank=r, world=2, bytes_total=int(off[-1]),
                               seqs_total=int(off.size - 1), allreduce=cbs[r], user=None)
        sess = ig.Session(device=0, collective=coll)
        sess.load(ig.Corpus(ld, loff))
        results[r] = sess.run(icfg)
        sess.close()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert ar.calls == max(n, 3) - 2
    for r in range(2):
        assert results[r] is not None
        assert results[r].topk == single.topk
        assert [p.bytes_processed for p in results[r].passes] == \
               [p.bytes_processed for p in single.passes]


@pytest.mark.parametrize("force_u64", [False, True])
def test_two_ranks_u64_tables_narrowed(gpu_lib, monkeypatch, force_u64):
    """Count-all with a total that might reach 2^32 (bytes_total 8 GiB): the
    dense table is u64, and its all-reduce goes through the hook as one u64
    bound (sum of the per-rank maxima) followed by the table as u32.  Every
    extension pass's counts are bounded by the previous pass's top count,
    so those tables are u32 from the start (one call each) -- unless u64
    tables are forced, when every pass takes the bound + u32 route."""
    if force_u64:
        monkeypatch.setenv("IG_FORCE_U64", "1")
    cfg = S.scaled(S.CONFIGS["c5"], num_seqs=16, seq_len=65536)
    data, off = S.generate(cfg)
    icfg = ig.IntergramConfig(n=6, k=300, z=1.5, mode=ig.CountMode.kAll)
    single = ig.run_intergrams(ig.Corpus(data, off), icfg)
    ar = HostAllreduce(2)
    results = [None, None]
    cbs = [ar.make(r) for r in range(2)]

    def rank_main(r):
        a, b = ig.shard_range(off, r, 2)
        ld = data[int(off[a]):int(off[b])]
        loff = (off[a:b + 1] - off[a]).astype(np.uint64)
        coll = N.ig_collective(rank=r, world=2, bytes_total=8 << 30,
                               seqs_total=int(off.size - 1), allreduce=cbs[r], user=None)
        sess = ig.Session(device=0, collective=coll)
        sess.load(ig.Corpus(ld, loff))
        results[r] = sess.run(icfg)
        sess.close()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    passes = 6 - 2
    # bound (u64), then the table (u32)
    want = [1, 0] * passes if force_u64 else [1, 0] + [0] * (passes - 1)
    assert ar.calls == len(want)
    assert [d for d, _ in ar.dtypes] == want
    assert all(c == 1 for d, c in ar.dtypes if d == 1)
    for r in range(2):
        assert results[r] is not None
        assert np.array_equal(results[r].keys, single.keys)
        assert np.array_equal(results[r].counts, single.counts)
