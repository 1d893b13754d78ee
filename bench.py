#!/usr/bin/env python
"""Benchmark of the B200-native Intergrams top-k n-gram run (BASELINE.json metric:
input GB/s per top-k n-gram run, and % of the HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one full run_intergrams (every counting pass, every top-k' selection
and prefix-set build, the final top-k list copied to the host) over the
config's synthetic corpus.  The default workload is BASELINE configs[2] (c3:
16 GiB lognormal-length Zipf-token corpus, n=8, k=100000, count-all), the
config the metric's 1/2/4/8-GPU figure is quoted on; it fits one B200.  For
N>1 (one process per GPU; `--gpus N` without torchrun re-launches itself
under torch.distributed.run) the fixed corpus is sharded by whole sequences,
balanced by bytes (strong scaling), and each pass's count table is summed
with an NCCL all-reduce.

`value` is device-timed with CUDA events on the library's stream with the corpus
resident in HBM; `e2e` is the same metric through the public session API with
the corpus in pinned host memory, the H2D copy and the result D2H inside the
timed region.  `--impl reference` times the reference CPU implementation
(compiled from its own sources into oracle/_ref) on the same config: each
timed step is one complete run over a bounded sample of whole sequences, the
samples spread evenly over the corpus.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input GB/s per top-k n-gram run (1/2/4/8 B200) and % of HBM roofline"
UNIT = "GB/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled from a thread (every ~2 ms for the first samples so that short
    regions such as c1's still get some, then every 50 ms), else
    nvidia-smi -lms 100."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.stop = threading.Event()
        self.t = None
        self.period = float(os.environ.get("IG_CLOCK_POLL_MS", "50")) * 1e-3

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml_sample(pynvml, h)  # fails here, not in the thread, without NVML
            self.t = threading.Thread(target=self._poll, args=(pynvml, h), daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _nvml_sample(self, pynvml, h):
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        return sm, mx, rs

    def _poll(self, pynvml, h):
        while not self.stop.is_set():
            try:
                s = self._nvml_sample(pynvml, h)
                self.samples.append((float(s[0]), float(s[1]), int(s[2])))
            except Exception:
                return
            # dense at first (a 7 ms c1 region still gets samples), then
            # every 50 ms: each NVML query takes driver locks the launching
            # thread also needs, and 2 ms polling cost a c3 step ~20 ms
            self.stop.wait(0.002 if len(self.samples) < 8 else self.period)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        elif self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = set()
        for s in self.samples:
            for bit, name in REASON_BITS.items():
                if s[2] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ collective

def make_collective(rank, world, bytes_total, seqs_total):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2511_14955_b200 import _native as N

    calls = [0]

    class _CAI:
        def __init__(self, ptr, n, typestr):
            self.__cuda_array_interface__ = {"data": (ptr, False), "shape": (n,),
                                             "typestr": typestr, "version": 3, "strides": None}

    def _allreduce(buf, count, dtype, stream, user):
        calls[0] += 1
        try:
            # sum of unsigned counters == sum of the same bits as signed ints (mod 2^w)
            t = torch.as_tensor(_CAI(buf, count, "<i4" if dtype == 0 else "<i8"), device="cuda")
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                dist.all_reduce(t)
            return 0
        except Exception as e:  # noqa: BLE001
            log("allreduce failed:", e)
            return 1

    cb = N.ALLREDUCE_FN(_allreduce)
    coll = N.ig_collective(rank=rank, world=world, bytes_total=bytes_total,
                           seqs_total=seqs_total, allreduce=cb, user=None)
    coll.calls = calls  # python-side counter (the ctypes struct keeps a reference)
    return coll, cb


# ------------------------------------------------------------------ reference arm

def ref_samples(cfg, nsamples, sample_bytes):
    """Whole-sequence samples of cfg spread over the corpus: sample i starts at
    the first sequence at or after byte i*total/nsamples and takes sequences
    until it holds >= sample_bytes (at least one)."""
    from paper_2511_14955_b200 import synth as S
    off = S.offsets(cfg)
    m, total = off.size - 1, int(off[-1])
    out = []
    for i in range(nsamples):
        q = int(np.searchsorted(off, i * total // nsamples, side="left"))
        q = min(q, m - 1)
        e = int(np.searchsorted(off, int(off[q]) + sample_bytes, side="left"))
        e = max(q + 1, min(e, m))
        out.append((q, e - q))
    return out


def ref_plan(args, cfg):
    """(timed steps, bytes per step) of the reference arm: --ref-bytes of the
    corpus in total, at most --steps samples of >= --ref-min-step bytes each."""
    from paper_2511_14955_b200 import synth as S
    total = int(S.offsets(cfg)[-1])
    budget = min(args.ref_bytes, total)
    steps = max(1, min(args.steps, budget // args.ref_min_step))
    return steps, budget // steps


def run_reference(args, cfg, rank, world):
    from oracle import oracle as O
    from paper_2511_14955_b200 import synth as S

    if rank != 0:
        return 0
    try:
        L = O.ref()
        kind = "reference"
        cores = int(L.igref_hardware_concurrency())
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"reference build missing: {e}"}))
        return 0
    steps, per = ref_plan(args, cfg)
    # warm-up: complete runs on a small sample (pages in the library and the
    # allocator); the timed steps are the spread samples
    wdata, woff = S.generate(cfg, 0, 1)
    wdata, woff = wdata[:1 << 20], np.minimum(woff, 1 << 20).astype(np.uint64)
    for _ in range(args.warmup):
        O.ref_run(wdata, woff, cfg.n, cfg.k, cfg.z, cfg.mode, 0)
    nbytes = 0
    secs = 0.0
    for q, cnt in ref_samples(cfg, steps, per):
        data, off = S.generate(cfg, q, cnt)
        rc, keys, counts, rows, diag, t, err = O.ref_run(data, off, cfg.n, cfg.k, cfg.z,
                                                         cfg.mode, 0)
        if rc != 0:
            print(json.dumps({"impl": "reference", "unavailable": f"reference failed: {err}"}))
            return 0
        nbytes += int(off[-1])
        secs += t
        del data
    v = nbytes / secs / 1e9
    sample = (f"{steps} complete runs, each over ~{per / 2**30:.2f} GiB of whole sequences "
              f"spread evenly over the {cfg.name} corpus ({nbytes} B in total), "
              f"n={cfg.n} k={cfg.k} z={cfg.z} {'once' if cfg.mode == 0 else 'all'}")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": secs / steps * 1e3,
            "higher_is_better": True, "scaling": scaling_of(cfg, args), "vs_baseline": None,
            "dtype": "u8", "data": DATA, "config": config_dict(cfg, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


DATA = "synthetic (seeded generator csrc/synth.c; BASELINE shapes)"


def scaling_of(cfg, args):
    return "weak" if args.weak else "strong"


def config_dict(cfg, world):
    """The workload (identical on both arms)."""
    from paper_2511_14955_b200 import synth as S
    off = S.offsets(cfg)
    return {"workload": f"{cfg.name}: {cfg.describe()}", "n": cfg.n, "k": cfg.k, "z": cfg.z,
            "mode": "once" if cfg.mode == 0 else "all", "corpus_bytes": int(off[-1]),
            "sequences": int(off.size - 1), "counting_passes": max(cfg.n, 3) - 2,
            "parallelism": f"dp{world} (whole-sequence shards balanced by bytes)",
            "l2": "inputs larger than L2 (corpus >> 126 MB), no flush needed"}


def cpu_baseline(args, cfg):
    """The reference CPU path (oracle/_ref) timed on this host: one complete
    run over the first spread sample of the reference arm."""
    from oracle import oracle as O
    from paper_2511_14955_b200 import synth as S
    steps, per = ref_plan(args, cfg)
    q, cnt = ref_samples(cfg, steps, per)[0]
    data, off = S.generate(cfg, q, cnt)
    nbytes = int(off[-1])
    try:
        L = O.ref()
        cores = int(L.igref_hardware_concurrency())
        rc, keys, counts, rows, diag, secs, err = O.ref_run(data, off, cfg.n, cfg.k, cfg.z,
                                                            cfg.mode, 0)
        kind = "reference"
        if rc != 0:
            raise RuntimeError(err)
    except Exception as e:  # noqa: BLE001
        log("reference build unavailable, timing the C oracle port:", e)
        t0 = time.perf_counter()
        O.oracle_run(data, off, cfg.n, cfg.k, cfg.z, cfg.mode)
        secs = time.perf_counter() - t0
        kind, cores = "port", 1
    return {"value": nbytes / secs / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"one complete run over sequences [{q}, {q + cnt}) ({nbytes} B) of "
                      f"{cfg.name}, n={cfg.n} k={cfg.k} z={cfg.z} "
                      f"{'once' if cfg.mode == 0 else 'all'}"}


# ------------------------------------------------------------------ our arm

def pipelined_e2e(args, ig, torch, sess, corpus, icfg, local, coll, bytes_total, world, res):
    """A stream of runs through the public API, `depth` in flight: one session
    per in-flight run (its own stream and HBM buffers), one host thread each.
    Every run still copies its whole corpus H2D and its list D2H; the copy of
    run i+1 overlaps the extension passes of run i.  Device-timed from an
    event after a full synchronize to an event after every run returned."""
    import threading
    depth = args.e2e_depth
    streams = [torch.cuda.Stream() for _ in range(depth - 1)]
    sessions = [sess] + [ig.Session(device=local, stream=s.cuda_stream, collective=coll)
                         for s in streams]
    runs = max(args.steps, depth) * depth
    errors = []

    def worker(i):
        try:
            for _ in range(i, runs, depth):
                r = sessions[i].load_and_run(corpus, icfg, materialize=False)
                if not (np.array_equal(r.keys, res.keys) and np.array_equal(r.counts, res.counts)):
                    errors.append("pipelined run differs")
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    for s in sessions[1:]:
        s.load_and_run(corpus, icfg, materialize=False)  # warm buffers
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    threads = [threading.Thread(target=worker, args=(i,)) for i in range(depth)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    # every load_and_run returns after its stream finished (the list is on the
    # host), so an event recorded after the joins closes the timed region
    ev1 = torch.cuda.Event(enable_timing=True)
    ev1.record()
    torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    for s in sessions[1:]:
        s.close()
    if errors:
        raise RuntimeError("; ".join(errors[:3]))
    ms = ms_total / runs
    te = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    ms = float(te.item())
    return {"value": bytes_total / (ms * 1e-3) / 1e9, "unit": UNIT, "depth": depth,
            "runs": runs, "ms_per_run": ms}


def relaunch_distributed(n):
    """`--gpus N` without a torchrun environment: re-run this command as N
    ranks under torch.distributed.run (one process per GPU, 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    log("relaunching as", n, "ranks:", " ".join(cmd[1:6]))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-bytes", type=int, default=1 << 30,
                    help="corpus bytes the CPU reference processes over its timed steps")
    ap.add_argument("--ref-min-step", type=int, default=256 << 20,
                    help="smallest reference sample per timed step (bytes)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank holds a full-size shard of the generator")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-depth", type=int, default=2,
                    help="runs in flight for e2e.pipelined (1 disables it)")
    ap.add_argument("--seqs", type=int, default=0, help="override sequences per GPU")
    ap.add_argument("--one-shot-runs", type=int, default=2,
                    help="timed calls of the one-shot drop-in entry point (0: skip)")
    ap.add_argument("--collective", default="lib", choices=["lib", "torch"],
                    help="N>1 table all-reduce: the library's own NCCL communicator "
                         "(ig_session_create_nccl) or a torch.distributed hook")
    ap.add_argument("--profile-run", action="store_true",
                    help="load, run once, exit (for ncu captures; prints nothing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    from paper_2511_14955_b200 import synth as S
    cfg = S.CONFIGS[args.config]
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                log(f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}")
                return 2
        return relaunch_distributed(args.gpus)
    if "WORLD_SIZE" in os.environ and args.gpus != world:
        log(f"--gpus {args.gpus} but WORLD_SIZE={world}")
        return 2

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2511_14955_b200 import intergrams as ig

    torch.cuda.set_device(local)
    # IG_BENCH_FORCE_COLLECTIVE=1 (tests): a 1-rank NCCL group with the
    # collective hook installed, to exercise the N>1 plumbing on one GPU
    force_coll = os.environ.get("IG_BENCH_FORCE_COLLECTIVE") == "1"
    if world > 1 or force_coll:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    # ---- this rank's shard.  Strong scaling (default): the config's fixed
    # corpus, whole sequences balanced by bytes.  Weak (--weak): every rank
    # holds `per` sequences of an N-times larger corpus of the same generator.
    off_all = S.offsets(cfg)
    m_all = off_all.size - 1
    if args.weak and cfg.kind != S.K_LOGNORMAL and world > 1:
        per = args.seqs or m_all
        gen_cfg = S.scaled(cfg, num_seqs=per * world)
        first, count = rank * per, per
    else:
        gen_cfg = cfg
        if args.seqs:
            gen_cfg = S.scaled(cfg, num_seqs=args.seqs) if cfg.kind != S.K_LOGNORMAL else cfg
        off_g = S.offsets(gen_cfg)
        first, last = ig.shard_range(off_g, rank, world) if world > 1 else (0, off_g.size - 1)
        if args.seqs and cfg.kind == S.K_LOGNORMAL and world == 1:
            last = min(last, args.seqs)
        count = last - first
    off_gen = S.offsets(gen_cfg)
    t0 = time.time()
    nbytes = int(off_gen[first + count] - off_gen[first])
    host = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
    data, off = S.generate(gen_cfg, first, count, out=host.numpy())
    log(f"rank {rank}: generated {nbytes / 2**30:.2f} GiB ({count} seqs) in {time.time() - t0:.1f}s")
    off_np = np.ascontiguousarray(off, np.uint64)
    # totals over all ranks (count-table widths and the metric's bytes)
    if args.weak and world > 1 and cfg.kind != S.K_LOGNORMAL:
        bytes_total, seqs_total = nbytes * world, count * world
    elif world > 1:
        bytes_total, seqs_total = int(off_gen[-1]), int(off_gen.size - 1)
    else:
        bytes_total, seqs_total = nbytes, count

    stream = torch.cuda.Stream()
    coll, _cb, nccl = None, None, None
    if (world > 1 or force_coll) and args.collective == "lib":
        # the library's own communicator: rank 0's NCCL id goes to every rank
        # over the torch group; forced on one rank, the library runs the
        # collective at world 1 too (a 1-rank all-reduce is the identity)
        if force_coll:
            os.environ["IG_COLLECTIVE_AT_WORLD1"] = "1"
        box = [ig.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        nccl = {"rank": rank, "world": world, "id": box[0], "bytes_total": bytes_total,
                "seqs_total": seqs_total}
    elif world > 1 or force_coll:
        # forced on one rank: the library skips the hook at world 1, so it is
        # told 2; the 1-rank NCCL all-reduce is the identity
        coll, _cb = make_collective(rank, max(world, 2), bytes_total, seqs_total)
    sess = ig.Session(device=local, stream=stream.cuda_stream, collective=coll, nccl=nccl)
    corpus = ig.Corpus(data, off_np)
    sess.load(corpus)
    icfg = ig.IntergramConfig(n=cfg.n, k=cfg.k, z=cfg.z, mode=ig.CountMode(cfg.mode))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if args.profile_run:
        res = sess.run(icfg)
        torch.cuda.synchronize()
        log("profile run:", [(p.label, round(p.seconds * 1e3, 3)) for p in res.passes])
        sess.close()
        return 0

    # ---- device-resident timing
    for _ in range(args.warmup):
        res = sess.run(icfg)
    barrier()
    l0 = sess.launches
    sess.set_profiling(True)  # per-kernel-family CUDA events on the library stream
    sess.kernel_stats(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rows = []
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        step_evs = []
        for _ in range(args.steps):
            res = sess.run(icfg, materialize=False)  # list lands in host numpy arrays
            rows.append(res.passes)
            step_evs.append(torch.cuda.Event(enable_timing=True))
            step_evs[-1].record(stream)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    log("ms of each timed step:", [round(a.elapsed_time(b), 2)
                                   for a, b in zip([ev0] + step_evs[:-1], step_evs)])
    kstats = sess.kernel_stats(reset=True)
    sess.set_profiling(False)
    launches = (sess.launches - l0) // args.steps
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    value = bytes_total / (ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel family.  Every counting kernel
    # (route count / route scatter / count-all) streams this rank's corpus once
    # per launch: algorithmic bytes per launch = corpus bytes.
    peak, peak_src = peaks()
    counting = {f: v for f, v in kstats.items()
                if f in ("route_count", "route_scatter", "count_all", "once_direct") and v[1] > 0}
    dom, (dom_ms, dom_n) = max(counting.items(), key=lambda kv: kv[1][0])
    # count-all splits a pass into < 4 GiB segment launches: normalise to the
    # corpus passes the family covered (one corpus read per counting pass)
    passes_alg = max(cfg.n, 3) - 2
    corpus_passes = dom_n if dom != "count_all" else passes_alg * args.steps
    dom_avg_ms = dom_ms / corpus_passes
    local_bytes = nbytes
    achieved = local_bytes / (dom_avg_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get(f"{cfg.name}:{dom}")
        except Exception:
            traffic = None
    ceiling = None
    cp = os.path.join(ROOT, "profiles", "ceiling.json")
    if os.path.exists(cp):
        try:
            with open(cp) as f:
                ceiling = json.load(f).get(f"{cfg.name}:{dom}")
        except Exception:
            ceiling = None
    step_breakdown = {}
    for step in rows:
        for p in step:
            step_breakdown[p.label] = step_breakdown.get(p.label, 0.0) + p.seconds * 1e3 / len(rows)
    kernel_breakdown = {f: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
                        for f, v in kstats.items() if v[1]}

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        barrier()
        t_e2e = []
        for i in range(2 + args.steps):
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(stream)
            # H2D of the pinned corpus (pipelined under the dense pass) + run +
            # result list D2H
            r2 = sess.load_and_run(corpus, icfg, materialize=False)
            eb.record(stream)
            eb.synchronize()
            if i >= 2:
                t_e2e.append(ea.elapsed_time(eb))
        e_ms = sum(t_e2e) / len(t_e2e)
        te = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = float(te.item())
        e2e = {"value": bytes_total / (e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(nbytes + off_np.nbytes),
               "d2h_bytes_per_step": int(16 * len(r2.keys)), "ms_per_step": e_ms}
        assert np.array_equal(r2.keys, res.keys) and np.array_equal(r2.counts, res.counts)
        if args.e2e_depth > 1 and world > 1:
            # in-flight sessions on separate host threads would issue their
            # all-reduces on the one default group in a rank-dependent order
            e2e["pipelined"] = {"skipped": "single-rank only (one NCCL group per process)"}
        elif args.e2e_depth > 1:
            # one more session per run in flight: only when its HBM fits
            free, total_mem = torch.cuda.mem_get_info()
            used = total_mem - free
            if free > 1.1 * used * (args.e2e_depth - 1):
                e2e["pipelined"] = pipelined_e2e(args, ig, torch, sess, corpus, icfg, local,
                                                 coll, bytes_total, world, res)
            else:
                e2e["pipelined"] = {"skipped": f"{args.e2e_depth} sessions do not fit in HBM "
                                               f"({used / 2**30:.0f} GiB used per session)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg)

    # ---- the drop-in one-shot call on an ordinary (pageable) host corpus:
    # ig_topk_ngrams = C++ run_intergrams (session, HBM allocation, streamed
    # upload through pinned slabs, run, result copy), wall-clocked per call.
    # The timing session is closed first: the one-shot call allocates its own.
    sess.close()
    sess = None
    if e2e is not None and world == 1 and args.one_shot_runs > 0:
        try:
            pageable = np.array(data, copy=True)
            t_os = []
            for _ in range(args.one_shot_runs):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r3 = ig.run_intergrams(ig.Corpus(pageable, off_np), icfg, materialize=False)
                t_os.append(time.perf_counter() - t0)
            assert np.array_equal(r3.counts, res.counts)
            del pageable
            os_s = sum(t_os) / len(t_os)
            e2e["one_shot"] = {"value": bytes_total / os_s / 1e9, "unit": UNIT,
                               "ms_per_run": os_s * 1e3, "runs": len(t_os),
                               "api": "ig_topk_ngrams (C++ run_intergrams), pageable host "
                                      "corpus, wall clock"}
        except Exception as ex:  # noqa: BLE001
            e2e["one_shot"] = {"skipped": f"{type(ex).__name__}: {str(ex)[:200]}"}

    if rank == 0:
        passes_alg = max(cfg.n, 3) - 2
        cd = config_dict(gen_cfg, world)
        if args.weak and world > 1:
            cd["workload"] += f" (weak scaling: {count} sequences per rank)"
        elif world == 1 and (gen_cfg is not cfg or count != off_gen.size - 1):
            cd["workload"] += f" (reduced: {count} sequences, {nbytes} B)"
            cd["corpus_bytes"], cd["sequences"] = nbytes, count
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": scaling_of(cfg, args), "vs_baseline": None,
            "dtype": "u8", "data": DATA,
            "config": cd,
            "hbm_roofline_frac_full_run": (bytes_total * passes_alg / (ms * 1e-3) / 1e9)
            / (world * peak),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"{dom} (dominant kernel family, {dom_n // args.steps} "
                                   f"launches/step; ms per corpus pass)",
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": local_bytes,
                         "avg_launch_ms": dom_avg_ms},
            "ceiling": ceiling,
            "step_breakdown_ms": step_breakdown,
            "kernel_breakdown": kernel_breakdown,
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
            "collective": ({"backend": "nccl", "owner": "library (ig_session_create_nccl)",
                            "world": world} if nccl is not None else
                           None if coll is None else
                           {"backend": "nccl", "owner": "torch.distributed hook",
                            "world": world, "allreduce_calls": coll.calls[0]}),
            "clocks": clk.summary(),
            "result_digest": hashlib.sha256(
                ig.topk_to_tsv(ig.run_result_topk(res, cfg.n)).encode()).hexdigest()[:16],
            "topk_len": int(len(res.keys)),
        }
        print(json.dumps(line), flush=True)
    if world > 1 or force_coll:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
