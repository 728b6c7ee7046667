#!/usr/bin/env python
"""Benchmark of the batched LOB hot path (BASELINE.json metric: whole-box messages/s,
ns/message and HBM-roofline fraction at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--scaling weak|strong]
                    [--impl reference]

A *step* is one pass of the whole hot path over one batch: lob_init (a0: empty
books + synthetic L2 seed) followed by lob_process_messages over every book's
1,000-message stream (a1-a11, L2 top-10 after each of the 10 steps of 100).
Inputs are resident in HBM before the timed region; the messages (2.1 GB per GPU
for C4) exceed the 126 MB L2, so no flush is needed between steps.

Multi-GPU: one process per GPU.  `--gpus N` without an enclosing torchrun
re-launches itself under `torch.distributed.run` with N ranks; every rank checks
that the world size equals N.  Books are independent, so the
path shards with no communication: rank r owns a contiguous range of GLOBAL book
ids (shard.py).  `--scaling weak` (default): every rank owns the config's 65,536
books; `strong`: the config's books are split (C4: 8,192 per GPU at N = 8).  At
N > 1 the line also carries the other scaling mode (`scaling_alt`).  NCCL is used
only after the timed regions: max of per-rank device times, gathers of per-book
counters and digests, and the parity mismatch count.

Parity in every line: each rank replays a sample of ITS OWN books on the CPU oracle
after the timed region and compares book, trade log, trade counts, per-step L2 and
counters element by element, and the device per-book digests (lob_digest) with the
host FNV of the oracle's state; the mismatch counts are summed over ranks.

--impl reference times the CPU oracle (the reference arm for this tier) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import lobgen  # noqa: E402

LOGICAL_ORDER_BYTES = 24   # Eq.2: 6 x int32
MSG_BYTES = 32             # Eq.6: 8 x int32
TRADE_BYTES = 24           # Eq.3: 6 x int32
L2_LEVEL_BYTES = 16        # [ask_p, ask_q, bid_p, bid_q]
STAT_BYTES = 80            # 10 x int64
STAT_KEYS = ["msgs", "bad", "trades", "trades_dropped", "traded_qty", "cancelled_qty",
             "unknown_cancels", "add_overflow", "overflow_qty", "market_discarded_qty"]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--books", type=int, default=0,
                    help="override the config's books (per GPU when weak, total when strong; SURVEY.md 8(d) K sweep)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="pipelined H2D / compute / D2H chunks (0: LobBatch.process_host's default)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--core-seconds", type=float, default=3.0,
                    help="CPU seconds of the one-core oracle sample (cpu_baseline.per_core)")
    ap.add_argument("--parity-books", type=int, default=1024,
                    help="books per rank replayed on the oracle after the timed region")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other scaling mode at N > 1")
    ap.add_argument("--l1", action="store_true",
                    help="also write the per-message Level-1 trace (NEXT row N1, lob_process_messages_l1)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every GPU owns the config's books; strong: the config's books are split")
    return ap.parse_args(argv)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback (B200_PROFILING.md)", 1965.0


def books_of(cfg, args, world):
    """(books per GPU of rank 0, total books) for the run's scaling mode."""
    n = args.books if args.books > 0 else cfg.n_books
    if args.scaling == "weak":
        return n, n * world
    return -(-n // world), n


def config_dict(cfg, args, world, scaling=None):
    """The `config` object of the JSON line -- identical in both arms for the same arguments."""
    scaling = scaling or args.scaling
    n = args.books if args.books > 0 else cfg.n_books
    per, total = (n, n * world) if scaling == "weak" else (-(-n // world), n)
    return {"workload": (f"{cfg.name}: {per} books/GPU x capacity {cfg.capacity}, {cfg.n_msgs} {cfg.profile} "
                         f"messages/book ({cfg.n_steps} steps x {cfg.msgs_per_step}), L2 top-{cfg.l2_levels} "
                         f"per step, init L2 seed {cfg.init_levels} levels/side"),
            "books_per_gpu": per, "books_total": total, "capacity": cfg.capacity, "msgs_per_book": cfg.n_msgs,
            "n_steps": cfg.n_steps, "msgs_per_step": cfg.msgs_per_step, "l2_levels": cfg.l2_levels,
            "trades_cap": cfg.trades_cap, "profile": cfg.profile, "seed": cfg.seed,
            "parallelism": f"books sharded x{world} ({scaling})",
            "l2_flush": "inputs larger than L2 (messages %.2f GB/GPU > 126 MB)" % (per * cfg.n_msgs * MSG_BYTES / 1e9)}


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover - no NVML
            self.err = str(exc)
        self._stop = threading.Event()

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._sample()                     # warm NVML outside the region ...
            self.samples.clear()
            self.reasons.clear()
            # ... and let the sampler thread in often while the host enqueues
            self._sw = sys.getswitchinterval()
            sys.setswitchinterval(0.0005)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._sample()                     # at least one sample at the end of the region
            self._stop.set()
            self.t.join()
            sys.setswitchinterval(self._sw)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ launching
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args, argv):
    """`--gpus N` outside torchrun: re-launch this script with N ranks (one process per
    GPU) under torch.distributed.run; returns its exit code."""
    backend = os.environ.get("LOB_DIST_BACKEND", "nccl")
    if args.impl == "ours" and backend == "nccl" and os.environ.get("LOB_BENCH_DRYRUN") != "1":
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} GPUs, {have} visible "
                                       "(LOB_DIST_BACKEND=gloo lets ranks share a GPU)"}), flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    import oracle
    cfg = lobgen.CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    # the oracle needs ~1 s per step for the whole C4 batch on a 16-core host, so each
    # step is one GPU's workload (capped at 65,536 books to keep the run short)
    per, _ = books_of(cfg, args, world)
    nb = min(per, 65536)
    msgs, init = lobgen.generate(cfg.with_(n_books=nb))
    o = oracle.OracleBatch(nb, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=cores)

    def step():
        o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
        o.process(msgs, cfg.n_steps, cfg.msgs_per_step)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    n = nb * cfg.n_msgs * args.steps
    v = n / dt
    sample = (f"{nb} books of {cfg.name} ({nb * cfg.n_msgs} messages) per step, "
              f"{args.steps} steps, {cores} threads over books")
    line = {"impl": "reference", "metric": "messages/sec", "value": v, "unit": "msg/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "ns_per_message": 1e9 / v, "config": config_dict(cfg, args, world),
            "cpu_baseline": {"value": v, "unit": "msg/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "msg/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- CPU baseline leg
def cpu_baseline(cfg, msgs_h, init_h, seconds, core_seconds, gpu):
    """The oracle as it stands, on the host cores, over a bounded sample of the same
    workload (leading books, growing until ~`seconds` of CPU time).  The oracle's
    outputs for the sampled books are then compared with the GPU's (`gpu`: host copies
    of the exported book, trade log, trade counts, per-step L2 and counters), so every
    bench run is also a full-size parity check on the sample (outside the timed region).
    `per_core`: the same oracle on ONE pinned core (the first core of the affinity set)
    over the leading books, ~`core_seconds` of work."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    nb, done_books, total = 512, 0, 0.0
    mism = set()
    while total < seconds and done_books < cfg.n_books:
        n = min(nb, cfg.n_books - done_books)
        sl = slice(done_books, done_books + n)
        o = oracle.OracleBatch(n, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=cores)
        m = np.ascontiguousarray(msgs_h[sl])
        i = np.ascontiguousarray(init_h[sl])
        t0 = time.perf_counter()
        o.init(i, lobgen.INIT_TS, lobgen.INIT_TNS)
        l2 = o.process(m, cfg.n_steps, cfg.msgs_per_step)
        total += time.perf_counter() - t0
        tr, cnt = o.trades()
        for key, want in (("stats", o.stats()), ("book", o.book()), ("trades", tr), ("n_trades", cnt), ("l2", l2)):
            if not np.array_equal(want, gpu[key][sl]):
                mism.add(key)
        done_books += n
        nb *= 2
    v = done_books * cfg.n_msgs / total
    out = {"value": v, "unit": "msg/s", "cores": cores, "kind": "oracle",
           "sample": f"first {done_books} of {cfg.n_books} books of {cfg.name} "
                     f"({done_books * cfg.n_msgs} messages, {total:.1f} s wall on {cores} threads over books)",
           "parity": {"books": done_books, "outputs": ["book", "trades", "n_trades", "l2", "stats"],
                      "bit_exact": not mism, "mismatched": sorted(mism)}}
    # one core: this thread pinned to a single CPU, oracle threads = 1
    old = os.sched_getaffinity(0)
    core = min(old)
    try:
        os.sched_setaffinity(0, {core})
        nb, done, t1 = 64, 0, 0.0
        while t1 < core_seconds and done < cfg.n_books:
            n = min(nb, cfg.n_books - done)
            sl = slice(done, done + n)
            o = oracle.OracleBatch(n, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=1)
            m = np.ascontiguousarray(msgs_h[sl])
            i = np.ascontiguousarray(init_h[sl])
            t0 = time.perf_counter()
            o.init(i, lobgen.INIT_TS, lobgen.INIT_TNS)
            o.process(m, cfg.n_steps, cfg.msgs_per_step)
            t1 += time.perf_counter() - t0
            done += n
            nb *= 2
    finally:
        os.sched_setaffinity(0, old)
    out["per_core"] = {"value": done * cfg.n_msgs / t1, "unit": "msg/s", "cores": 1, "core": core,
                       "sample": f"first {done} books of {cfg.name} ({done * cfg.n_msgs} messages, "
                                 f"{t1:.1f} s on one pinned core)"}
    return out


# ------------------------------------------------------------------------ our arm
def init_dist(args):
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: one rank per GPU is required")
    # one process per GPU; LOB_DIST_BACKEND=gloo lets several ranks share one GPU to
    # exercise the multi-rank logic on a single-GPU box (NCCL refuses shared GPUs)
    backend = os.environ.get("LOB_DIST_BACKEND", "nccl") if world > 1 else None
    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise SystemExit("bench.py: no CUDA device (there is no CPU fallback)")
    if backend == "nccl" and ndev < world:
        raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, {ndev} visible")
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        assert dist.get_world_size() == args.gpus, (dist.get_world_size(), args.gpus)
    return world, rank, local, dev, backend


class Phase:
    """One timed measurement: this rank's shard of `cfg` resident in HBM, W warm-up
    steps, then K steps bracketed by barriers + synchronize, device time max over ranks."""

    def __init__(self, args, cfg, scaling, world, rank, dev):
        from paper_2308_13289_b200 import LobBatch
        from paper_2308_13289_b200.shard import shard_books
        self.args, self.world, self.rank, self.dev = args, world, rank, dev
        n = args.books if args.books > 0 else cfg.n_books
        self.book0, K = shard_books(rank, world, n, scaling)
        self.cfg = cfg.with_(n_books=K)
        self.K, self.scaling = K, scaling
        c = self.cfg
        S, M, L = c.n_steps, c.msgs_per_step, c.l2_levels
        # inputs: generated on the host (seeded by GLOBAL book id), pinned, then resident in HBM
        self.msgs_h = torch.empty((K, c.n_msgs, 8), dtype=torch.int32).pin_memory()
        self.init_h = torch.empty((K, c.init_levels, 4), dtype=torch.int32).pin_memory()
        t0 = time.time()
        lobgen.generate(c, book_begin=self.book0, msgs_out=self.msgs_h.numpy(), init_out=self.init_h.numpy())
        self.gen_s = time.time() - t0
        self.msgs_d = self.msgs_h.to(dev)
        self.init_d = self.init_h.to(dev)
        self.l2_d = torch.empty((K, S, L, 4), dtype=torch.int32, device=dev)
        self.l1_d = torch.empty((K, c.n_msgs, 4), dtype=torch.int32, device=dev) if args.l1 else None
        self.b = LobBatch(K, c.capacity, c.trades_cap, L, device=dev)

    def step(self, stream, evs=None):
        c = self.cfg
        self.b.init(self.init_d, lobgen.INIT_TS, lobgen.INIT_TNS)
        if evs is not None:
            evs[0].record(stream)
        self.b.process(self.msgs_d, c.n_steps, c.msgs_per_step, l2_out=self.l2_d, l1=self.args.l1,
                       l1_out=self.l1_d)
        if evs is not None:
            evs[1].record(stream)

    def run(self, local):
        import torch.distributed as dist
        from paper_2308_13289_b200 import launch_count
        from paper_2308_13289_b200.shard import reduce_max, reduce_sum
        args = self.args
        stream = torch.cuda.current_stream()
        for _ in range(max(3, args.warmup)):
            self.step(stream)
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.sampler = ClockSampler(local)
        n_launch0 = launch_count()
        torch.cuda.synchronize()
        with self.sampler:
            start.record(stream)
            for i in range(args.steps):
                self.step(stream, kev[i])
            end.record(stream)
            while not end.query():             # poll (GIL released in sleep) so the clock
                time.sleep(0.0005)             # sampler runs during the device work
            torch.cuda.synchronize()
        self.n_launch = launch_count() - n_launch0
        if self.world > 1:
            dist.barrier()
        self.elapsed_ms = reduce_max(start.elapsed_time(end), self.dev)   # the slowest rank's device time
        self.kernel_ms = [a.elapsed_time(z) for a, z in kev]
        self.total_books = reduce_sum(self.K, self.dev)
        self.value = self.total_books * self.cfg.n_msgs * args.steps / (self.elapsed_ms / 1e3)
        self.ms_per_step = self.elapsed_ms / args.steps
        return self

    def digests(self):
        """Per-book counters + device digests of every rank (NCCL gather), xor-folded: over
        all books and over global books [0, n) -- the latter is the same at every world size
        and scaling mode, because each book's stream depends only on its global id."""
        from paper_2308_13289_b200.shard import gather_rows
        allst = gather_rows(torch.cat([self.b.stats(), self.b.digest()[:, None]], 1))
        dg = allst[:, 10].cpu().numpy().view(np.uint64)
        n = self.args.books if self.args.books > 0 else lobgen.CONFIGS[self.args.config].n_books
        self.stats_sum = allst[:, :10].sum(0).cpu().tolist()
        return {"all_books": "%016x" % int(np.bitwise_xor.reduce(dg)),
                "first_books": "%016x" % int(np.bitwise_xor.reduce(dg[:n])), "first_books_n": int(min(n, len(dg)))}

    def parity(self, n_books):
        """This rank's sample of its own books replayed on the CPU oracle, compared element
        by element (book, trade log, counts, per-step L2, counters) and by digest; mismatch
        counts summed over ranks."""
        import oracle
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from digest import state_digest
        from paper_2308_13289_b200.shard import reduce_sum
        K, c = self.K, self.cfg
        rng = np.random.default_rng(1234 + self.book0)
        m = min(n_books, K)
        idx = np.unique(np.concatenate([[0, K - 1], rng.choice(K, m, replace=False)])) if K else np.zeros(0, int)
        cores = max(1, len(os.sched_getaffinity(0)) // self.world)
        o = oracle.OracleBatch(len(idx), c.capacity, c.trades_cap, c.l2_levels, threads=cores)
        o.init(np.ascontiguousarray(self.init_h.numpy()[idx]), lobgen.INIT_TS, lobgen.INIT_TNS)
        l2o = o.process(np.ascontiguousarray(self.msgs_h.numpy()[idx]), c.n_steps, c.msgs_per_step)
        tro, cnto = o.trades()
        want = {"book": o.book(), "trades": tro, "n_trades": cnto, "l2": l2o, "stats": o.stats()}
        ti = torch.from_numpy(idx).to(self.dev)
        tr, cnt = self.b.trades()
        got = {"book": self.b.book()[ti], "trades": tr[ti], "n_trades": cnt[ti], "l2": self.l2_d[ti],
               "stats": self.b.stats()[ti]}
        bad = {k: int((got[k].cpu().numpy() != want[k]).any(axis=tuple(range(1, want[k].ndim))).sum())
               if want[k].ndim > 1 else int((got[k].cpu().numpy() != want[k]).sum()) for k in want}
        dg = self.b.digest()[ti].cpu().numpy().view(np.uint64)
        bad["digest"] = int((dg != state_digest(want["book"], want["trades"], want["n_trades"], want["stats"])).sum())
        keys = sorted(bad)
        tot = [reduce_sum(bad[k], self.dev) for k in keys]
        nb = reduce_sum(len(idx), self.dev)
        mism = {k: v for k, v in zip(keys, tot) if v}
        return {"books": nb, "ranks": self.world, "per_rank": len(idx), "bit_exact": not mism,
                "mismatched_books": mism, "outputs": ["book", "trades", "n_trades", "l2", "stats", "digest"],
                "how": "each rank replays a seeded sample of its own books on the CPU oracle after the timed region"}


def roofline(ph, args, build_id):
    """HBM roofline of the dominant kernel (lob_step): algorithmic bytes per launch / the
    kernel's mean CUDA-event time; plus the issue and ALU-pipe ceilings from the committed
    per-message instruction counts, marked stale when they were measured on another build."""
    c, K = ph.cfg, ph.K
    S, L = c.n_steps, c.l2_levels
    _, ntr = ph.b.trades()
    trades_logged = int(ntr.sum().item())
    book_bytes = 2 * K * 2 * c.capacity * LOGICAL_ORDER_BYTES     # state read + written once
    alg_bytes = (K * c.n_msgs * MSG_BYTES + trades_logged * TRADE_BYTES + K * S * L * L2_LEVEL_BYTES
                 + book_bytes + 2 * K * STAT_BYTES + (K * c.n_msgs * L2_LEVEL_BYTES if args.l1 else 0))
    kmean_ms = statistics.mean(ph.kernel_ms)
    peak, peak_src, max_mhz = load_peaks()
    achieved = alg_bytes / (kmean_ms / 1e3) / 1e9
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": None, "kernel": "lobk::lob_step (lob_process_messages; C4 launches MODE 3 = the 8-CTA/SM "
                                      "build for many-wave batches)",
           "kernel_ms": kmean_ms, "kernel_share_of_step": kmean_ms / ph.ms_per_step,
           "alg_bytes_per_launch": alg_bytes, "alg_bytes_per_msg": alg_bytes / max(1, K * c.n_msgs),
           "peak_source": peak_src,
           "note": "HBM fraction as BASELINE.json asks; the kernel is instruction-bound -- the binding "
                   "ceilings are roofline_alu_pipe and roofline_issue (DESIGN.md section 8)"}
    issue = alu = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    tr = json.load(open(prof)).get(c.name) if os.path.exists(prof) else None
    if tr:
        stale = tr.get("build_id") != build_id
        prov = {"profiled_build_id": tr.get("build_id"), "loaded_build_id": build_id, "stale": stale}
        out["traffic"] = tr["dram_bytes_per_launch"] / tr.get("books", K) * K
        out["traffic_source"] = tr["source"]
        out["traffic_provenance"] = prov
        ipm = tr.get("warp_instructions_per_msg")
        if ipm:
            peak_issue = 148 * 4 * max_mhz * 1e6 / 1e12
            ach = ipm * K * c.n_msgs / (kmean_ms / 1e3) / 1e12
            issue = {"bound": "alu", "achieved": ach, "peak": peak_issue, "unit": "Twarp-instr/s",
                     "frac": ach / peak_issue, "warp_instructions_per_msg": ipm, "source": tr.get("instr_source"),
                     "peak_derivation": "148 SMs x 4 schedulers x 1 warp-instr/clk x sm_max_mhz", **prov}
        apm = tr.get("alu_pipe_instructions_per_msg")
        if apm:
            peak_alu = 148 * 2 * max_mhz * 1e6 / 1e12
            ach = apm * K * c.n_msgs / (kmean_ms / 1e3) / 1e12
            alu = {"bound": "alu", "achieved": ach, "peak": peak_alu, "unit": "Twarp-instr/s",
                   "frac": ach / peak_alu, "alu_pipe_instructions_per_msg": apm, "source": tr.get("instr_source"),
                   "peak_derivation": "148 SMs x 4 schedulers x 0.5 ALU-pipe warp-instr/clk "
                                      "(B300_MICROARCH.md: alu rt_SMSP = 2; ncu pct_of_peak agrees) x sm_max_mhz",
                   **prov}
    return out, issue, alu, trades_logged


def e2e(ph, args):
    """End to end through the public API with HOST buffers: pinned H2D of the step's
    messages and L2 seed, processing, D2H of the per-step L2 snapshots, the counters, the
    logged trade rows (packed) and their per-book counts."""
    import torch.distributed as dist
    from paper_2308_13289_b200.shard import reduce_max, reduce_sum
    c, K, b = ph.cfg, ph.K, ph.b
    S, M, L = c.n_steps, c.msgs_per_step, c.l2_levels
    h_l2 = torch.empty((K, S, L, 4), dtype=torch.int32).pin_memory()
    h_st = torch.empty((K, 10), dtype=torch.int64).pin_memory()
    h_tr = torch.empty((K * c.trades_cap, 6), dtype=torch.int32).pin_memory()
    h_cnt = torch.empty((K,), dtype=torch.int32).pin_memory()
    stream = torch.cuda.current_stream()
    e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def e2e_step():
        ph.init_d.copy_(ph.init_h, non_blocking=True)
        b.init(ph.init_d, lobgen.INIT_TS, lobgen.INIT_TNS)
        b.process_host(ph.msgs_h, S, M, h_l2, h_st, ph.msgs_d, ph.l2_d, chunks=args.e2e_chunks or None, h_trades_out=h_tr,
                       h_trade_counts_out=h_cnt)

    e2e_step()
    torch.cuda.synchronize()
    if ph.world > 1:
        dist.barrier()
    e_s.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e_e.record(stream)
    torch.cuda.synchronize()
    et = reduce_max(e_s.elapsed_time(e_e), ph.dev)
    rows = int(h_cnt.sum())
    v = reduce_sum(K, ph.dev) * c.n_msgs * args.e2e_steps / (et / 1e3)
    # the host outputs are the device path's
    assert torch.equal(h_st, b.stats().cpu()), "end-to-end counters differ from the device run"
    assert torch.equal(h_l2, ph.l2_d.cpu()), "end-to-end L2 differs from the device run"
    tr, cnt = b.trades()
    mask = torch.arange(c.trades_cap, device=ph.dev)[None, :] < cnt[:, None]
    assert torch.equal(h_tr[:rows], tr[mask].cpu()), "end-to-end trade rows differ from the device run"
    # the bound: a plain pinned host->device copy of the same message bytes, timed alike
    h2d = ph.msgs_h.numel() * 4 + ph.init_h.numel() * 4
    c_s, c_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ph.msgs_d.copy_(ph.msgs_h, non_blocking=True)
    c_s.record(stream)
    for _ in range(2):
        ph.msgs_d.copy_(ph.msgs_h, non_blocking=True)
    c_e.record(stream)
    torch.cuda.synchronize()
    copy_gbs = 2 * ph.msgs_h.numel() * 4 / (c_s.elapsed_time(c_e) / 1e3) / 1e9
    achieved_gbs = h2d * args.e2e_steps / (et / 1e3) / 1e9
    return {"value": v, "unit": "msg/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": h_l2.numel() * 4 + h_st.numel() * 8 + rows * TRADE_BYTES + h_cnt.numel() * 4,
            "trade_rows_per_step": rows,
            "path": f"LobBatch.process_host -> lob_process_messages_host ({args.e2e_chunks or min(64, max(1, K // 1024))} pipelined chunks; L2, "
                    "counters, packed logged trade rows + counts to pinned host memory)",
            "pcie": {"bound": "h2d", "achieved_gbs": achieved_gbs, "copy_gbs": copy_gbs,
                     "frac": achieved_gbs / copy_gbs,
                     "note": "the step's input bytes over the e2e step time, against a plain pinned "
                             "host->device copy of the same messages in this run"}}


def clocks_all(sampler, world):
    """Clock summary over ranks: reasons united, the lowest median SM clock."""
    s = sampler.summary()
    if world == 1:
        return s
    import torch.distributed as dist
    allv = [None] * world
    dist.all_gather_object(allv, s)
    reasons = sorted({r for x in allv for r in (x.get("reasons") or [])})
    mhz = [x["sm_mhz"] for x in allv if x.get("sm_mhz")]
    return {"sm_mhz": min(mhz) if mhz else None, "sm_max_mhz": s.get("sm_max_mhz"), "reasons": reasons,
            "samples": sum(x.get("samples", 0) for x in allv), "ranks": world}


def dry_run(args):
    """LOB_BENCH_DRYRUN=1 (CPU test of the launcher): the rank bookkeeping without a GPU --
    the world-size check, a gloo process group and one all-reduce over the ranks."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: one rank per GPU is required")
    ranks = rank
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([rank], dtype=torch.int64)
        dist.all_reduce(t)
        ranks = int(t.item())
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "rank_sum": ranks,
                          "communicator_size": dist.get_world_size() if world > 1 else 1}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args, argv)
    if os.environ.get("LOB_BENCH_DRYRUN") == "1":
        return dry_run(args)
    import torch.distributed as dist

    from paper_2308_13289_b200 import build_id
    world, rank, local, dev, backend = init_dist(args)
    bid = build_id()
    cfg = lobgen.CONFIGS[args.config]

    ph = Phase(args, cfg, args.scaling, world, rank, dev).run(local)
    digest = ph.digests()
    clocks = clocks_all(ph.sampler, world)
    roof, roof_issue, roof_alu, trades_logged = roofline(ph, args, bid)
    from paper_2308_13289_b200.shard import reduce_sum
    trades_total = reduce_sum(trades_logged, dev)
    parity = ph.parity(args.parity_books) if args.parity_books > 0 else None
    e2e_line = e2e(ph, args) if args.e2e_steps > 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tr_d, cnt_d = ph.b.trades()
        gpu = {"stats": ph.b.stats().cpu().numpy(), "book": ph.b.book().cpu().numpy(), "trades": tr_d.cpu().numpy(),
               "n_trades": cnt_d.cpu().numpy(), "l2": ph.l2_d.cpu().numpy()}
        del tr_d
        cpu = cpu_baseline(ph.cfg, ph.msgs_h.numpy(), ph.init_h.numpy(), args.cpu_seconds, args.core_seconds, gpu)
        del gpu

    alt = None
    if world > 1 and not args.no_alt:   # the other scaling mode, same ranks
        other = "strong" if args.scaling == "weak" else "weak"
        n_launch, stats_sum = ph.n_launch, ph.stats_sum
        del ph.b, ph.msgs_d
        torch.cuda.empty_cache()
        pa = Phase(args, cfg, other, world, rank, dev).run(local)
        alt = {"scaling": other, "value": pa.value, "unit": "msg/s", "ms_per_step": pa.ms_per_step,
               "books_per_gpu_rank0": pa.K, "books_total": pa.total_books, "steps": args.steps,
               "kernel_ms_mean": statistics.mean(pa.kernel_ms), "digest": pa.digests(),
               "config": config_dict(cfg, args, world, other),
               "parity": pa.parity(max(64, args.parity_books // 4)) if args.parity_books > 0 else None}
        ph.n_launch, ph.stats_sum = n_launch, stats_sum

    if rank == 0:
        line = {"metric": "messages/sec", "value": ph.value, "unit": "msg/s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ph.ms_per_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "ns_per_message": 1e9 / ph.value, "ns_per_message_per_gpu": 1e9 / ph.value * world,
                "config": config_dict(cfg, args, world),
                "dist": {"backend": backend, "world_size": world,
                         "communicator_size": dist.get_world_size() if world > 1 else 1},
                "roofline": roof, "roofline_issue": roof_issue, "roofline_alu_pipe": roof_alu,
                "cpu_baseline": cpu, "parity": parity, "e2e": e2e_line,
                "gpu_launches": ph.n_launch, "digest": digest, "clocks": clocks,
                "build_id": bid, "scaling_alt": alt,
                "totals": dict(zip(STAT_KEYS, ph.stats_sum)),
                "trades_logged_last_step": trades_total, "generate_s": ph.gen_s,
                "l1_trace": bool(args.l1)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
