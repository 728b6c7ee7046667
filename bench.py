#!/usr/bin/env python
"""Benchmark of the batched LOB hot path (BASELINE.json metric: whole-box messages/s,
ns/message and HBM-roofline fraction at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A *step* is one pass of the whole hot path over one batch: lob_init (a0: empty
books + synthetic L2 seed) followed by lob_process_messages over every book's
1,000-message stream (a1-a11, L2 top-10 after each of the 10 steps of 100).
Inputs are resident in HBM before the timed region; the messages (2.1 GB per GPU
for C4) exceed the 126 MB L2, so no flush is needed between steps.

Multi-GPU (torchrun, one process per GPU): every rank owns its own 65,536 books
(global ids rank*K..), so per-GPU work is fixed ("weak" scaling); there is no
communication on the hot path; NCCL only gathers per-book counters and the max
elapsed time afterwards.

--impl reference times the CPU oracle (the reference arm for this tier) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--books", type=int, default=0,
                    help="override the config's books per GPU (the K sweep of SURVEY.md 8(d))")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l1", action="store_true",
                    help="also write the per-message Level-1 trace (NEXT row N1, lob_process_messages_l1)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every GPU owns the config's books; strong: the config's books are split")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback (B200_PROFILING.md)", 1965.0


def workload_desc(cfg, K):
    return (f"{cfg.name}: {K} books/GPU x capacity {cfg.capacity}, {cfg.n_msgs} {cfg.profile} messages/book "
            f"({cfg.n_steps} steps x {cfg.msgs_per_step}), L2 top-{cfg.l2_levels} per step, "
            f"init L2 seed {cfg.init_levels} levels/side")


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
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    cfg = lobgen.CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    # the oracle needs ~1 s per step for the whole C4 batch on a 16-core host, so each
    # step is the full single-GPU workload; larger configs are capped to keep the run short
    nb = min(cfg.n_books, 65536)
    msgs, init = lobgen.generate(cfg, n_books=nb)
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
    sample = (f"{nb} of {cfg.n_books} books of {cfg.name} ({nb * cfg.n_msgs} messages) per step, "
              f"{args.steps} steps, {cores} threads over books")
    line = {"impl": "reference", "metric": "messages/sec", "value": v, "unit": "msg/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "ns_per_message": 1e9 / v,
            "config": {"workload": workload_desc(cfg, nb), "books": nb, "capacity": cfg.capacity},
            "cpu_baseline": {"value": v, "unit": "msg/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "msg/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- CPU baseline leg
def cpu_baseline(cfg, msgs_h, init_h, seconds, gpu):
    """The oracle as it stands, on the host cores, over a bounded sample of the same
    workload (leading books, growing until ~`seconds` of CPU time).  The oracle's
    outputs for the sampled books are then compared with the GPU's (`gpu`: host copies
    of the exported book, trade log, trade counts, per-step L2 and counters), so every
    bench run is also a full-size parity check on the sample (outside the timed region)."""
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
    return {"value": v, "unit": "msg/s", "cores": cores, "kind": "oracle",
            "sample": f"first {done_books} of {cfg.n_books} books of {cfg.name} "
                      f"({done_books * cfg.n_msgs} messages, {total:.1f} s wall on {cores} threads over books)",
            "parity": {"books": done_books, "outputs": ["book", "trades", "n_trades", "l2", "stats"],
                       "bit_exact": not mism, "mismatched": sorted(mism)}}


# ------------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch.distributed as dist

    from paper_2308_13289_b200 import LobBatch, launch_count
    from paper_2308_13289_b200.shard import gather_rows, reduce_max, reduce_sum, shard_books
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; LOB_DIST_BACKEND=gloo lets several ranks share one GPU to
    # exercise the multi-rank logic on a single-GPU box (NCCL refuses shared GPUs)
    backend = os.environ.get("LOB_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = lobgen.CONFIGS[args.config]
    if args.books > 0:
        cfg = cfg.with_(n_books=args.books)
    book0, K = shard_books(rank, world, cfg.n_books, args.scaling)
    cfg = cfg.with_(n_books=K)
    S, M, L = cfg.n_steps, cfg.msgs_per_step, cfg.l2_levels

    # inputs: generated on the host (seeded by GLOBAL book id), pinned, then resident in HBM
    msgs_h = torch.empty((K, cfg.n_msgs, 8), dtype=torch.int32).pin_memory()
    init_h = torch.empty((K, cfg.init_levels, 4), dtype=torch.int32).pin_memory()
    t0 = time.time()
    lobgen.generate(cfg, book_begin=book0, msgs_out=msgs_h.numpy(), init_out=init_h.numpy())
    gen_s = time.time() - t0
    msgs_d = msgs_h.to(dev)
    init_d = init_h.to(dev)
    l2_d = torch.empty((K, S, L, 4), dtype=torch.int32, device=dev)
    l1_d = torch.empty((K, cfg.n_msgs, 4), dtype=torch.int32, device=dev) if args.l1 else None
    b = LobBatch(K, cfg.capacity, cfg.trades_cap, L, device=dev)
    stream = torch.cuda.current_stream()

    def step(evs=None):
        b.init(init_d, lobgen.INIT_TS, lobgen.INIT_TNS)
        if evs is not None:
            evs[0].record(stream)
        b.process(msgs_d, S, M, l2_out=l2_d, l1=args.l1, l1_out=l1_d)
        if evs is not None:
            evs[1].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    n_launch0 = launch_count()
    torch.cuda.synchronize()
    with sampler:
        start.record(stream)
        for i in range(args.steps):
            step(kev[i])
        end.record(stream)
        torch.cuda.synchronize()
    n_launch = launch_count() - n_launch0
    if world > 1:
        dist.barrier()
    elapsed_ms = reduce_max(start.elapsed_time(end), dev)       # the slowest rank's device time
    kernel_ms = [a.elapsed_time(z) for a, z in kev]

    # per-book counters and the trade counts of the last step (algorithmic bytes)
    st = b.stats()
    _, ntr = b.trades()
    trades_logged = int(ntr.sum().item())
    # NCCL gather of per-book counters + state digests (lob_digest)
    allst = gather_rows(torch.cat([st, b.digest()[:, None]], 1))
    trades_total = reduce_sum(trades_logged, dev)
    stats_sum = allst[:, :10].sum(0).cpu().tolist()
    dg = allst[:, 10].cpu().numpy().view(np.uint64)
    # xor-folds: over every book, and over global books [0, K) -- the latter is the same at
    # every world size (each book's stream depends only on its global id)
    digest = {"all_books": "%016x" % int(np.bitwise_xor.reduce(dg)),
              "first_books": "%016x" % int(np.bitwise_xor.reduce(dg[:cfg.n_books])),
              "first_books_n": cfg.n_books}
    total_books = reduce_sum(K, dev)

    total_msgs = total_books * cfg.n_msgs * args.steps
    value = total_msgs / (elapsed_ms / 1e3)
    ms_per_step = elapsed_ms / args.steps

    # roofline of the dominant kernel (lob_step): algorithmic bytes per launch
    book_bytes = 2 * K * 2 * cfg.capacity * LOGICAL_ORDER_BYTES     # state read + written once
    alg_bytes = (K * cfg.n_msgs * MSG_BYTES + trades_logged * TRADE_BYTES + K * S * L * L2_LEVEL_BYTES
                 + book_bytes + 2 * K * STAT_BYTES + (K * cfg.n_msgs * L2_LEVEL_BYTES if args.l1 else 0))
    kmean_ms = statistics.mean(kernel_ms)
    peak, peak_src, _ = load_peaks()
    achieved = alg_bytes / (kmean_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "kernel": "lobk::lob_step<4,1,4,3> (lob_process_messages; MODE 3 = the 8-CTA/SM build for many-wave batches)",
                "kernel_ms": kmean_ms, "kernel_share_of_step": kmean_ms / ms_per_step,
                "alg_bytes_per_launch": alg_bytes, "alg_bytes_per_msg": alg_bytes / (K * cfg.n_msgs),
                "peak_source": peak_src,
                "note": "HBM fraction as BASELINE.json asks; the kernel is instruction-bound -- the binding "
                        "ceilings are roofline_alu_pipe and roofline_issue (DESIGN.md section 8)"}
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    roofline_issue = None
    roofline_alu_pipe = None
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof)).get(cfg.name)
            if tr:
                roofline["traffic"] = tr["dram_bytes_per_launch"]
                roofline["traffic_source"] = tr["source"]
                # the bound that actually binds: warp-instruction issue
                ipm = tr.get("warp_instructions_per_msg")
                if ipm:
                    _, _, max_mhz = load_peaks()
                    peak_issue = 148 * 4 * max_mhz * 1e6 / 1e12            # warp-instr/ps -> T/s
                    ach = ipm * K * cfg.n_msgs / (kmean_ms / 1e3) / 1e12
                    roofline_issue = {"bound": "alu", "achieved": ach, "peak": peak_issue,
                                      "unit": "Twarp-instr/s", "frac": ach / peak_issue,
                                      "warp_instructions_per_msg": ipm, "source": tr.get("instr_source"),
                                      "peak_derivation": "148 SMs x 4 schedulers x 1 warp-instr/clk x sm_max_mhz"}
                # the ALU pipe (ISETP/SEL/LOP3/IADD3/SHF/IMNMX) issues one warp-instruction
                # every 2 cycles per scheduler: the ceiling that binds first
                apm = tr.get("alu_pipe_instructions_per_msg")
                if apm:
                    peak_alu = 148 * 2 * max_mhz * 1e6 / 1e12
                    ach = apm * K * cfg.n_msgs / (kmean_ms / 1e3) / 1e12
                    roofline_alu_pipe = {"bound": "alu", "achieved": ach, "peak": peak_alu,
                                         "unit": "Twarp-instr/s", "frac": ach / peak_alu,
                                         "alu_pipe_instructions_per_msg": apm, "source": tr.get("instr_source"),
                                         "peak_derivation": "148 SMs x 4 schedulers x 0.5 ALU-pipe warp-instr/clk "
                                                            "(B300_MICROARCH.md: alu rt_SMSP = 2; ncu pct_of_peak agrees) "
                                                            "x sm_max_mhz"}
        except Exception:
            pass

    # end-to-end through the public API with HOST buffers: pinned H2D of the step's
    # messages and L2 seed, processing, D2H of the L2 snapshots and counters
    e2e = None
    if args.e2e_steps > 0:
        h_l2 = torch.empty((K, S, L, 4), dtype=torch.int32).pin_memory()
        h_st = torch.empty((K, 10), dtype=torch.int64).pin_memory()
        e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def e2e_step():
            init_d.copy_(init_h, non_blocking=True)
            b.init(init_d, lobgen.INIT_TS, lobgen.INIT_TNS)
            b.process_host(msgs_h, S, M, h_l2, h_st, msgs_d, l2_d, chunks=8)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e_s.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e_e.record(stream)
        torch.cuda.synchronize()
        et = reduce_max(e_s.elapsed_time(e_e), dev)
        e2e_v = total_books * cfg.n_msgs * args.e2e_steps / (et / 1e3)
        e2e = {"value": e2e_v, "unit": "msg/s",
               "h2d_bytes_per_step": msgs_h.numel() * 4 + init_h.numel() * 4,
               "d2h_bytes_per_step": h_l2.numel() * 4 + h_st.numel() * 8,
               "path": "LobBatch.process_host -> lob_process_messages_host (8 pipelined chunks)"}
        assert torch.equal(h_st, st.cpu()), "end-to-end counters differ from the device run"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tr_d, cnt_d = b.trades()
        gpu = {"stats": st.cpu().numpy(), "book": b.book().cpu().numpy(), "trades": tr_d.cpu().numpy(),
               "n_trades": cnt_d.cpu().numpy(), "l2": l2_d.cpu().numpy()}
        del tr_d
        cpu = cpu_baseline(cfg, msgs_h.numpy(), init_h.numpy(), args.cpu_seconds, gpu)
        del gpu

    if rank == 0:
        line = {"metric": "messages/sec", "value": value, "unit": "msg/s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "ns_per_message": 1e9 / value, "ns_per_message_per_gpu": 1e9 / value * world,
                "config": {"workload": workload_desc(cfg, K), "books_per_gpu": K, "books_total": total_books,
                           "capacity": cfg.capacity, "msgs_per_book": cfg.n_msgs, "n_steps": S,
                           "msgs_per_step": M, "l2_levels": L, "trades_cap": cfg.trades_cap,
                           "profile": cfg.profile, "seed": cfg.seed, "parallelism": f"books sharded x{world}",
                           "l2_flush": "inputs larger than L2 (messages %.2f GB/GPU > 126 MB)"
                                       % (msgs_h.numel() * 4 / 1e9)},
                "roofline": roofline, "roofline_issue": roofline_issue, "roofline_alu_pipe": roofline_alu_pipe, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": n_launch, "digest": digest,
                "clocks": sampler.summary(),
                "totals": dict(zip(["msgs", "bad", "trades", "trades_dropped", "traded_qty", "cancelled_qty",
                                    "unknown_cancels", "add_overflow", "overflow_qty", "market_discarded_qty"],
                                   stats_sum)),
                "trades_logged_last_step": trades_total, "generate_s": gen_s,
                "l1_trace": bool(args.l1)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
