#!/usr/bin/env python
"""Small parity run for compute-sanitizer (memcheck/racecheck/synccheck/initcheck):
every book geometry (W = 1 and W > 1), L2 + L1 outputs, exports, the host path."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import lobgen  # noqa: E402
import oracle  # noqa: E402
from gpu_engine import GpuEngine  # noqa: E402

fails = 0
for N, K, prof in [(100, 9, "lobster"), (33, 5, "garbage"), (200, 3, "heavy_market"), (512, 2, "ties"),
                   (2048, 1, "lobster")]:
    cfg = lobgen.Config("san", K, N, 2, 20, min(N, 10), 16, 4, prof, 3)
    msgs, init = lobgen.generate(cfg)
    g, o = GpuEngine(K, N, 16, 4), oracle.OracleBatch(K, N, 16, 4)
    out = []
    for e in (g, o):
        e.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
        l2, l1 = e.process(msgs, cfg.n_steps, cfg.msgs_per_step, l1=True)
        l2b = e.process(msgs, cfg.n_steps, cfg.msgs_per_step)
        out.append((l2, l1, l2b, e.book(), e.trades()[0], e.l2(), e.stats()))
    ok = all(np.array_equal(a, b) for a, b in zip(*out))
    fails += not ok
    print(N, K, prof, "ok" if ok else "MISMATCH", flush=True)
from paper_2308_13289_b200 import LobBatch  # noqa: E402
cfg = lobgen.CONFIGS["C4"].with_(n_books=40)
msgs, init = lobgen.generate(cfg)
b = LobBatch(40, 100, cfg.trades_cap, 10)
b.init(torch.from_numpy(init).cuda(), lobgen.INIT_TS, lobgen.INIT_TNS)
h = torch.from_numpy(msgs).pin_memory()
hl2 = torch.empty((40, cfg.n_steps, 10, 4), dtype=torch.int32).pin_memory()
htr = torch.empty((40 * cfg.trades_cap, 6), dtype=torch.int32).pin_memory()
hcnt = torch.empty((40,), dtype=torch.int32).pin_memory()
hst = torch.empty((40, 10), dtype=torch.int64).pin_memory()
b.process_host(h, cfg.n_steps, cfg.msgs_per_step, hl2, hst, torch.empty_like(h, device="cuda"),
               torch.empty_like(hl2, device="cuda"), chunks=3, h_trades_out=htr, h_trade_counts_out=hcnt)
torch.cuda.synchronize()
print("host path ok", int(hcnt.sum()), "trade rows")
# NEXT N3: a few env steps (agent messages, data, reward epilogue) in two geometries
from paper_2308_13289_b200 import EnvConfig, LobEnv  # noqa: E402
for N, K in [(100, 9), (2048, 2)]:
    cfg = lobgen.Config("san_env", K, N, 3, 20, min(N // 3, 20), 64, 4, "lobster", 5)
    msgs, init = lobgen.generate(cfg)
    be = LobBatch(K, N, 64, 4)
    be.init(torch.from_numpy(init), lobgen.INIT_TS, lobgen.INIT_TNS)
    env = LobEnv(be, EnvConfig(task_side=-1, task_size=500, n_passive=2, tick=100, episode_s=600, agent_tid=7,
                               agent_oid_base=2_000_000_000, reserved=0, lam=0.5), 20)
    env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    rng = np.random.default_rng(N)
    for s in range(3):
        acts = torch.from_numpy(rng.uniform(0, 300, (K, 4)).astype(np.float32))
        env.step(acts, torch.from_numpy(np.ascontiguousarray(msgs[:, s * 20:(s + 1) * 20])))
    torch.cuda.synchronize()
    print("env", N, "ok")
    # the same steps through a resident session (N3 residency), from the same books
    be.init(torch.from_numpy(init), lobgen.INIT_TS, lobgen.INIT_TNS)
    env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    from paper_2308_13289_b200 import LobSession  # noqa: E402
    sess = LobSession(env, torch.from_numpy(np.ascontiguousarray(msgs[:, :60])), 3)
    rng = np.random.default_rng(N)
    for s in range(3):
        sess.step(torch.from_numpy(rng.uniform(0, 300, (K, 4)).astype(np.float32)))
    sess.end()
    torch.cuda.current_stream().synchronize()
    print("session", N, "ok")
sys.exit(1 if fails else 0)
