#!/usr/bin/env python
"""Per-step cost of the resident session vs the per-step fused launch (CUDA graph), at
two data sizes per step (M = 100 and M = 1), 1,000 envs of N = 100: separates the fixed
per-step cost (release / wait, launch, book load / store) from the per-message cost;
then both at M = 100 for larger books (N = 512: 1,000 envs; N = 2048: 400 envs), where
the per-step book load / store the session avoids is larger.  Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lobgen  # noqa: E402
from paper_2308_13289_b200 import EnvConfig, LobBatch, LobEnv, LobSession  # noqa: E402


def run(K, M, steps, N=100):
    cfg = lobgen.Config("env", K, N, steps, M, min(N // 3, 33), 256, 10, "lobster", 7)
    msgs, init = lobgen.generate(cfg)
    b = LobBatch(K, N, 256, 10)
    ti = torch.from_numpy(init).cuda()
    env = LobEnv(b, EnvConfig(-1, 10**6, 2, 100, 3600, 77, 2_000_000_000, 0, 0.0), M)
    dall = torch.from_numpy(msgs).cuda()
    data = [dall[:, s * M:(s + 1) * M].contiguous() for s in range(steps)]
    acts = torch.zeros((K, 4), device="cuda")
    st = torch.cuda.current_stream()
    out = {}

    def graph_episode():
        for s in range(steps):
            env.step(acts, data[s])
    b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
    env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    graph_episode()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graph_episode()
    ts = []
    for _ in range(5):
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["graph_us_per_step"] = 1e3 * sorted(ts)[2] / steps
    ts = []
    for _ in range(5):
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
        sess = LobSession(env, dall, steps)
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for s in range(steps):
            sess.step(None)
        e1.record(st)
        sess.end()
        st.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["session_us_per_step"] = 1e3 * sorted(ts)[2] / steps
    # the same steps captured once into a CUDA graph after begin (no host work per step)
    ts = []
    for _ in range(5):
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
        sess = LobSession(env, dall, steps)
        st.synchronize()
        # capture on a side stream WITHOUT torch.cuda.graph(), whose entry synchronises
        # the device (that would wait for the resident kernel)
        g2 = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(st)
        with torch.cuda.stream(cs):
            g2.capture_begin(capture_error_mode="relaxed")
            for s in range(steps):
                sess.step(None)
            g2.capture_end()
        st.wait_stream(cs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g2.replay()
        e1.record(st)
        sess.end()
        st.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["session_graph_us_per_step"] = 1e3 * sorted(ts)[2] / steps
    return out


if __name__ == "__main__":
    res = {}
    for M in (100, 1):
        res[M] = run(1000, M, 100 if M == 1 else 20)
    t = {k: (res[100][k] - res[1][k]) / 99 for k in res[100]}
    big = {f"N{N}_K{K}_M100": run(K, 100, 20, N) for N, K in ((512, 1000), (2048, 400))}
    print(json.dumps({"N100_K1000_M100": res[100], "N100_K1000_M1": res[1], "per_message_us": t,
                      "fixed_us_per_step": {k: res[1][k] - t[k] for k in t}, **big}))
