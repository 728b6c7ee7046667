#!/usr/bin/env python
"""C2, the paper's RL-environment shape (1,000 books, N = 100, 100 messages per env
step, L2 top-10 after each step): time it three ways.

  mode B        one lob_process_messages call of 100 steps
  mode A eager  100 calls of one step each (what an env.step loop does)
  mode A graph  the same 100 calls captured once in a CUDA graph and replayed

Prints one JSON line; msgs/s counts every book-message.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lobgen  # noqa: E402
from paper_2308_13289_b200 import LobBatch  # noqa: E402


def main():
    cfg = lobgen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    reps = 5
    msgs, init = lobgen.generate(cfg)
    K, S, M, L = cfg.n_books, cfg.n_steps, cfg.msgs_per_step, cfg.l2_levels
    dm = torch.from_numpy(msgs).cuda()
    di = torch.from_numpy(init).cuda()
    steps = [dm[:, s * M:(s + 1) * M].contiguous() for s in range(S)]
    l2 = torch.empty((K, S, L, 4), dtype=torch.int32, device="cuda")
    l2s = [torch.empty((K, 1, L, 4), dtype=torch.int32, device="cuda") for _ in range(S)]
    b = LobBatch(K, cfg.capacity, cfg.trades_cap, L)
    st = torch.cuda.current_stream()

    def mode_b():
        b.init(di, lobgen.INIT_TS, lobgen.INIT_TNS)
        b.process(dm, S, M, l2_out=l2)

    def mode_a():
        b.init(di, lobgen.INIT_TS, lobgen.INIT_TNS)
        for s in range(S):
            b.process(steps[s], 1, M, l2_out=l2s[s])

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {"config": cfg.name, "books": K, "msgs_per_book": cfg.n_msgs}
    tb = timed(mode_b)
    ref_l2 = l2.clone()
    ta = timed(mode_a)
    assert torch.equal(torch.cat(l2s, 1), ref_l2), "mode A differs from mode B"
    g = torch.cuda.CUDAGraph()
    mode_a()  # warm
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        mode_a()
    tg = timed(g.replay)
    assert torch.equal(torch.cat(l2s, 1), ref_l2), "graph replay differs from mode B"
    n = K * cfg.n_msgs
    for name, t in (("mode_B_one_call", tb), ("mode_A_eager", ta), ("mode_A_cuda_graph", tg)):
        out[name] = {"ms": t, "msgs_per_s": n / (t / 1e3), "us_per_env_step": 1e3 * t / S}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
