#!/usr/bin/env python
"""NEXT row N3 measurement: execution-env steps on the device (the shape of PAPER.md
Table 6): K envs (one book each, N = 100, 10-level initial book), 100
data messages per step, random actions.  Times lob_env_step (one fused launch) eagerly and
as a captured CUDA graph, and as a resident session (lob_session_*: one persistent
launch for the episode, books on chip across steps; K within one wave only); prints one
JSON line."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lobgen  # noqa: E402
from paper_2308_13289_b200 import EnvConfig, LobBatch, LobEnv, LobError, LobSession  # noqa: E402


def run(K, steps=20):
    cfg = lobgen.Config("env", K, 100, steps, 100, 10, 256, 10, "lobster", 7)
    msgs, init = lobgen.generate(cfg)
    b = LobBatch(K, 100, 256, 10)
    ti = torch.from_numpy(init).cuda()
    env = LobEnv(b, EnvConfig(-1, 10**6, 2, 100, 3600, 77, 2_000_000_000, 0, 0.0), 100)
    data = [torch.from_numpy(np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100])).cuda() for s in range(steps)]
    acts = torch.rand((K, 4), device="cuda") * 300
    st = torch.cuda.current_stream()

    def episode():
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
        for s in range(steps):
            env.step(acts, data[s])

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    t_eager = timed(episode)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        episode()
    t_graph = timed(g.replay)
    out = {"envs": K, "steps_per_episode": steps, "data_msgs_per_step": 100}
    res = [("eager", t_eager), ("cuda_graph", t_graph)]
    # resident session: the episode's data up front, one persistent launch; the timed
    # region is the per-step loop (actions copied in, release, wait), as in an RL loop
    dall = torch.cat(data, 1).contiguous()
    zero = torch.zeros_like(acts)
    for name, a in (("session", acts), ("session_zero_actions", zero), ("session_actions_in_place", None)):
        try:
            ts = []
            for _ in range(3):
                b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
                env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
                sess = LobSession(env, dall, steps)
                if a is None:
                    sess.actions.copy_(acts)  # the policy writes its output here
                st.synchronize()  # stream only: a device sync would wait for the resident kernel
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for s in range(steps):
                    sess.step(a)
                e1.record(st)
                sess.end()
                st.synchronize()
                ts.append(e0.elapsed_time(e1))
            res.append((name, sorted(ts)[1]))
        except LobError as ex:
            out[name] = {"unsupported": str(ex)}
    for name, t in res:
        out[name] = {"ms_per_episode": t, "us_per_step": 1e3 * t / steps,
                     "env_steps_per_s": K * steps / (t / 1e3), "data_msgs_per_s": K * steps * 100 / (t / 1e3)}
    return out


if __name__ == "__main__":
    print(json.dumps([run(K) for K in (1000, 2000, 10000)]))
