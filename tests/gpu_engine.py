"""Numpy adapter over the CUDA path (LobBatch -> C ABI) with the oracle's engine surface."""
from __future__ import annotations

import numpy as np
import torch

from paper_2308_13289_b200 import LobBatch


class GpuEngine:
    def __init__(self, n_books, capacity, trades_cap=None, l2_levels=10):
        self.b = LobBatch(n_books, capacity, trades_cap, l2_levels)
        self.K = n_books

    def init(self, init_l2=None, init_ts=0, init_tns=0):
        self.b.init(None if init_l2 is None else torch.from_numpy(np.ascontiguousarray(init_l2)),
                    init_ts, init_tns)

    def process(self, msgs, n_steps, msgs_per_step, l2=True, l1=False):
        out = self.b.process(torch.from_numpy(np.ascontiguousarray(msgs, dtype=np.int32)),
                             n_steps, msgs_per_step, l2=l2, l1=l1)
        torch.cuda.synchronize()
        if l1:
            a, b = out
            return (None if a is None else a.cpu().numpy()), b.cpu().numpy()
        return None if out is None else out.cpu().numpy()

    def book(self):
        return self.b.book().cpu().numpy()

    def trades(self):
        t, c = self.b.trades()
        return t.cpu().numpy(), c.cpu().numpy()

    def l2(self):
        return self.b.l2().cpu().numpy()

    def step_reward(self, agent_oids, p_init, side, lam):
        r, v, q = self.b.step_reward(torch.as_tensor(np.asarray(agent_oids, np.int32)),
                                     torch.as_tensor(np.asarray(p_init, np.float64)),
                                     torch.as_tensor(np.asarray(side, np.int32)), lam)
        return r.cpu().numpy(), v.cpu().numpy(), q.cpu().numpy()

    def stats(self):
        return self.b.stats().cpu().numpy()


def make_gpu(N, T_cap, L):
    return GpuEngine(1, N, T_cap, L)
