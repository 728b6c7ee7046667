#!/usr/bin/env python
"""Diagnostic: watch the session's go / done words while a step is pending."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lobgen  # noqa: E402
from paper_2308_13289_b200 import EnvConfig, LobBatch, LobEnv, LobSession, lib  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = lobgen.Config("env", K, 100, 3, 100, 10, 64, 10, "lobster", 3)
msgs, init = lobgen.generate(cfg)
b = LobBatch(K, 100, 64, 10)
b.init(torch.from_numpy(init), 34200, 0)
env = LobEnv(b, EnvConfig(-1, 100, 1, 100, 600, 7, 2_000_000_000, 0, 0.0), 100)
env.reset(34200, 0)
torch.cuda.synchronize()
total = lib().lob_state_bytes(ctypes.byref(b._cfg))
off = b._state_ptr.value - b.state.data_ptr() + total - 256
words = b.state[off:off + 256].view(torch.int32)
side = torch.cuda.Stream()
h = torch.empty(words.numel(), dtype=torch.int32).pin_memory()
caller = torch.cuda.Stream() if os.environ.get("CALLER_SIDE") else torch.cuda.current_stream()
caller.wait_stream(torch.cuda.current_stream())
sess = LobSession(env, torch.from_numpy(msgs), 3, stream=caller)
print("begun", flush=True)
sess.step(None, stream=caller)
print("step enqueued", flush=True)
for i in range(10):
    with torch.cuda.stream(side):
        h.copy_(words, non_blocking=True)
    side.synchronize()
    print(f"t={i * 0.3:.1f}s go={h[0].item():#x} done={h[32].item()}", flush=True)
    time.sleep(0.3)
caller.synchronize()
print("step 1 done", flush=True)
sess.end(stream=caller)
caller.synchronize()
print("ended", flush=True)
