#!/usr/bin/env python
"""The CPU oracle on ONE core (SURVEY.md 8(d) "oracle timed beside it"): C1 and C2 in
full, a 256-book sample of C3, C4 and each C5 capacity; run under `taskset -c 0` on
the GPU box's host.  Baseline only (never a target).  Prints one JSON document."""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lobgen  # noqa: E402
import oracle  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


out = {"cores": len(os.sched_getaffinity(0)), "cpu": cpu_model(), "configs": {}}
for name, nb in [("C1", None), ("C2", None), ("C3", 256), ("C4", 256), ("C5_32", 256), ("C5_100", 256),
                 ("C5_512", 256), ("C5_2048", 256)]:
    cfg = lobgen.CONFIGS[name]
    n = cfg.n_books if nb is None else min(nb, cfg.n_books)
    msgs, init = lobgen.generate(cfg, n_books=n)
    o = oracle.OracleBatch(n, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=1)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    t0 = time.perf_counter()
    o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    dt = time.perf_counter() - t0
    m = n * cfg.n_msgs
    out["configs"][name] = {"books": n, "messages": m, "seconds": dt, "msgs_per_s": m / dt}
print(json.dumps(out))
