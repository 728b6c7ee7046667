"""World-size-2 CPU (gloo) tests of the multi-GPU host logic: book sharding by global
id, the max-over-ranks timing rule and the post-run gather of per-book counters.
The per-rank engine here is the oracle (no GPU on this box); on the B200 box the
same code paths run with NCCL and the CUDA engine (bench.py)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_13289_b200.shard import gather_rows, reduce_max, reduce_sum, shard_books


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scaling, books, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import lobgen
        import oracle
        cfg = lobgen.CONFIGS["C4"]
        b0, nb = shard_books(rank, world, books, scaling)
        msgs, init = lobgen.generate(cfg, book_begin=b0, n_books=nb, threads=2)
        o = oracle.OracleBatch(nb, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
        o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
        o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
        st = torch.from_numpy(o.stats())
        allst = gather_rows(st)
        t = reduce_max(float(rank + 1))
        n = reduce_sum(nb * cfg.n_msgs)
        if rank == 0:
            q.put((allst.numpy(), t, n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scaling,books", [("weak", 24), ("strong", 37)])
def test_two_ranks_match_single_process(scaling, books):
    import lobgen
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scaling, books, q)) for r in range(world)]
    for p in procs:
        p.start()
    allst, t, n = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    total = books * world if scaling == "weak" else books
    cfg = lobgen.CONFIGS["C4"]
    msgs, init = lobgen.generate(cfg, n_books=total, threads=4)
    o = oracle.OracleBatch(total, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    np.testing.assert_array_equal(allst, o.stats())   # sharding invariance
    assert t == 2.0                                   # max over ranks, not rank 0's time
    assert n == total * cfg.n_msgs


def test_shard_ranges():
    assert shard_books(0, 1, 65536) == (0, 65536)
    assert [shard_books(r, 4, 65536) for r in range(4)] == [(r * 65536, 65536) for r in range(4)]
    rs = [shard_books(r, 8, 65539, "strong") for r in range(8)]
    assert sum(n for _, n in rs) == 65539
    assert all(rs[i][0] + rs[i][1] == rs[i + 1][0] for i in range(7))
    with pytest.raises(ValueError):
        shard_books(2, 2, 10)


def _bench(args, env_extra):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_extra)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, env=env, capture_output=True,
                         text=True, timeout=300)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    return out.returncode, [json.loads(l) for l in lines], out.stderr


@pytest.mark.parametrize("n", [2, 3])
def test_bench_spawns_its_own_ranks(n):
    """`bench.py --gpus N` without torchrun re-launches itself with N ranks (one process
    per GPU) under torch.distributed.run; every rank checks WORLD_SIZE == N; rank 0 alone
    prints.  Dry run: gloo, no GPU work."""
    rc, lines, err = _bench(["--gpus", str(n)], {"LOB_BENCH_DRYRUN": "1", "LOB_DIST_BACKEND": "gloo"})
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, lines
    assert lines[0]["n_gpus"] == n and lines[0]["communicator_size"] == n
    assert lines[0]["rank_sum"] == n * (n - 1) // 2


def test_bench_refuses_world_size_mismatch():
    """A launcher that starts fewer ranks than --gpus asks for is an error, not a silent
    one-GPU measurement."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LOB_BENCH_DRYRUN="1", WORLD_SIZE="1", RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4"], env=env,
                         capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "one rank per GPU" in out.stderr


def test_bench_config_dicts_match_between_arms():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import lobgen
    for argv in (["--gpus", "1"], ["--gpus", "8", "--scaling", "strong"], ["--gpus", "2", "--books", "1000"]):
        a = bench.parse(argv)
        cfg = lobgen.CONFIGS[a.config]
        c = bench.config_dict(cfg, a, a.gpus)
        assert c["books_total"] == (c["books_per_gpu"] * a.gpus if a.scaling == "weak" else
                                    (a.books or cfg.n_books))
    a = bench.parse(["--gpus", "8", "--scaling", "strong"])
    assert bench.config_dict(lobgen.CONFIGS["C4"], a, 8)["books_per_gpu"] == 8192
