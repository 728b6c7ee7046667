"""NEXT row N3, residency (books resident on chip across env steps, a
persistent kernel for K <~ 7k): the resident env session
(include/lob.h lob_session_*) against the CPU oracle's env, step by step."""
import numpy as np
import pytest
import torch

import lobgen
import oracle
from common import assert_outputs_equal  # noqa: F401  (shared helpers)

# a hung session would block the stream forever: fail the process instead (thread method)
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300, method="thread")]


def _setup(K, N, side, episode, seed, Tcap=512, L=10, steps=12):
    from paper_2308_13289_b200 import EnvConfig, LobBatch, LobEnv
    cfg = lobgen.Config("env", K, N, steps, 100, min(N // 3, 33), Tcap, L, "lobster", seed)
    msgs, init = lobgen.generate(cfg)
    kw = dict(task_side=side, task_size=3000, n_passive=2, tick=100, episode_s=episode, agent_tid=77,
              agent_oid_base=2_000_000_000, reserved=0, lam=0.5)
    b = LobBatch(K, N, Tcap, L)
    b.init(torch.from_numpy(init), lobgen.INIT_TS, lobgen.INIT_TNS)
    env = LobEnv(b, EnvConfig(**kw), 100)
    env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    oe = oracle.OracleBatch(K, N, Tcap, L)
    oe.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    oenv = oracle.OracleEnv(oe, oracle.EnvConfig(side, 3000, 2, 100, episode, 77, 2_000_000_000, 0, 0.5))
    oenv.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    return cfg, msgs, b, env, oe, oenv


def _check_step(s, env, sess, oe, oenv, acts, data, prev):
    r, d, x = sess.step(torch.from_numpy(acts))
    ro, do, xo, am = oenv.step(acts, data, 100)
    np.testing.assert_array_equal(env.work[:, :8].cpu().numpy(), am, err_msg=f"agent msgs step {s}")
    np.testing.assert_array_equal(d.cpu().numpy(), do, err_msg=f"done step {s}")
    np.testing.assert_array_equal(x.cpu().numpy(), xo, err_msg=f"executed step {s}")
    np.testing.assert_array_equal(sess.l2.cpu().numpy(), oe.l2(), err_msg=f"L2 step {s}")
    rg = r.cpu().numpy()
    scale = (xo - prev).astype(np.float64) * 4e6 * 1.5  # eq:rewardfunc's terms (see test_env_rollout_parity)
    assert np.all(np.abs(rg - ro) <= 1e-12 * np.maximum(1.0, scale)), (s, np.abs(rg - ro).max())
    return xo.copy()


@pytest.mark.parametrize("K,N,side,episode", [(1000, 100, -1, 1800), (500, 100, 1, 40), (64, 512, -1, 600),
                                               (24, 2048, 1, 600), (37, 32, -1, 900)])
def test_session_rollout_parity(K, N, side, episode):
    """12 env steps of a resident session with random actions: agent messages, done,
    executed, post-step L2 bit-exact and rewards within 1e-12 of their terms at every
    step; books, counters and the last step's trade log bit-exact after end()."""
    from paper_2308_13289_b200 import LobSession
    cfg, msgs, b, env, oe, oenv = _setup(K, N, side, episode, 60 + K)
    sess = LobSession(env, torch.from_numpy(msgs), cfg.n_steps)
    rng = np.random.default_rng(K)
    prev = np.zeros(K, np.int64)
    for s in range(cfg.n_steps):
        acts = rng.uniform(-100, 600, (K, 4)).astype(np.float32)
        acts[rng.random((K, 4)) < 0.03] = np.nan
        data = np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100])
        prev = _check_step(s, env, sess, oe, oenv, acts, data, prev)
    sess.end()
    np.testing.assert_array_equal(b.book().cpu().numpy(), oe.book())
    np.testing.assert_array_equal(b.stats().cpu().numpy(), oe.stats())
    t, c = b.trades()
    to, co = oe.trades()
    np.testing.assert_array_equal(c.cpu().numpy(), co)
    np.testing.assert_array_equal(t.cpu().numpy(), to)


def test_session_stopped_early_then_env_steps():
    """end() after 5 of 12 steps writes the books back; plain lob_env_step calls then
    continue the episode from them, equal to the oracle."""
    from paper_2308_13289_b200 import LobSession
    K = 300
    cfg, msgs, b, env, oe, oenv = _setup(K, 100, -1, 1800, 5)
    sess = LobSession(env, torch.from_numpy(msgs), cfg.n_steps)
    rng = np.random.default_rng(1)
    prev = np.zeros(K, np.int64)
    for s in range(5):
        acts = rng.uniform(0, 400, (K, 4)).astype(np.float32)
        prev = _check_step(s, env, sess, oe, oenv, acts, np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100]), prev)
    sess.end()
    np.testing.assert_array_equal(b.book().cpu().numpy(), oe.book())
    np.testing.assert_array_equal(b.stats().cpu().numpy(), oe.stats())
    for s in range(5, 8):
        acts = rng.uniform(0, 400, (K, 4)).astype(np.float32)
        data = np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100])
        r, d, x = env.step(torch.from_numpy(acts), torch.from_numpy(data))
        ro, do, xo, am = oenv.step(acts, data, 100)
        np.testing.assert_array_equal(x.cpu().numpy(), xo)
    np.testing.assert_array_equal(b.book().cpu().numpy(), oe.book())


def test_session_on_a_side_stream_and_a_second_session():
    """A session driven from a non-default stream, then a second session on the same
    context (state carried over), equal to the oracle."""
    from paper_2308_13289_b200 import LobSession
    K = 200
    cfg, msgs, b, env, oe, oenv = _setup(K, 100, 1, 1800, 9)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    rng = np.random.default_rng(2)
    prev = np.zeros(K, np.int64)
    half = 6
    first, second = (np.ascontiguousarray(msgs[:, :half * 100]), np.ascontiguousarray(msgs[:, half * 100:]))
    for part, s0 in ((first, 0), (second, half)):
        with torch.cuda.stream(st):
            sess = LobSession(env, torch.from_numpy(part), half, stream=st)
            for s in range(half):
                acts = rng.uniform(0, 300, (K, 4)).astype(np.float32)
                r, d, x = sess.step(torch.from_numpy(acts), stream=st)
                ro, do, xo, am = oenv.step(acts, np.ascontiguousarray(msgs[:, (s0 + s) * 100:(s0 + s + 1) * 100]), 100)
                st.synchronize()
                np.testing.assert_array_equal(x.cpu().numpy(), xo)
                np.testing.assert_array_equal(env.work[:, :8].cpu().numpy(), am)
            sess.end(stream=st)
        st.synchronize()
    np.testing.assert_array_equal(b.book().cpu().numpy(), oe.book())
    np.testing.assert_array_equal(b.stats().cpu().numpy(), oe.stats())


def test_session_errors_and_destroy_while_running():
    from paper_2308_13289_b200 import EnvConfig, LobBatch, LobEnv, LobError, LobSession
    kw = dict(task_side=-1, task_size=100, n_passive=1, tick=100, episode_s=600, agent_tid=7,
              agent_oid_base=2_000_000_000, reserved=0, lam=0.0)
    K = 64
    cfg = lobgen.Config("env", K, 100, 3, 100, 10, 64, 10, "lobster", 3)
    msgs, init = lobgen.generate(cfg)
    b = LobBatch(K, 100, 64, 10)
    b.init(torch.from_numpy(init), lobgen.INIT_TS, lobgen.INIT_TNS)
    env = LobEnv(b, EnvConfig(**kw), 100)
    env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    sess = LobSession(env, torch.from_numpy(msgs), 3)
    with pytest.raises(LobError):  # one session per context
        LobSession(env, torch.from_numpy(msgs), 3)
    acts = torch.full((K, 4), 5.0)
    for _ in range(3):
        sess.step(acts)
    with pytest.raises(LobError):  # the episode's data are exhausted
        sess.step(acts)
    sess.end()
    from paper_2308_13289_b200.lob import _check, lib
    with pytest.raises(LobError):  # no session running
        _check(lib().lob_session_step(b.ctx, None), "lob_session_step")
    # too many books for one wave
    big = LobBatch(200_000, 100, 4, 1)
    big.init(None, 0, 0)
    benv = LobEnv(big, EnvConfig(**kw), 1)
    benv.reset(0, 0)
    with pytest.raises(LobError):
        LobSession(benv, torch.zeros((200_000, 1, 8), dtype=torch.int32), 1)
    # a context destroyed while its session waits for a step stops the kernel.  (While a
    # session runs, only STREAM synchronisation is allowed: a device-wide synchronize
    # would wait for the resident kernel, which waits for the next step.)
    s2 = LobSession(env, torch.from_numpy(msgs), 3)
    s2.step(acts)
    torch.cuda.current_stream().synchronize()
    del s2, env
    b.__del__()
    torch.cuda.synchronize()  # the kernel has exited


def test_session_memops_hook(monkeypatch):
    """The A/B hook LOB_SESSION_MEMOPS=1 (release / wait by the driver's stream memory
    operations instead of the step launch) gives the same results."""
    from paper_2308_13289_b200 import LobSession
    monkeypatch.setenv("LOB_SESSION_MEMOPS", "1")
    K = 100
    cfg, msgs, b, env, oe, oenv = _setup(K, 100, -1, 1800, 11, steps=4)
    sess = LobSession(env, torch.from_numpy(msgs), cfg.n_steps)
    rng = np.random.default_rng(3)
    prev = np.zeros(K, np.int64)
    for s in range(cfg.n_steps):
        acts = rng.uniform(0, 400, (K, 4)).astype(np.float32)
        prev = _check_step(s, env, sess, oe, oenv, acts, np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100]), prev)
    sess.end()
    np.testing.assert_array_equal(b.book().cpu().numpy(), oe.book())


def test_session_steps_in_cuda_graph():
    """A whole episode's steps captured once in a CUDA graph after lob_session_begin (on a
    side stream with capture_begin / capture_end: torch.cuda.graph() would synchronise the
    device, i.e. wait for the resident kernel) and replayed: per-step rewards, executed
    quantities and L2, and the final books equal the oracle env."""
    from paper_2308_13289_b200 import LobSession
    K, S = 200, 6
    cfg, msgs, b, env, oe, oenv = _setup(K, 100, 1, 1800, 21, steps=S)
    rng = np.random.default_rng(8)
    acts_h = [rng.uniform(0, 300, (K, 4)).astype(np.float32) for _ in range(S)]
    acts = [torch.from_numpy(a).cuda() for a in acts_h]
    rew = torch.zeros((S, K), dtype=torch.float64, device="cuda")
    ex = torch.zeros((S, K), dtype=torch.int64, device="cuda")
    l2s = torch.zeros((S, K, 10, 4), dtype=torch.int32, device="cuda")
    cur = torch.cuda.current_stream()
    sess = LobSession(env, torch.from_numpy(msgs), S)
    # every kernel the captured loop uses has run once (lazy module loading, see lob.h)
    sess.actions.copy_(acts[0]); rew[0].copy_(env.reward); ex[0].copy_(env.executed); l2s[0].copy_(sess.l2)
    cs = torch.cuda.Stream()
    cs.wait_stream(cur)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cs):
        g.capture_begin(capture_error_mode="relaxed")
        for s in range(S):
            sess.actions.copy_(acts[s])
            sess.step(None)
            rew[s].copy_(env.reward)
            ex[s].copy_(env.executed)
            l2s[s].copy_(sess.l2)
        g.capture_end()
    cur.wait_stream(cs)
    g.replay()
    sess.end()
    cur.synchronize()
    prev = np.zeros(K, np.int64)
    for s in range(S):
        ro, do, xo, am = oenv.step(acts_h[s], np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100]), 100)
        np.testing.assert_array_equal(ex[s].cpu().numpy(), xo, err_msg=f"executed step {s}")
        np.testing.assert_array_equal(l2s[s].cpu().numpy(), oe.l2(), err_msg=f"L2 step {s}")
        scale = (xo - prev).astype(np.float64) * 4e6 * 1.5
        assert np.all(np.abs(rew[s].cpu().numpy() - ro) <= 1e-12 * np.maximum(1.0, scale)), s
        prev = xo.copy()
    np.testing.assert_array_equal(b.book().cpu().numpy(), oe.book())
