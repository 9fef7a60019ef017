"""Device level sums (north_star subsystem 4), residual history through the batch seam, and the
multi-GPU layer of the C-ABI (osc_group / osc_comm) on the B200, all through libosc_b200.so."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan(api, m=32, ell=2, lam=0.1, seed=3):
    prob = api.ProblemSpec(api.CovarianceModel.matern(1.0, lam, 0.5))
    opt = api.EstimatorOptions(seed=seed)
    return prob, opt, api.make_level_plan(ell, 1.0 / (m >> ell), prob, opt)


def _draw_raw(P, lev, prob, opt, ell, frm, to, sums=None, coarse=True):
    api, L = P.api, P._lib
    n = to - frm
    qf, qc = np.empty(n), np.empty(n)
    st = np.zeros(n, dtype=np.int32)
    ps = api._problem_struct(prob, opt.solver)
    rc = L.lib().osc_level_draws(lev.h, C.byref(ps), opt.seed, ell, frm, to, L.DRAW_HAS_COARSE if coarse else 0,
                                 None, qf.ctypes.data, qc.ctypes.data, None, None, st.ctypes.data,
                                 None if sums is None else sums.ctypes.data)
    return rc, qf, qc, st


def _sums(qf, qc, ky, kq):
    y = qf - qc - ky
    q = qf - kq
    return np.array([qf.size, y.sum(), (y * y).sum(), q.sum(), (q * q).sum()])


def test_level_sums_per_call_and_running(P, ctx, port):
    """level_sums of osc_level_draws (per call, shifted) and the level's running device sums over
    several multi-chunk calls equal the slot-order sums of the returned QoIs to 1e-12; the moments
    derived from them equal the reference's Welford (port oo_moments) on the same QoIs, and the QoIs
    equal the port's own draws (1e-7)."""
    api = P.api
    prob, opt, plan = _plan(api)
    lev = plan.op.device_level(ctx, 0)
    ky, kq = 0.01, 0.2  # near the level means (pilot-style shifts)
    ctx.set_mem_budget(3 << 20)  # a few samples per chunk: the sums accumulate across chunks
    try:
        lev.sums_reset(ky, kq)
        allf, allc = [], []
        for frm, to in [(0, 9), (9, 10), (10, 31)]:
            sums = np.zeros(8)
            sums[5], sums[6] = ky, kq
            rc, qf, qc, st = _draw_raw(P, lev, prob, opt, plan.ell, frm, to, sums)
            assert rc == 0 and np.all(st == 0)
            want = _sums(qf, qc, ky, kq)
            assert sums[0] == to - frm
            assert np.allclose(sums[:5], want, rtol=1e-12, atol=1e-14 * np.abs(want).max())
            allf.append(qf)
            allc.append(qc)
        qf, qc = np.concatenate(allf), np.concatenate(allc)
        run = lev.sums_read()
        want = _sums(qf, qc, ky, kq)
        assert run[0] == 31 and run[5] == ky and run[6] == kq
        assert np.allclose(run[:5], want, rtol=1e-12, atol=1e-14 * np.abs(want).max())
    finally:
        ctx.set_mem_budget(0)
    from paper_2306_13493_b200.dist import moments_from_sums
    n, my, vy, mq, vq = moments_from_sums(run[:5], ky, kq)
    o = port.moments(qf, qc, True)
    assert n == o["n"]
    assert abs(my - o["mean_y"]) <= 1e-12 * (abs(o["mean_y"]) + np.sqrt(o["var_y"]))
    assert abs(vy - o["var_y"]) <= 1e-10 * o["var_y"]
    assert abs(mq - o["mean_q"]) <= 1e-12 * abs(o["mean_q"])
    assert abs(vq - o["var_q"]) <= 1e-10 * o["var_q"]
    # the QoIs themselves against the port's draws of the same indices
    sl = np.sqrt(np.maximum(plan.op.eigenvalues, 0))
    pf, pc, _, _ = port.coupled(plan.grid.m(0), plan.op.n, sl, None, True, opt.seed, plan.ell, 0, 31)
    assert np.max(np.abs(qf - pf) / np.abs(pf)) < 1e-7 and np.max(np.abs(qc - pc) / np.abs(pc)) < 1e-7
    # reset restarts; an empty call contributes nothing
    lev.sums_reset(ky, kq)
    sums = np.zeros(8)
    assert _draw_raw(P, lev, prob, opt, plan.ell, 5, 5, sums)[0] == 0
    assert np.all(lev.sums_read()[:5] == 0) and np.all(sums[:5] == 0)


def test_failure_history_through_level_draws(P, ctx):
    """A non-converging batch: OSC_ERR_SOLVER, per-slot status, and (history capture on) the first
    failing slot's residual history, re-solved alone — the reference's SolverError::history."""
    api = P.api
    prob = api.ProblemSpec(api.CovarianceModel.matern(1.0, 0.1, 0.5))
    opt = api.EstimatorOptions(seed=1, solver=api.SolverOptions(max_iter_factor=0))
    plan = api.make_level_plan(1, 1.0 / 32, prob, opt)  # 64² fine / 32² coarse: the streaming solver
    d = api.LevelDraws()
    ctx.set_history(4096)
    try:
        with pytest.raises(api.SolverError) as ei:
            api.run_level_draws(plan, api.GridSpec.square(32), False, False, prob, opt, 3, 7, d, ctx=ctx)
        st = ei.value.status
        assert np.all(st == P._lib.OSC_ERR_SOLVER)
        slot, h = ctx.failure_history()
        assert slot == 3
        h2 = ei.value.residual_history
        assert h2 is not None and np.array_equal(h, h2)
        assert len(h) == 1 and np.isfinite(h[0]) and h[0] > 1e-10  # a zero cap fails before iterating (fem.cpp:374)
    finally:
        ctx.set_history(0)
    # history off: the error still carries the per-slot status, no re-run
    with pytest.raises(api.SolverError):
        api.run_level_draws(plan, api.GridSpec.square(32), False, False, prob, opt, 3, 5, d, ctx=ctx)


def test_group_single_device_matches_context(P, ctx):
    """osc_group over the one visible device: slots, per-call level sums (NCCL all-reduce of the device
    buffers) and the running sums (all-reduce into a separate buffer) equal the single-context path."""
    api = P.api
    prob, opt, plan = _plan(api, m=64, ell=1, seed=6)
    cg = api.GridSpec.square(32)
    a = api.LevelDraws()
    api.run_level_draws(plan, cg, False, False, prob, opt, 0, 21, a, ctx=ctx)
    g = api.DeviceGroup(1)
    try:
        gl = g.level(plan.op, 0)
        gl.sums_reset(0.0, 0.1)
        b = api.LevelDraws()
        sums = np.zeros(8)
        sums[6] = 0.1
        g.run_level_draws(plan, cg, False, False, prob, opt, 0, 21, b, level_sums=sums)
        assert np.array_equal(a.q_fine[:21], b.q_fine[:21]) and np.array_equal(a.q_coarse[:21], b.q_coarse[:21])
        assert np.array_equal(a.iters_fine[:21], b.iters_fine[:21])
        want = _sums(b.q_fine[:21], b.q_coarse[:21], 0.0, 0.1)
        assert np.allclose(sums[:5], want, rtol=1e-12)
        r1 = gl.sums_allreduce()
        r2 = gl.sums_allreduce()  # reducing twice does not double-count
        assert np.allclose(r1[:5], want, rtol=1e-12) and np.array_equal(r1, r2)
        # slots in the middle of a larger vector, and an empty range
        c = api.LevelDraws()
        g.run_level_draws(plan, cg, False, False, prob, opt, 5, 9, c)
        assert np.array_equal(c.q_fine[5:9], a.q_fine[5:9]) and np.all(c.q_fine[:5] == 0)
        g.run_level_draws(plan, cg, False, False, prob, opt, 9, 9, c)
    finally:
        g.close()


def test_comm_single_rank(P, ctx):
    """osc_comm with one rank (NCCL unique id → communicator on the context's device): the all-reduce
    of a level's running sums and the slot all-gather are identities."""
    api = P.api
    prob, opt, plan = _plan(api, m=32, ell=1, seed=2)
    lev = plan.op.device_level(ctx, 0)
    lev.sums_reset(0.0, 0.0)
    d = api.LevelDraws()
    api.run_level_draws(plan, api.GridSpec.square(16), False, False, prob, opt, 0, 12, d, ctx=ctx)
    cm = api.Comm(ctx, 1, 0, api.Comm.unique_id())
    try:
        red = cm.allreduce_level_sums(lev)
        assert np.array_equal(red, lev.sums_read())
        x = np.stack([d.q_fine[:12], d.q_coarse[:12]], axis=1)
        assert np.array_equal(cm.allgather(x).reshape(12, 2), x)
    finally:
        cm.close()
    with pytest.raises(api.ConfigError):
        api.DeviceGroup(1, devices=[7])  # no such device
