"""GPU parity tests: every hot-path kernel through the C-ABI against the CPU
oracle on the same seeded inputs (instances are the reference tests' own
generators, tests/support.py).  Tolerances (north_star / SURVEY.md 8(c)):
half-sweep relative 1e-9 per column; loss and quartic 1e-12 relative;
gradient 1e-11 of its scale; vector ops within 8 ulp; ALS-NCG identical
iteration / backtrack / restart sequence with loss within 1e-9."""
import numpy as np
import pytest

import paper_1508_03110_b200 as P
from oracle.pyoracle import Oracle, OracleRatings, make_config
from support import (fd_gradient, movielens_like, naive_loss, random_flat, random_ratings,
                     rank_one_ratings, ulps_between)

pytestmark = pytest.mark.gpu
orc = Oracle("port")


def both(T):
    R = P.RatingsMatrix.from_triples(T.n_u, T.n_m, users=T.users, items=T.items, values=T.values)
    O = OracleRatings(T.n_u, T.n_m, T.users, T.items, T.values)
    return R, O


def flat(x, n_f, T):
    return P.FlatVector.from_array(x, n_f, T.n_u, T.n_m)


def dense(n_u, n_m, seed):
    """Fully dense instance: every item column has n_u ratings (heavy rows ->
    multi-segment split paths)."""
    rng = np.random.default_rng(seed)
    from support import Triples
    u, i = np.meshgrid(np.arange(n_u), np.arange(n_m), indexing="ij")
    v = np.round(rng.uniform(0.5, 5.0, size=n_u * n_m) * 2) / 2
    return Triples(n_u, n_m, u.ravel(), i.ravel(), v)


RANKS = [1, 2, 3, 5, 7, 10, 15, 25, 31, 50, 100]


@pytest.mark.parametrize("n_f", RANKS)
def test_gradient_matches_oracle(n_f):
    for seed in range(2):
        T = random_ratings(40, 30, 0.3, 30 + seed)
        R, O = both(T)
        x = random_flat(n_f, T.n_u, T.n_m, 40 + seed)
        for lam in (0.0, 0.1):
            g = P.ncg.gradient(flat(x, n_f, T), R, lam).array()
            gr = orc.gradient(O, n_f, x, lam)
            assert np.max(np.abs(g - gr)) <= 1e-11 * max(1.0, np.max(np.abs(gr)))


def test_gradient_heavy_rows_and_fd():
    T = dense(2500, 4, 1)  # items with 2500 > 2048 ratings -> split segments
    R, O = both(T)
    x = random_flat(3, T.n_u, T.n_m, 2)
    g = P.ncg.gradient(flat(x, 3, T), R, 0.1).array()
    gr = orc.gradient(O, 3, x, 0.1)
    assert np.max(np.abs(g - gr)) <= 1e-11 * np.max(np.abs(gr))
    # test_ncg.cpp:84-96 finite differences
    T = random_ratings(12, 8, 0.3, 31)
    R, _ = both(T)
    x = random_flat(3, 12, 8, 41)
    g = P.ncg.gradient(flat(x, 3, T), R, 0.1).array()
    fd = fd_gradient(x, T, 3, 0.1)
    big = np.abs(g) > 1e-8
    assert np.all(np.abs(fd[big] - g[big]) / np.abs(g[big]) <= 1e-5)


def test_gradient_empty_blocks():
    # test_ncg.cpp:71-82
    R = P.RatingsMatrix.from_triples(2, 1, [(0, 0, 3.0)])
    x = P.FlatVector.from_array(random_flat(3, 2, 1, 3), 3, 2, 1)
    g = P.ncg.gradient(x, R, 0.25)
    assert np.all(g.user_col(1) == 0.0)


@pytest.mark.parametrize("n_f", RANKS)
def test_loss_and_quartic_match_oracle(n_f):
    for seed in range(2):
        T = random_ratings(35, 20, 0.3, 100 + seed)
        R, O = both(T)
        x = random_flat(n_f, T.n_u, T.n_m, 200 + seed)
        p = random_flat(n_f, T.n_u, T.n_m, 300 + seed)
        for lam in (0.0, 0.1):
            lo = P.ncg.loss(flat(x, n_f, T), R, lam)
            lr = orc.loss(O, n_f, x, lam)
            assert abs(lo - lr) <= 1e-12 * max(1.0, abs(lr))
            assert abs(lo - naive_loss(x, T, n_f, lam)) <= 1e-12 * max(1.0, abs(lr))
            q = P.linesearch.quartic_coefficients(flat(x, n_f, T), flat(p, n_f, T), R, lam).c
            qr = orc.quartic(O, n_f, x, p, lam)
            scale = max(1.0, np.max(np.abs(qr)))
            assert np.max(np.abs(np.array(q) - qr)) <= 1e-12 * scale


def test_quartic_kats_and_direct_loss():
    # test_linesearch.cpp:28-66
    T = random_ratings(12, 8, 0.4, 1)
    R, O = both(T)
    x = random_flat(3, 12, 8, 2)
    q = P.linesearch.quartic_coefficients(flat(x, 3, T), P.FlatVector.zeros(3, 12, 8), R, 0.3)
    assert abs(q.c[0] - orc.loss(O, 3, x, 0.3)) <= 1e-13 * q.c[0]
    assert q.c[1:] == [0.0, 0.0, 0.0, 0.0]
    R1 = P.RatingsMatrix.from_triples(1, 1, [(0, 0, 1.0)])
    q = P.linesearch.quartic_coefficients(P.FlatVector.zeros(1, 1, 1),
                                          P.FlatVector(1, 1, 1, [1.0], [1.0]), R1, 0.0)
    assert q.c == [1.0, 0.0, -2.0, 0.0, 1.0]
    for seed in range(6):
        T = random_ratings(25, 15, 0.3, 100 + seed)
        R, O = both(T)
        lam = 0.0 if seed % 2 == 0 else 0.1
        x = random_flat(4, 25, 15, 200 + seed)
        p = random_flat(4, 25, 15, 300 + seed)
        q = P.linesearch.quartic_coefficients(flat(x, 4, T), flat(p, 4, T), R, lam)
        for a in (0.3, 1.0, 2.7):
            direct = orc.loss(O, 4, x + a * p, lam)
            assert abs(q(a) - direct) <= 1e-10 * max(1.0, direct)


def _col_rel_err(a, b, n_f):
    a = a.reshape(-1, n_f)
    b = b.reshape(-1, n_f)
    nb = np.linalg.norm(b, axis=1)
    err = np.linalg.norm(a - b, axis=1)
    nz = nb > 0
    assert np.all(err[~nz] == 0.0)
    return float(np.max(err[nz] / nb[nz])) if nz.any() else 0.0


HS_RANKS = [1, 2, 3, 5, 7, 10, 15, 25, 30, 31, 50, 64, 75, 85, 100, 110, 127, 136, 150, 160, 180, 200]


@pytest.mark.parametrize("n_f", HS_RANKS)
def test_half_sweep_matches_oracle(n_f):
    T = movielens_like(80, 40, 0.4, 7 + n_f)
    R, O = both(T)
    um, im = random_flat(n_f, T.n_u, T.n_m, 9)[: n_f * T.n_u], random_flat(n_f, T.n_u, T.n_m, 9)[n_f * T.n_u:]
    model = P.FactorModel(n_f, T.n_u, T.n_m)
    model.user_data, model.item_data = um, im
    for lam in (0.1, 0.01):
        stats = P.als.SolveStats()
        u = P.als.update_users(model, R, lam, stats)
        ur, fb = orc.half_sweep(O, True, n_f, im, lam)
        assert stats.fallback_columns == fb == 0
        assert _col_rel_err(u, ur, n_f) <= 1e-9
        m = P.als.update_items(model, R, lam)
        mr, _ = orc.half_sweep(O, False, n_f, um, lam)
        assert _col_rel_err(m, mr, n_f) <= 1e-9


@pytest.mark.parametrize("n_f", [3, 10, 31, 100])
def test_half_sweep_heavy_columns_split(n_f):
    # items rated by 9000 users (> every segment size) -> split-K partials
    T = dense(9000, 3, 5)
    R, O = both(T)
    x = random_flat(n_f, T.n_u, T.n_m, 6)
    model = P.FactorModel(n_f, T.n_u, T.n_m)
    model.user_data, model.item_data = x[: n_f * T.n_u], x[n_f * T.n_u:]
    m = P.als.update_items(model, R, 0.05)
    mr, _ = orc.half_sweep(O, False, n_f, model.user_data, 0.05)
    assert _col_rel_err(m, mr, n_f) <= 1e-9


def test_half_sweep_kats_and_fallback():
    # test_als.cpp:40-76 exact scalar solves and zero columns
    R = P.RatingsMatrix.from_triples(1, 1, [(0, 0, 2.0)])
    m = P.FactorModel(1, 1, 1)
    m.item_data = np.array([1.0])
    assert abs(P.als.update_users(m, R, 0.0)[0] - 2.0) <= 2e-15
    m.user_data = np.array([1.0])
    assert abs(P.als.update_items(m, R, 0.0)[0] - 2.0) <= 2e-15
    R = P.RatingsMatrix.from_triples(1, 2, [(0, 0, 1.0), (0, 1, 3.0)])
    m = P.FactorModel(1, 1, 2)
    m.item_data = np.array([1.0, 1.0])
    assert abs(P.als.update_users(m, R, 0.0)[0] - 2.0) <= 2e-15
    R = P.RatingsMatrix.from_triples(2, 2, [(0, 0, 4.0)])
    m = P.FactorModel(3, 2, 2)
    m.user_data, m.item_data = random_flat(3, 2, 2, 5)[:6], random_flat(3, 2, 2, 5)[6:]
    assert np.all(P.als.update_users(m, R, 0.1)[3:] == 0.0)
    assert np.all(P.als.update_items(m, R, 0.1)[3:] == 0.0)
    # test_als.cpp:108-122 rank-deficient least-norm fallback
    R = P.RatingsMatrix.from_triples(1, 1, [(0, 0, 2.0)])
    m = P.FactorModel(3, 1, 1)
    m.item_data = np.array([1.0, 2.0, 2.0])
    stats = P.als.SolveStats()
    m.user_data = P.als.update_users(m, R, 0.0, stats)
    assert stats.fallback_columns == 1
    assert abs(float(m.user_data @ m.item_data) - 2.0) <= 2e-12
    g = P.ncg.gradient(P.flatten(m), R, 0.0)
    assert np.max(np.abs(g.user_part)) <= 1e-10


def test_half_sweep_unregularised_stationarity():
    # test_als.cpp:78-96 (lambda = 0 -> every column through the fallback)
    T = random_ratings(30, 20, 0.5, 701)
    R, O = both(T)
    um, im = random_flat(5, 30, 20, 801)[:150], random_flat(5, 30, 20, 801)[150:]
    model = P.FactorModel(5, 30, 20)
    model.user_data, model.item_data = um, im
    model.user_data = P.als.update_users(model, R, 0.0)
    g = P.ncg.gradient(P.flatten(model), R, 0.0)
    assert np.max(np.abs(g.user_part)) <= 1e-8


def test_vector_ops_within_8_ulps():
    # test_core.cpp:97-112, test_ncg.cpp:126-154
    from oracle.pyoracle import beta_bar as orc_beta_bar, dot as orc_dot
    ctx = P.default_context()
    for seed in range(3):
        x = P.FlatVector.from_array(random_flat(4, 800, 1200, 100 + seed), 4, 800, 1200)
        y = P.FlatVector.from_array(random_flat(4, 800, 1200, 200 + seed), 4, 800, 1200)
        # API-level dot: the reference's sequential order, bit for bit
        assert P.dot(x, y) == orc_dot(x.array(), y.array())
        # driver reduction (compensated): within 8 ulps of the exact sum
        dx, dy = P.DeviceBuffer.from_array(ctx, x.array()), P.DeviceBuffer.from_array(ctx, y.array())
        import ctypes as C
        out = C.c_double()
        P._lib.check(P.lib().alsncg_dev_dot(ctx.handle, x.size(), dx.ptr, dy.ptr, C.byref(out)))
        exact = float(np.sum(np.longdouble(x.array()) * np.longdouble(y.array())))
        assert ulps_between(out.value, exact) <= 8
        z = P.axpby(1.5, x, -2.5, y).array()
        assert np.array_equal(z, 1.5 * x.array() + (-2.5) * y.array())  # bitwise
        gn, gp, bn, bp = (P.FlatVector.from_array(random_flat(2, 10, 6, s), 2, 10, 6)
                          for s in (60 + seed, 70 + seed, 80 + seed, 90 + seed))
        assert P.ncg.beta_bar(gn, gp, bn, bp) == orc_beta_bar(gn.array(), gp.array(), bn.array(),
                                                              bp.array())
    a = P.FlatVector(1, 2, 0, [1.0, 0.0], [])
    b = P.FlatVector(1, 2, 0, [0.0, 1.0], [])
    assert P.ncg.beta_bar(a, b, a, a) == 0.0  # degenerate denominator restarts
    assert P.ncg.normalized_grad_norm(P.FlatVector(1, 2, 2, [2.0, 0.0], [0.0, 0.0])) == 0.5


def _trace_equal(mine, ref, tol=1e-9):
    assert len(mine) == len(ref)
    for a, b in zip(mine, ref):
        assert a.iter == b["iter"]
        assert a.backtracks == b["backtracks"]
        assert a.restarted == b["restarted"]
        assert a.shuffled_columns == b["shuffled_columns"]
        assert abs(a.loss - b["loss"]) <= tol * max(1.0, abs(b["loss"]))
        assert abs(a.grad_norm - b["grad_norm"]) <= 1e-7 * b["grad_norm"] + 1e-15


def test_ncg_solve_config0_matches_oracle():
    R = P.generate(0)
    O = OracleRatings.from_csr(R.n_users(), R.n_items(), R.uptr, R.uidx, R.uval)
    cfg = P.SolverConfig(lambda_=0.1, n_f=10, max_iters=20, tol=0.0, seed=0)
    res = P.ncg.als_ncg_solve(R, cfg)
    x, trace, info = orc.ncg_solve(O, make_config(lambda_=0.1, n_f=10, max_iters=20, tol=0.0, seed=0))
    _trace_equal(res.trace.records, trace)
    assert (res.iterations, res.restarts, res.fallback_steps) == (
        info["iterations"], info["restarts"], info["fallback_steps"])
    mine = np.concatenate([res.model.user_data, res.model.item_data])
    assert np.linalg.norm(mine - x) <= 1e-8 * np.linalg.norm(x)


def test_ncg_solve_to_tolerance_same_iterations():
    T = movielens_like(60, 24, 0.3, 13)  # test_ncg.cpp:241-263 instance
    R, O = both(T)
    kw = dict(lambda_=0.1, n_f=4, tol=1e-6, max_iters=600, seed=3)
    res = P.ncg.als_ncg_solve(R, P.SolverConfig(**kw))
    x, trace, info = orc.ncg_solve(O, make_config(**kw))
    assert res.iterations == info["iterations"] and res.converged == info["converged"]
    _trace_equal(res.trace.records, trace, tol=1e-8)


def test_forced_beta_zero_alpha_one_is_plain_als_bitwise():
    # test_ncg.cpp:265-288
    T = movielens_like(40, 16, 0.3, 17)
    R, _ = both(T)
    cfg = P.SolverConfig(lambda_=0.1, n_f=3, tol=0.0, max_iters=10, seed=9)
    a = P.als.als_solve(R, cfg)
    b = P.ncg.als_ncg_solve(R, cfg, overrides=P.ncg.NcgOverrides(1.0, True))
    assert np.array_equal(a.model.user_data, b.model.user_data)
    assert np.array_equal(a.model.item_data, b.model.item_data)
    assert len(a.trace) == len(b.trace)
    for ra, rb in zip(a.trace.records, b.trace.records):
        assert ra.loss == rb.loss and ra.grad_norm == rb.grad_norm


def test_als_solve_matches_oracle_and_realizable():
    T = movielens_like(40, 16, 0.3, 81)
    R, O = both(T)
    kw = dict(lambda_=0.1, n_f=3, tol=1e-8, max_iters=200, seed=4)
    a = P.als.als_solve(R, P.SolverConfig(**kw))
    x, trace, info = orc.als_solve(O, make_config(**kw))
    assert a.iterations == info["iterations"]
    mine = np.concatenate([a.model.user_data, a.model.item_data])
    assert np.linalg.norm(mine - x) <= 1e-8 * np.linalg.norm(x)
    # test_als.cpp:188-201 / test_ncg.cpp:228-239 (lambda = 0: fallback path)
    T = rank_one_ratings(12, 8, 71)
    R, _ = both(T)
    r = P.als.als_solve(R, P.SolverConfig(lambda_=0.0, n_f=1, tol=1e-9, max_iters=500, seed=2))
    assert r.converged and r.final_loss <= 1e-10
    r = P.ncg.als_ncg_solve(R, P.SolverConfig(lambda_=0.0, n_f=1, tol=1e-10, max_iters=400, seed=5))
    assert r.converged and r.final_loss <= 1e-8


def test_stepping_solver_equals_one_shot():
    R = P.generate(0)
    cfg = P.SolverConfig(lambda_=0.1, n_f=10, max_iters=12, tol=0.0, seed=1)
    one = P.ncg.als_ncg_solve(R, cfg)
    s = P.ncg.Solver(R, cfg)
    assert s.step(5) == 5 and s.step(100) == 7
    assert np.array_equal(s.model(), np.concatenate([one.model.user_data, one.model.item_data]))
    assert [r.loss for r in s.trace().records] == [r.loss for r in one.trace.records]


def test_snapshot_cadence():
    R = P.generate(0)
    seen = []
    cfg = P.SolverConfig(lambda_=0.1, n_f=10, max_iters=6, tol=0.0, seed=0, snapshot_every=2)
    res = P.ncg.als_ncg_solve(R, cfg, snapshot=lambda m, it: seen.append((it, m.user_data[0])))
    assert [it for it, _ in seen] == [0, 2, 4, 6]
    assert seen[-1][1] == res.model.user_data[0]


@pytest.mark.parametrize("n_f,seed", [(10, 0), (7, 12345), (100, 2**63 + 11)])
def test_device_random_init_is_the_host_stream(n_f, seed):
    # factors.cpp:24-32: x0 is generated on the device (mt19937_64 twists in
    # one CTA); it must be bitwise the host Rng stream
    T = random_ratings(37, 23, 0.3, 99)
    R, _ = both(T)
    cfg = P.SolverConfig(lambda_=0.1, n_f=n_f, max_iters=0, tol=0.0, seed=seed)
    s = P.ncg.Solver(R, cfg)
    m = s.model()
    s.close()
    want = P.random_init(n_f, T.n_u, T.n_m, seed)
    assert np.array_equal(np.asarray(m), np.concatenate([want.user_data, want.item_data]))


@pytest.mark.parametrize("n_f,n_u,n_m,seed", [(100, 20000, 300, 3),       # 26 chunks: jumps of 1 and 8 chunks
                                              (64, 100000, 2000, 0),      # 84 chunks: adds the 64-chunk jump
                                              (100, 450000, 1000, 77)])   # 565 chunks: adds the 512-chunk jump
def test_device_random_init_jump_ahead_is_the_host_stream(n_f, n_u, n_m, seed):
    # x0 is generated in chunks of 312*256 draws whose start states come from
    # mt19937_64 jump-ahead (k_vec.cu, tools/gen_mt_jump.py): still bitwise the
    # host stream, across every jump level
    users = np.arange(n_u, dtype=np.int32)
    items = (users % n_m).astype(np.int32)
    values = np.full(n_u, 3.0)
    R = P.RatingsMatrix.from_triples(n_u, n_m, users=users, items=items, values=values)
    cfg = P.SolverConfig(lambda_=0.1, n_f=n_f, max_iters=0, tol=0.0, seed=seed)
    s = P.ncg.Solver(R, cfg)
    m = s.model()
    s.close()
    want = P.random_init(n_f, n_u, n_m, seed)
    assert np.array_equal(np.asarray(m), np.concatenate([want.user_data, want.item_data]))


def test_cuda_graph_replay_is_bitwise_the_plain_iteration(monkeypatch):
    # ALSNCG_GRAPH=1 replays gradient + P(x) + the fused gbar pass as a CUDA
    # graph (solver.cpp gradient_als_gbar): same kernels, same arguments, so
    # the trace and the model must be identical bit for bit
    T = random_ratings(60, 24, 0.35, 5)
    R, _ = both(T)
    out = []
    for on in (False, True):
        if on:
            monkeypatch.setenv("ALSNCG_GRAPH", "1")
        else:
            monkeypatch.delenv("ALSNCG_GRAPH", raising=False)
        cfg = P.SolverConfig(lambda_=0.05, n_f=6, max_iters=25, tol=0.0, seed=3)
        res = P.ncg.als_ncg_solve(R, cfg)
        out.append(res)
    a, b = out
    assert a.iterations == b.iterations == 25
    for ra, rb in zip(a.trace.records, b.trace.records):
        assert (ra.loss, ra.grad_norm, ra.backtracks, ra.restarted) == (rb.loss, rb.grad_norm, rb.backtracks, rb.restarted)
    assert np.array_equal(a.model.user_data, b.model.user_data)
    assert np.array_equal(a.model.item_data, b.model.item_data)
