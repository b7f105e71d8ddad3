"""Pins the CPU oracle (plain-C port) against the reference compiled in place
(oracle/_ref) bitwise, and against the reference tests' known answers.

These are the "trust the oracle" tests: the port is only used as the parity
checker for the CUDA path once it agrees with the reference here (and with
the committed golden fixtures, tests/test_golden.py, which also run on hosts
without /root/reference).
"""
import numpy as np
import pytest

from oracle.pyoracle import OracleRatings, Rng, make_config, ref, ref_available
from support import movielens_like, random_flat, random_ratings, rank_one_ratings


def R(T):
    return OracleRatings(T.n_u, T.n_m, T.users, T.items, T.values)


def test_mt19937_64_known_answer():
    # std::mt19937_64 default seed 5489: the 10000th draw is 9981545732273789042
    # (C++ standard [rand.predef]).
    rng = Rng(5489)
    for _ in range(9999):
        rng.next_u64()
    assert rng.next_u64() == 9981545732273789042


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_rng_streams_match_reference():
    n = 257
    raw = np.zeros(n, np.uint64)
    uni, nrm = np.zeros(n), np.zeros(n)
    ref().ref_rng_draws(12345, n, raw, uni, nrm)
    a, b, c = Rng(12345), Rng(12345), Rng(12345)
    assert [a.next_u64() for _ in range(n)] == [int(v) for v in raw]
    assert np.array_equal([b.uniform() for _ in range(n)], uni)
    assert np.array_equal([c.normal() for _ in range(n)], nrm)


def test_build_rejects_bad_input():
    # test_core.cpp:125-132
    with pytest.raises(ValueError):
        OracleRatings(2, 2, [0], [2], [1.0])
    with pytest.raises(ValueError):
        OracleRatings(2, 2, [-1], [0], [1.0])
    with pytest.raises(ValueError):
        OracleRatings(2, 2, [0], [0], [float("nan")])
    with pytest.raises(ValueError):
        OracleRatings(2, 2, [0, 0, 0], [0, 1, 0], [1.0, 2.0, 3.0])


def test_port_csr_csc_bitwise_vs_reference(refimpl):
    from oracle.pyoracle import ref as reflib
    for seed in range(3):
        T = movielens_like(50, 30, 0.3, 100 + seed)
        Rp = R(T)
        h = Rp.ref_handle()
        uptr = np.zeros(T.n_u + 1, np.int64)
        iptr = np.zeros(T.n_m + 1, np.int64)
        uidx = np.zeros(Rp.nnz, np.int32)
        iidx = np.zeros(Rp.nnz, np.int32)
        uval = np.zeros(Rp.nnz)
        ival = np.zeros(Rp.nnz)
        reflib().ref_ratings_export(h, uptr, uidx, uval, iptr, iidx, ival)
        for a, b in [(uptr, Rp.uptr), (iptr, Rp.iptr), (uidx, Rp.uidx), (iidx, Rp.iidx),
                     (uval, Rp.uval), (ival, Rp.ival)]:
            assert a.tobytes() == b.tobytes()


def test_port_kernels_bitwise_vs_reference(port, refimpl):
    for seed in range(4):
        T = random_ratings(30, 20, 0.3, 700 + seed)
        Rp = R(T)
        n_f = 5
        x = random_flat(n_f, 30, 20, 800 + seed)
        p = random_flat(n_f, 30, 20, 900 + seed)
        for lam in (0.0, 0.1):
            assert port.loss(Rp, n_f, x, lam) == refimpl.loss(Rp, n_f, x, lam)
            assert np.array_equal(port.gradient(Rp, n_f, x, lam), refimpl.gradient(Rp, n_f, x, lam))
            for chunks in (1, 3):
                assert np.array_equal(port.quartic(Rp, n_f, x, p, lam, chunks),
                                      refimpl.quartic(Rp, n_f, x, p, lam, chunks))
        for users in (True, False):
            src = x[n_f * 30:] if users else x[: n_f * 30]
            a, fa = port.half_sweep(Rp, users, n_f, src, 0.1)
            b, fb = refimpl.half_sweep(Rp, users, n_f, src, 0.1, n_blocks=4, n_workers=2)
            assert np.array_equal(a, b) and fa == fb
        assert port.routing_totals(Rp, 4) == refimpl.routing_totals(Rp, 4)
    assert np.array_equal(port.random_init(7, 11, 5, 3), refimpl.random_init(7, 11, 5, 3))


def test_port_drivers_bitwise_vs_reference(port, refimpl):
    T = movielens_like(40, 16, 0.3, 17)
    Rp = R(T)
    for kw in (dict(), dict(has_fixed_alpha=1, fixed_alpha=1.0, force_beta_zero=1)):
        cfg = make_config(lambda_=0.1, n_f=3, tol=0.0, max_iters=25, seed=9, n_blocks=3, **kw)
        xa, ta, ra = port.ncg_solve(Rp, cfg)
        xb, tb, rb = refimpl.ncg_solve(Rp, cfg)
        assert np.array_equal(xa, xb)
        for a, b in zip(ta, tb):
            a = dict(a); b = dict(b)
            a.pop("elapsed_seconds"); b.pop("elapsed_seconds")
            assert a == b
        assert ra == rb
    cfg = make_config(lambda_=0.1, n_f=3, tol=0.0, max_iters=10, seed=9)
    xa, ta, ra = port.als_solve(Rp, cfg)
    xb, tb, rb = refimpl.als_solve(Rp, cfg)
    assert np.array_equal(xa, xb) and ra == rb


def test_kat_quartic_single_rating(port):
    # test_linesearch.cpp:37-51: coefficients (1, 0, -2, 0, 1)
    Rp = OracleRatings(1, 1, [0], [0], [1.0])
    c = port.quartic(Rp, 1, np.zeros(2), np.ones(2), 0.0)
    assert list(c) == [1.0, 0.0, -2.0, 0.0, 1.0]


def test_kat_backtracking_22(port):
    # test_linesearch.cpp:98-116: Q(a) = (a-1)^2, slope -2 -> 22 shrinks
    st, alpha, k = port.backtracking([1.0, -2.0, 1.0, 0.0, 0.0], -2.0, 10.0, 0.5, 0.9, 100)
    assert st == 0 and k == 22
    a = 10.0
    for _ in range(22):
        a *= 0.9
    assert alpha == a
    # :118-124 immediate acceptance; :126-138 statuses
    assert port.backtracking([5.0, -1.0, 0, 0, 0], -1.0, 2.0, 0.5, 0.9, 100) == (0, 2.0, 0)
    assert port.backtracking([1.0, 1.0, 0, 0, 0], 0.0, 1.0, 0.5, 0.9, 10)[0] == 1
    assert port.backtracking([3.0, 0, 0, 0, 0], -1.0, 1.0, 0.5, 0.9, 10)[0:3:2] == (2, 10)


def test_kat_scalar_solves(port):
    # test_als.cpp:40-65: u = 2
    Rp = OracleRatings(1, 1, [0], [0], [2.0])
    out, fb = port.half_sweep(Rp, True, 1, np.array([1.0]), 0.0)
    assert abs(out[0] - 2.0) <= 1e-15 * 2
    Rp = OracleRatings(1, 2, [0, 0], [0, 1], [1.0, 3.0])
    out, fb = port.half_sweep(Rp, True, 1, np.array([1.0, 1.0]), 0.0)
    assert abs(out[0] - 2.0) <= 1e-15 * 2


def test_kat_rank_deficient_fallback(port):
    # test_als.cpp:108-122
    Rp = OracleRatings(1, 1, [0], [0], [2.0])
    item = np.array([1.0, 2.0, 2.0])
    out, fb = port.half_sweep(Rp, True, 3, item, 0.0)
    assert fb == 1
    assert abs(float(out @ item) - 2.0) <= 1e-12 * 2
    g = port.gradient(Rp, 3, np.concatenate([out, item]), 0.0)
    assert np.max(np.abs(g[:3])) <= 1e-10


def test_oracle_als_solve_rank_one(port):
    # test_als.cpp:188-201
    T = rank_one_ratings(12, 8, 71)
    x, trace, res = port.als_solve(R(T), make_config(lambda_=0.0, n_f=1, tol=1e-9,
                                                      max_iters=500, seed=2))
    assert res["converged"] and res["final_loss"] <= 1e-10
