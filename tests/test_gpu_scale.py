"""Parity AT SCALE against the CPU oracle: the CUDA path
through the C-ABI versus the reference compiled in place (oracle/_ref; the
bitwise-pinned port when _ref was not built) on BASELINE configs 1, 2 and 3 at
full size, same seeded inputs:

  * device CSR/CSC downloaded back and compared byte for byte with the
    oracle's restatement of RatingsMatrix::from_triples (ratings.cpp:28-89);
  * both half-sweeps on EVERY column, relative 1e-9 per column
    (north_star; als.cpp:40-121, parallel.cpp:144-185), at n_f = 10, 25, 50,
    100, 200 on the config-1 matrix and n_f = 50 on config 3;
  * loss (ncg.cpp:43-68) within 1e-12, gradient (ncg.cpp:70-116) within 1e-11
    of its scale, quartic coefficients (linesearch.cpp:46-111) within 1e-12 of
    the coefficient scale, at x0 and at a seeded direction.

The oracle runs on every host core (n_workers = nproc); the whole module takes
a few minutes on a 16-core GPU box.
"""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1508_03110_b200 as P
from oracle.pyoracle import Oracle, OracleRatings, ref_available

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
CORES = os.cpu_count() or 1
ORC = Oracle("ref" if ref_available() else "port")


@pytest.fixture(scope="module")
def m1():
    R = P.generate(1)
    O = OracleRatings.from_csr(R.n_users(), R.n_items(), R.uptr, R.uidx, R.uval)
    return R, O


@pytest.fixture(scope="module")
def m3():
    R = P.generate(3)
    O = OracleRatings.from_csr(R.n_users(), R.n_items(), R.uptr, R.uidx, R.uval)
    return R, O


def _download(R):
    L = P._lib.lib()
    U, M, Z = R.n_users(), R.n_items(), R.nnz()
    a = [np.empty(U + 1, np.int64), np.empty(Z, np.int32), np.empty(Z, np.float64),
         np.empty(M + 1, np.int64), np.empty(Z, np.int32), np.empty(Z, np.float64)]
    P._lib.check(L.alsncg_ratings_download(R.device(), *[C.c_void_p(x.ctypes.data) for x in a]))
    return a


def _col_rel(got, want, n_f):
    g = np.asarray(got).reshape(-1, n_f)
    w = np.asarray(want).reshape(-1, n_f)
    num = np.linalg.norm(g - w, axis=1)
    den = np.linalg.norm(w, axis=1)
    rel = np.where(den > 0, num / np.where(den > 0, den, 1.0), num)
    return rel


def _check_half_sweeps(R, O, n_f, lam, seed):
    n_u, n_m = R.n_users(), R.n_items()
    x0 = ORC.random_init(n_f, n_u, n_m, seed)
    model = P.FactorModel(n_f, n_u, n_m)
    model.user_data = x0[: n_f * n_u]
    model.item_data = x0[n_f * n_u:]
    stats = P.als.SolveStats()
    users = P.als.update_users(model, R, lam, stats)
    want_u, fb = ORC.half_sweep(O, True, n_f, x0[n_f * n_u:], lam, n_blocks=CORES, n_workers=CORES)
    assert fb == stats.fallback_columns == 0
    rel = _col_rel(users, want_u, n_f)
    assert rel.max() <= 1e-9, (n_f, "users", int(rel.argmax()), float(rel.max()))
    # item half from the ORACLE's users: identical inputs for both sides
    model.user_data = want_u
    items = P.als.update_items(model, R, lam, stats)
    want_i, fb = ORC.half_sweep(O, False, n_f, want_u, lam, n_blocks=CORES, n_workers=CORES)
    assert fb == stats.fallback_columns == 0
    rel_i = _col_rel(items, want_i, n_f)
    assert rel_i.max() <= 1e-9, (n_f, "items", int(rel_i.argmax()), float(rel_i.max()))
    return float(rel.max()), float(rel_i.max())


def test_config1_device_csr_csc_bytes(m1):
    R, O = m1
    got = _download(R)
    for g, w in zip(got, (O.uptr, O.uidx, O.uval, O.iptr, O.iidx, O.ival)):
        assert g.tobytes() == np.ascontiguousarray(w).tobytes()


@pytest.mark.parametrize("n_f", [100, 10, 25, 50, 200])
def test_config1_config2_half_sweeps_every_column(m1, n_f):
    R, O = m1
    _check_half_sweeps(R, O, n_f, 0.01, seed=0)


def test_config1_loss_gradient_quartic(m1):
    R, O = m1
    n_f, lam = 100, 0.01
    n_u, n_m = R.n_users(), R.n_items()
    x0 = ORC.random_init(n_f, n_u, n_m, 0)
    rng = np.random.default_rng(3)
    p = rng.normal(0.0, 0.02, x0.size)
    X = P.FlatVector.from_array(x0, n_f, n_u, n_m)
    Pd = P.FlatVector.from_array(p, n_f, n_u, n_m)
    lo = P.ncg.loss(X, R, lam)
    lw = ORC.loss(O, n_f, x0, lam)
    assert abs(lo - lw) <= 1e-12 * abs(lw), (lo, lw)
    g = P.ncg.gradient(X, R, lam).array()
    gw = ORC.gradient(O, n_f, x0, lam, n_workers=CORES)
    assert np.max(np.abs(g - gw)) <= 1e-11 * np.max(np.abs(gw))
    q = P.linesearch.quartic_coefficients(X, Pd, R, lam)
    qw = ORC.quartic(O, n_f, x0, p, lam, n_chunks=CORES, n_workers=CORES)
    scale = np.max(np.abs(qw))
    assert np.max(np.abs(np.asarray(q.c) - qw)) <= 1e-12 * scale, (q.c, qw)
    # the quartic's constant term is the loss at x (test_linesearch.cpp:28-35)
    assert abs(q.c[0] - lw) <= 1e-12 * abs(lw)


def test_config3_csr_half_sweeps_every_column(m3):
    R, O = m3
    got = _download(R)
    for g, w in zip(got, (O.uptr, O.uidx, O.uval, O.iptr, O.iidx, O.ival)):
        assert g.tobytes() == np.ascontiguousarray(w).tobytes()
    _check_half_sweeps(R, O, 50, 0.05, seed=0)


def test_config3_loss_gradient(m3):
    R, O = m3
    n_f, lam = 50, 0.05
    n_u, n_m = R.n_users(), R.n_items()
    x0 = ORC.random_init(n_f, n_u, n_m, 0)
    X = P.FlatVector.from_array(x0, n_f, n_u, n_m)
    lo = P.ncg.loss(X, R, lam)
    lw = ORC.loss(O, n_f, x0, lam)
    assert abs(lo - lw) <= 1e-12 * abs(lw), (lo, lw)
    g = P.ncg.gradient(X, R, lam).array()
    gw = ORC.gradient(O, n_f, x0, lam, n_workers=CORES)
    assert np.max(np.abs(g - gw)) <= 1e-11 * np.max(np.abs(gw))
