"""Parity at BASELINE config 1's full size (138,493 users x 26,744 items,
20,000,263 ratings, n_f = 100, lambda = 0.01) through checks that do not need
a full CPU run of the oracle:
  * CSR/CSC: the product's host build equals the oracle's restatement of
    RatingsMatrix::from_triples (ratings.cpp:28-89) bitwise, and so does the
    device copy;
  * half-sweeps: sampled columns (the heaviest users/items plus random ones)
    re-solved exactly in float64 from their normal equations (als.cpp:49-70)
    -- relative error <= 1e-9 per column (north_star tolerance);
  * quartic: loss(x + a p) equals the device quartic at several a (the
    profile is exact up to rounding, linesearch.cpp:46-111) -- 1e-10 relative.
"""
import numpy as np
import pytest

import paper_1508_03110_b200 as P
from oracle.pyoracle import OracleRatings

pytestmark = pytest.mark.gpu
N_F, LAM = 100, 0.01


@pytest.fixture(scope="module")
def cfg1():
    return P.generate(1)


def _exact_columns(ptr, idx, val, src, cols, n_f, lam):
    out = {}
    for c in cols:
        b, e = int(ptr[c]), int(ptr[c + 1])
        G = np.zeros((n_f, n_f))
        rhs = np.zeros(n_f)
        for s in range(b, e, 200_000):  # chunked: the heaviest items have ~1.9M ratings
            t = min(e, s + 200_000)
            M = src[idx[s:t]]
            G += M.T @ M
            rhs += val[s:t] @ M
        G[np.diag_indices(n_f)] += lam * (e - b)
        out[c] = np.linalg.solve(G, rhs)
    return out


def _pick(ptr, k_heavy, k_rand, seed):
    cnt = np.diff(ptr)
    heavy = np.argsort(-cnt, kind="stable")[:k_heavy]
    rng = np.random.default_rng(seed)
    return sorted(set(heavy.tolist()) | set(rng.choice(len(cnt), k_rand, replace=False).tolist()))


def test_config1_csr_csc_bitwise(cfg1):
    R = cfg1
    O = OracleRatings.from_csr(R.n_users(), R.n_items(), R.uptr, R.uidx, R.uval)
    for a, b in ((R.uptr, O.uptr), (R.uidx, O.uidx), (R.uval, O.uval), (R.iptr, O.iptr),
                 (R.iidx, O.iidx), (R.ival, O.ival)):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    assert R.nnz() == 20_000_263


def test_config1_half_sweeps_sampled_columns(cfg1):
    R = cfg1
    n_u, n_m = R.n_users(), R.n_items()
    rng = np.random.default_rng(11)
    model = P.FactorModel(N_F, n_u, n_m)
    model.user_data = rng.uniform(0.0, 1.0, N_F * n_u)
    model.item_data = rng.uniform(0.0, 1.0, N_F * n_m)
    stats = P.als.SolveStats()
    users = P.als.update_users(model, R, LAM, stats)
    assert stats.fallback_columns == 0
    U = np.asarray(users).reshape(n_u, N_F)
    Mi = np.asarray(model.item_data).reshape(n_m, N_F)
    want = _exact_columns(R.uptr, R.uidx, R.uval, Mi, _pick(R.uptr, 10, 300, 1), N_F, LAM)
    for c, w in want.items():
        assert np.linalg.norm(U[c] - w) <= 1e-9 * np.linalg.norm(w), c
    model.user_data = users
    items = P.als.update_items(model, R, LAM, stats)
    I = np.asarray(items).reshape(n_m, N_F)
    want = _exact_columns(R.iptr, R.iidx, R.ival, U, _pick(R.iptr, 3, 60, 2), N_F, LAM)
    for c, w in want.items():
        assert np.linalg.norm(I[c] - w) <= 1e-9 * np.linalg.norm(w), c


def test_config1_quartic_is_the_exact_profile(cfg1):
    R = cfg1
    n_u, n_m = R.n_users(), R.n_items()
    rng = np.random.default_rng(5)
    x = P.FlatVector.from_array(rng.uniform(0.0, 0.3, N_F * (n_u + n_m)), N_F, n_u, n_m)
    p = P.FlatVector.from_array(rng.normal(0.0, 0.05, N_F * (n_u + n_m)), N_F, n_u, n_m)
    q = P.linesearch.quartic_coefficients(x, p, R, LAM)
    for a in (0.0, 0.25, 1.0, 2.5):
        xa = P.FlatVector.from_array(x.array() + a * p.array(), N_F, n_u, n_m)
        f = P.ncg.loss(xa, R, LAM)
        assert abs(q(a) - f) <= 1e-10 * abs(f), (a, q(a), f)
