"""Ranking evaluation (ranking.cpp:40-109).

CPU: the host utilities rank_items / ranking_accuracy equal the reference's
on seeded models and random permutations (the swap walk's closed form).
GPU: mean_ranking_accuracy on the device equals the reference's
(oracle/_ref) EXACTLY -- the scores use the reference's arithmetic, so every
tie and order is the same -- including tied scores and t = 1 / t = n."""
import numpy as np
import pytest

import paper_1508_03110_b200 as P
from oracle.pyoracle import ref_available, ref_mean_ranking_accuracy


def walk(p1, p2, t):  # ranking.cpp:66-85 verbatim semantics, as a check of the closed form
    working = list(p2)
    pos = {v: r for r, v in enumerate(working)}
    swaps = 0
    for r in range(t):
        item = p1[r]
        cur = pos[item]
        swaps += cur - r
        for k in range(cur, r, -1):
            working[k] = working[k - 1]
            pos[working[k]] = k
        working[r] = item
        pos[item] = r
    n = len(p1)
    smax = t * (2 * n - t - 1) // 2
    return 1.0 if smax == 0 else 1.0 - swaps / smax


def model(n_f, n_u, n_m, seed, ties=False):
    rng = np.random.default_rng(seed)
    m = P.FactorModel(n_f, n_u, n_m)
    m.user_data = rng.normal(size=n_f * n_u)
    it = rng.normal(size=n_f * n_m)
    if ties:  # duplicate item columns -> exactly tied scores
        it = it.reshape(n_m, n_f)
        it[1::3] = it[0::3][: it[1::3].shape[0]]
        it = it.ravel()
    m.item_data = it
    return m


def test_ranking_accuracy_closed_form_equals_walk():
    rng = np.random.default_rng(1)
    for n in (1, 2, 7, 50):
        for _ in range(20):
            p1, p2 = rng.permutation(n), rng.permutation(n)
            for t in {1, max(1, n // 2), n}:
                assert P.ranking.ranking_accuracy(p1, p2, t) == walk(list(p1), list(p2), t)
    with pytest.raises(ValueError):
        P.ranking.ranking_accuracy([0, 1], [0, 0], 1)
    with pytest.raises(ValueError):
        P.ranking.ranking_accuracy([0, 1], [1, 0], 3)


def test_rank_items_ties_by_item_id():
    m = model(3, 4, 30, 2, ties=True)
    for u in range(4):
        r = P.ranking.rank_items(m, u)
        s = P.ranking._scores(m, u)
        for a, b in zip(r[:-1], r[1:]):
            assert s[a] > s[b] or (s[a] == s[b] and a < b)


@pytest.mark.gpu
@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n_f,n_u,n_m,t,ties", [(5, 300, 80, 10, False), (8, 257, 200, 1, True),
                                                  (4, 64, 33, 33, True), (16, 1000, 700, 20, False),
                                                  (100, 600, 2000, 50, False)])
def test_device_mean_ranking_accuracy_equals_reference(n_f, n_u, n_m, t, ties):
    mk, mf = model(n_f, n_u, n_m, 10, ties), model(n_f, n_u, n_m, 11, ties)
    mk.item_data = 0.7 * mk.item_data + 0.3 * mf.item_data  # correlated rankings
    got = P.ranking.mean_ranking_accuracy(mk, mf, t)
    want = ref_mean_ranking_accuracy(n_f, n_u, n_m, mk.user_data, mk.item_data, mf.user_data,
                                     mf.item_data, t, 4)
    assert got == want, (got, want)
    with pytest.raises(ValueError):
        P.ranking.mean_ranking_accuracy(mk, mf, n_m + 1)
