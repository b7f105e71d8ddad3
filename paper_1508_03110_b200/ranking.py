"""alsncg::ranking (ranking.hpp:20-41).  rank_items / ranking_accuracy are
per-user host utilities (numpy); mean_ranking_accuracy runs on the device
(k_ranking.cu) with the reference's exact score arithmetic."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib, ptr


def _scores(model, user):
    u = np.asarray(model.user_data).reshape(model.n_u, model.n_f)[user]
    M = np.asarray(model.item_data).reshape(model.n_m, model.n_f)
    s = np.zeros(model.n_m)
    for k in range(model.n_f):  # sequential in k, separate rounding (ranking.cpp:45-47)
        s = s + u[k] * M[:, k]
    return s


def rank_items(model, user):
    """ranking.cpp:40-57 (ties by ascending item id)."""
    if user < 0 or user >= model.n_u:
        raise IndexError("rank_items: user index")
    s = _scores(model, user)
    return np.lexsort((np.arange(model.n_m), -s)).astype(np.int64)


def ranking_accuracy(p1, p2, t):
    """ranking.cpp:59-88."""
    p1, p2 = np.asarray(p1), np.asarray(p2)
    n = p1.size
    for p in (p1, p2):
        if p.size != n:
            raise ValueError("ranking_accuracy: size mismatch")
        if p.size and (p.min() < 0 or p.max() >= n or np.unique(p).size != n):
            raise ValueError("ranking_accuracy: not a permutation")
    if t < 1 or t > n:
        raise ValueError("ranking_accuracy: t out of range")
    pos = np.empty(n, np.int64)
    pos[p2] = np.arange(n)
    r2 = pos[p1[:t]]
    swaps = int(sum(int(r2[r]) - int(np.count_nonzero(r2[:r] < r2[r])) for r in range(t)))
    smax = t * (2 * n - t - 1) // 2
    return 1.0 if smax == 0 else 1.0 - swaps / smax


def mean_ranking_accuracy(model_at_k, model_final, t, n_workers=1, ctx=None):
    """ranking.cpp:90-109 on the device; n_workers accepted for API parity."""
    from .device import default_context
    if (model_at_k.n_f, model_at_k.n_u, model_at_k.n_m) != (model_final.n_f, model_final.n_u, model_final.n_m):
        raise ValueError("mean_ranking_accuracy: model shape mismatch")
    ctx = ctx or default_context()
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
            (model_at_k.user_data, model_at_k.item_data, model_final.user_data, model_final.item_data)]
    out = C.c_double(0.0)
    check(lib().alsncg_mean_ranking_accuracy(ctx.handle, model_at_k.n_f, model_at_k.n_u, model_at_k.n_m,
                                             *[ptr(a) for a in arrs], t, C.byref(out)))
    return out.value
