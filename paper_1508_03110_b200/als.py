"""alsncg::als (als.hpp:25-58) on the B200 half-sweep kernels."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib, ptr
from .factors import FlatVector


@dataclass
class SolveStats:
    fallback_columns: int = 0


def _half(model, ratings, lambda_, stats, kind, ctx):
    n_f = model.n_f
    src = model.item_data if kind == 0 else model.user_data
    n_dest = ratings.n_users() if kind == 0 else ratings.n_items()
    out = np.zeros(n_f * n_dest)
    fb = C.c_int(0)
    src = np.ascontiguousarray(src, dtype=np.float64)
    check(lib().alsncg_half_sweep(ratings.device(ctx), kind, n_f, ptr(src), lambda_, ptr(out),
                                  C.byref(fb)))
    if stats is not None:
        stats.fallback_columns += fb.value
    return out


def update_users(model, ratings, lambda_, stats=None, ctx=None):
    """als.cpp:85-102: every user column from the item factors."""
    return _half(model, ratings, lambda_, stats, 0, ctx)


def update_items(model, ratings, lambda_, stats=None, ctx=None):
    """als.cpp:104-121."""
    return _half(model, ratings, lambda_, stats, 1, ctx)


def als_sweep(x, ratings, lambda_, ctx=None):
    """als.cpp:123-128: P(x) = items(users(x))."""
    arr = x.array()
    out = np.empty_like(arr)
    fb = C.c_int(0)
    check(lib().alsncg_als_sweep(ratings.device(ctx), x.n_f, ptr(arr), lambda_, ptr(out),
                                 C.byref(fb)))
    return FlatVector.from_array(out, x.n_f, x.n_u, x.n_m)


def als_solve(ratings, config, snapshot=None, ctx=None):
    """als.cpp:130-195: plain ALS on the device."""
    from .ncg import _solve
    return _solve("als", ratings, config, snapshot, None, ctx)
