"""alsncg::linesearch (linesearch.hpp:29-54)."""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib, ptr
from .config import QuarticPoly


class LineSearchStatus(enum.IntEnum):
    kAccepted = 0
    kNotDescent = 1
    kMaxBacktracks = 2


@dataclass
class LineSearchResult:
    status: LineSearchStatus = LineSearchStatus.kNotDescent
    alpha: float = 0.0
    backtracks: int = 0


def quartic_coefficients(x, p, ratings, lambda_, n_chunks=1, n_workers=1, ctx=None):
    """linesearch.cpp:46-111 (K7: one pass over the ratings on the device).
    n_chunks/n_workers are accepted for API parity; the device reduction is
    compensated and independent of both."""
    if not x.same_shape(p):
        raise ValueError("quartic_coefficients: shape mismatch")
    if x.n_u != ratings.n_users() or x.n_m != ratings.n_items():
        raise ValueError("quartic_coefficients: vector/ratings dimension mismatch")
    xa, pa = x.array(), p.array()
    c = np.zeros(5)
    check(lib().alsncg_quartic(ratings.device(ctx), x.n_f, ptr(xa), ptr(pa), lambda_, ptr(c)))
    return QuarticPoly(list(c))


def armijo_slope(g, p, ctx=None):
    from .factors import dot
    return dot(g, p, ctx)


def backtracking_search(q, slope, alpha0, c, tau, max_backtracks):
    """linesearch.cpp:115-131 (host scalar loop, as in the reference)."""
    coeffs = np.ascontiguousarray(q.c, dtype=np.float64)
    a, k = C.c_double(0.0), C.c_int(0)
    st = lib().alsncg_backtracking_search(ptr(coeffs), slope, alpha0, c, tau, max_backtracks,
                                          C.byref(a), C.byref(k))
    if st < 0:
        check(-st)
    return LineSearchResult(LineSearchStatus(st), a.value, k.value)
