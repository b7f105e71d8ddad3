"""alsncg::ncg (ncg.hpp:30-65) on the B200 kernels."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .config import ConvergenceTrace, SolveResult, TraceRecord
from .factors import FactorModel, FlatVector


@dataclass
class NcgOverrides:
    fixed_alpha: Optional[float] = None
    force_beta_zero: bool = False


def _check_shape(x, ratings):
    if x.n_u != ratings.n_users() or x.n_m != ratings.n_items():
        raise ValueError("vector/ratings dimension mismatch")


def loss(x, ratings, lambda_, ctx=None):
    """ncg.cpp:43-68 (K6, deterministic compensated reduction)."""
    _check_shape(x, ratings)
    out = C.c_double()
    arr = x.array()
    check(lib().alsncg_loss(ratings.device(ctx), x.n_f, ptr(arr), lambda_, C.byref(out)))
    return out.value


def gradient(x, ratings, lambda_, n_workers=1, ctx=None):
    """ncg.cpp:70-116 (K5).  n_workers is accepted for API parity; the
    result never depends on it (rows are independent)."""
    _check_shape(x, ratings)
    arr = x.array()
    g = np.empty_like(arr)
    check(lib().alsncg_gradient(ratings.device(ctx), x.n_f, ptr(arr), lambda_, ptr(g)))
    return FlatVector.from_array(g, x.n_f, x.n_u, x.n_m)


def beta_bar(g_next, g_prev, gbar_next, gbar_prev, ctx=None):
    """ncg.cpp:118-132."""
    from .device import DeviceBuffer, default_context
    if not (g_next.same_shape(g_prev) and gbar_next.same_shape(g_next)
            and gbar_prev.same_shape(g_next)):
        raise ValueError("beta_bar: shape mismatch")
    ctx = ctx or default_context()
    bufs = [DeviceBuffer.from_array(ctx, v.array()) for v in (g_next, g_prev, gbar_next, gbar_prev)]
    out = C.c_double()
    check(lib().alsncg_dev_beta_bar_seq(ctx.handle, g_next.size(), bufs[0].ptr, bufs[1].ptr,
                                    bufs[2].ptr, bufs[3].ptr, C.byref(out)))
    return out.value


def normalized_grad_norm(g, ctx=None):
    """ncg.cpp:134-136."""
    from .factors import norm
    n = g.size()
    return norm(g, ctx) / float(n) if n else 0.0


def _trace_from_c(recs, n):
    t = ConvergenceTrace()
    for r in recs[:n]:
        t.records.append(TraceRecord(r.iter, r.loss, r.grad_norm, r.elapsed_seconds, r.backtracks,
                                     r.shuffled_columns, bool(r.restarted)))
    return t


def _solve(which, ratings, config, snapshot, overrides, ctx):
    config.validate()
    n_f, n_u, n_m = config.n_f, ratings.n_users(), ratings.n_items()
    ov = overrides or NcgOverrides()
    cfg = config.to_c(ov.fixed_alpha, ov.force_beta_zero)
    model = np.zeros(max(n_f * (n_u + n_m), 1))
    cap = config.max_iters + 2
    recs = (_lib.TraceRecordC * cap)()
    n = C.c_int(0)
    res = _lib.ResultC()

    def _cb(it, nf, nu, nm, u, m, _user):
        fm = FactorModel(nf, nu, nm)
        fm.user_data = np.ctypeslib.as_array(u, shape=(nf * nu,)).copy() if nf * nu else fm.user_data
        fm.item_data = np.ctypeslib.as_array(m, shape=(nf * nm,)).copy() if nf * nm else fm.item_data
        snapshot(fm, it)

    cb = _lib.SNAPSHOT_FN(_cb) if snapshot else _lib.SNAPSHOT_FN()
    fn = lib().alsncg_ncg_solve if which == "ncg" else lib().alsncg_als_solve
    check(fn(ratings.device(ctx), C.byref(cfg), cb, None, C.byref(res), ptr(model), recs, cap,
             C.byref(n)))
    out = SolveResult()
    fm = FactorModel(n_f, n_u, n_m)
    fm.user_data = model[:n_f * n_u].copy()
    fm.item_data = model[n_f * n_u:n_f * (n_u + n_m)].copy()
    out.model = fm
    out.trace = _trace_from_c(recs, min(n.value, cap))
    out.converged, out.iterations = bool(res.converged), res.iterations
    out.final_loss, out.final_grad_norm = res.final_loss, res.final_grad_norm
    out.restarts, out.fallback_steps = res.restarts, res.fallback_steps
    out.fallback_columns = res.fallback_columns
    return out


def als_ncg_solve(ratings, config, snapshot=None, overrides=None, ctx=None):
    """ncg.cpp:138-307: the device-resident ALS-NCG driver."""
    return _solve("ncg", ratings, config, snapshot, overrides, ctx)


class Solver:
    """Stepping interface (alsncg_solver_*): setup on construction, then
    step(n) runs n outer iterations on the device."""

    def __init__(self, ratings, config, ctx=None):
        config.validate()
        self.ratings, self.config = ratings, config
        self.handle = C.c_void_p()
        cfg = config.to_c()
        check(lib().alsncg_solver_create(ratings.device(ctx), C.byref(cfg), C.byref(self.handle)))

    def step(self, n=1):
        ran = C.c_int(0)
        check(lib().alsncg_solver_step(self.handle, n, C.byref(ran)))
        return ran.value

    def state(self):
        it, conv, rs, fs, fc = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        gn = C.c_double()
        check(lib().alsncg_solver_state(self.handle, C.byref(it), C.byref(conv), C.byref(gn),
                                        C.byref(rs), C.byref(fs), C.byref(fc)))
        return dict(iterations=it.value, converged=bool(conv.value), grad_norm=gn.value,
                    restarts=rs.value, fallback_steps=fs.value, fallback_columns=fc.value)

    def trace(self):
        n = C.c_int(0)
        check(lib().alsncg_solver_trace(self.handle, None, 0, C.byref(n)))
        recs = (_lib.TraceRecordC * max(n.value, 1))()
        check(lib().alsncg_solver_trace(self.handle, recs, n.value, C.byref(n)))
        return _trace_from_c(recs, n.value)

    def model(self):
        c = self.config
        out = np.zeros(c.n_f * (self.ratings.n_users() + self.ratings.n_items()))
        check(lib().alsncg_solver_model(self.handle, ptr(out)))
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib().alsncg_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["loss", "gradient", "beta_bar", "normalized_grad_norm", "NcgOverrides",
           "als_ncg_solve", "Solver", "math"]
