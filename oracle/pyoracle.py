"""ctypes bindings for the CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle_port.so`` (the plain-C restatement, always present
after ``make -C oracle port``) and, when it was built in this container,
``oracle/_ref/libalsncg_ref.so`` (the reference's own sources compiled in
place).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module; the product
package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libalsncg_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class Ratings(C.Structure):
    _fields_ = [("n_u", C.c_int), ("n_m", C.c_int), ("nnz", C.c_int64),
                ("uptr", C.c_void_p), ("uidx", C.c_void_p), ("uval", C.c_void_p),
                ("iptr", C.c_void_p), ("iidx", C.c_void_p), ("ival", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("n_f", C.c_int), ("max_iters", C.c_int),
                ("tol", C.c_double), ("seed", C.c_uint64), ("alpha0", C.c_double),
                ("armijo_c", C.c_double), ("tau", C.c_double), ("max_backtracks", C.c_int),
                ("n_blocks", C.c_int), ("n_workers", C.c_int), ("trace_every", C.c_int),
                ("snapshot_every", C.c_int), ("paper_timing", C.c_int),
                ("has_fixed_alpha", C.c_int), ("fixed_alpha", C.c_double),
                ("force_beta_zero", C.c_int)]


class TraceRec(C.Structure):
    _fields_ = [("iter", C.c_int), ("loss", C.c_double), ("grad_norm", C.c_double),
                ("elapsed_seconds", C.c_double), ("backtracks", C.c_int),
                ("shuffled_columns", C.c_int64), ("restarted", C.c_int)]


class Result(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("final_loss", C.c_double),
                ("final_grad_norm", C.c_double), ("restarts", C.c_int),
                ("fallback_steps", C.c_int), ("fallback_columns", C.c_int)]


class RngState(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int), ("has_spare", C.c_int),
                ("spare", C.c_double)]


def _build(target):
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            _build("port")
        lib = C.CDLL(PORT_SO)
        lib.orc_rng_seed.argtypes = [C.POINTER(RngState), C.c_uint64]
        lib.orc_rng_next.argtypes = [C.POINTER(RngState)]
        lib.orc_rng_next.restype = C.c_uint64
        lib.orc_rng_uniform.argtypes = [C.POINTER(RngState)]
        lib.orc_rng_uniform.restype = C.c_double
        lib.orc_rng_normal.argtypes = [C.POINTER(RngState)]
        lib.orc_rng_normal.restype = C.c_double
        lib.orc_rng_uniform_below.argtypes = [C.POINTER(RngState), C.c_uint64]
        lib.orc_rng_uniform_below.restype = C.c_uint64
        lib.orc_sample_cumulative.argtypes = [_dp, C.c_int, C.c_double]
        lib.orc_build.argtypes = [C.c_int, C.c_int, C.c_int64, _ip, _ip, _dp, C.c_int,
                                  _lp, _ip, _dp, _lp, _ip, _dp, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int)]
        lib.orc_random_init.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _dp, _dp]
        lib.orc_synth_generate.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_uint64,
                                           _ip, _ip, _dp]
        lib.orc_dot.argtypes = [C.c_int64, C.c_int64, _dp, _dp, _dp, _dp]
        lib.orc_dot.restype = C.c_double
        lib.orc_axpby.argtypes = [C.c_int64, C.c_int64, C.c_double, _dp, _dp, C.c_double,
                                  _dp, _dp, _dp, _dp]
        lib.orc_loss.argtypes = [C.POINTER(Ratings), C.c_int, _dp, _dp, C.c_double]
        lib.orc_loss.restype = C.c_double
        lib.orc_gradient.argtypes = [C.POINTER(Ratings), C.c_int, _dp, _dp, C.c_double,
                                     C.c_int, _dp, _dp]
        lib.orc_beta_bar.argtypes = [C.c_int64, C.c_int64] + [_dp] * 8
        lib.orc_beta_bar.restype = C.c_double
        lib.orc_quartic.argtypes = [C.POINTER(Ratings), C.c_int, _dp, _dp, _dp, _dp,
                                    C.c_double, C.c_int, C.c_int, _dp]
        lib.orc_backtracking.argtypes = [_dp, C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int)]
        lib.orc_update_users.argtypes = [C.POINTER(Ratings), C.c_int, _dp, C.c_double, C.c_int,
                                         _dp, C.POINTER(C.c_int)]
        lib.orc_update_items.argtypes = lib.orc_update_users.argtypes
        lib.orc_routing_totals.argtypes = [C.POINTER(Ratings), C.c_int, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]
        solve_args = [C.POINTER(Ratings), C.POINTER(Config), _dp, _dp, C.POINTER(TraceRec),
                      C.c_int, C.POINTER(C.c_int), C.POINTER(Result)]
        lib.orc_ncg_solve.argtypes = solve_args
        lib.orc_als_solve.argtypes = solve_args
        _port = lib
    return _port


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.ref_ratings_from_triples.argtypes = [C.c_int, C.c_int, C.c_int64, _ip, _ip, _dp,
                                                 C.c_int, C.POINTER(C.c_int),
                                                 C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.ref_ratings_from_triples.restype = C.c_void_p
        lib.ref_ratings_free.argtypes = [C.c_void_p]
        lib.ref_ratings_export.argtypes = [C.c_void_p, _lp, _ip, _dp, _lp, _ip, _dp]
        lib.ref_random_init.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _dp, _dp]
        lib.ref_rng_draws.argtypes = [C.c_uint64, C.c_int,
                                      np.ctypeslib.ndpointer(dtype=np.uint64), _dp, _dp]
        lib.ref_loss.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_double]
        lib.ref_loss.restype = C.c_double
        lib.ref_gradient.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_double, C.c_int,
                                     _dp, _dp]
        lib.ref_quartic.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, C.c_double,
                                    C.c_int, C.c_int, _dp]
        lib.ref_backtracking.argtypes = [_dp, C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int)]
        lib.ref_beta_bar.argtypes = [C.c_int, C.c_int, C.c_int] + [_dp] * 8
        lib.ref_beta_bar.restype = C.c_double
        lib.ref_dot.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        lib.ref_dot.restype = C.c_double
        lib.ref_half_sweep.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_double, C.c_int,
                                       C.c_int, _dp, C.POINTER(C.c_int)]
        lib.ref_routing_totals.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]
        solve_args = [C.c_void_p, C.POINTER(Config), _dp, _dp, C.POINTER(TraceRec), C.c_int,
                      C.POINTER(C.c_int), C.POINTER(Result)]
        lib.ref_ncg_solve.argtypes = solve_args
        lib.ref_als_solve.argtypes = solve_args
        _ref = lib
    return _ref


# --------------------------------------------------------------------------
class Rng:
    """alsncg::Rng (rng.hpp:26-45) on the oracle's mt19937_64."""

    def __init__(self, seed):
        self.s = RngState()
        port().orc_rng_seed(C.byref(self.s), seed)

    def next_u64(self):
        return port().orc_rng_next(C.byref(self.s))

    def uniform(self):
        return port().orc_rng_uniform(C.byref(self.s))

    def normal(self):
        return port().orc_rng_normal(C.byref(self.s))

    def uniform_below(self, n):
        return port().orc_rng_uniform_below(C.byref(self.s), n)


class OracleRatings:
    """CSR/CSC arrays built by the oracle's from_triples restatement."""

    def __init__(self, n_u, n_m, users, items, values, single=False):
        users = np.ascontiguousarray(users, dtype=np.int32)
        items = np.ascontiguousarray(items, dtype=np.int32)
        values = np.ascontiguousarray(values, dtype=np.float64)
        nnz = len(users)
        self.n_u, self.n_m, self.nnz = n_u, n_m, nnz
        self.uptr = np.zeros(max(n_u, 0) + 1, np.int64)
        self.iptr = np.zeros(max(n_m, 0) + 1, np.int64)
        self.uidx = np.zeros(max(nnz, 1), np.int32)
        self.iidx = np.zeros(max(nnz, 1), np.int32)
        self.uval = np.zeros(max(nnz, 1), np.float64)
        self.ival = np.zeros(max(nnz, 1), np.float64)
        du, di = C.c_int(-1), C.c_int(-1)
        st = port().orc_build(n_u, n_m, nnz, users if nnz else np.zeros(1, np.int32),
                              items if nnz else np.zeros(1, np.int32),
                              values if nnz else np.zeros(1), int(single), self.uptr,
                              self.uidx, self.uval, self.iptr, self.iidx, self.ival,
                              C.byref(du), C.byref(di))
        self.status, self.dup = st, (du.value, di.value)
        if st != 0:
            raise ValueError(f"oracle from_triples status {st}")
        self.uidx, self.iidx = self.uidx[:nnz], self.iidx[:nnz]
        self.uval, self.ival = self.uval[:nnz], self.ival[:nnz]
        self.triples = (users, items, values)
        self.s = Ratings(n_u, n_m, nnz, self.uptr.ctypes.data, self.uidx.ctypes.data,
                         self.uval.ctypes.data, self.iptr.ctypes.data, self.iidx.ctypes.data,
                         self.ival.ctypes.data)
        self._ref = None

    @classmethod
    def from_csr(cls, n_u, n_m, uptr, uidx, uval):
        users = np.repeat(np.arange(n_u, dtype=np.int32), np.diff(uptr))
        return cls(n_u, n_m, users, uidx, uval)

    def user_count(self):
        return np.diff(self.uptr)

    def item_count(self):
        return np.diff(self.iptr)

    def ref_handle(self):
        if self._ref is None:
            u, i, v = self.triples
            st, du, di = C.c_int(0), C.c_int(0), C.c_int(0)
            h = ref().ref_ratings_from_triples(self.n_u, self.n_m, self.nnz, u, i, v, 0,
                                               C.byref(st), C.byref(du), C.byref(di))
            assert st.value == 0
            self._ref = h
        return self._ref

    def __del__(self):
        if getattr(self, "_ref", None) is not None and _ref is not None:
            _ref.ref_ratings_free(self._ref)


def _split(x, n_f, n_u):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return x[: n_f * n_u], x[n_f * n_u:]


def _nonempty(a):
    return a if a.size else np.zeros(1)


def make_config(**kw):
    c = Config()
    defaults = dict(lambda_=0.1, n_f=10, max_iters=10000, tol=1e-6, seed=0, alpha0=10.0,
                    armijo_c=0.5, tau=0.9, max_backtracks=100, n_blocks=0, n_workers=1,
                    trace_every=1, snapshot_every=0, paper_timing=0, has_fixed_alpha=0,
                    fixed_alpha=0.0, force_beta_zero=0)
    defaults.update(kw)
    for k, v in defaults.items():
        setattr(c, k, v)
    return c


class Oracle:
    """Uniform facade over the port ("port") or the compiled reference ("ref")."""

    def __init__(self, kind="port"):
        self.kind = kind
        if kind == "ref" and not ref_available():
            raise RuntimeError("oracle/_ref not built")

    def random_init(self, n_f, n_u, n_m, seed):
        u = np.zeros(max(n_f * n_u, 1))
        m = np.zeros(max(n_f * n_m, 1))
        f = port().orc_random_init if self.kind == "port" else ref().ref_random_init
        f(n_f, n_u, n_m, seed, u, m)
        return np.concatenate([u[: n_f * n_u], m[: n_f * n_m]])

    def loss(self, R, n_f, x, lam):
        xu, xm = _split(x, n_f, R.n_u)
        if self.kind == "port":
            return port().orc_loss(C.byref(R.s), n_f, _nonempty(xu), _nonempty(xm), lam)
        return ref().ref_loss(R.ref_handle(), n_f, _nonempty(xu), _nonempty(xm), lam)

    def gradient(self, R, n_f, x, lam, n_workers=1):
        xu, xm = _split(x, n_f, R.n_u)
        gu, gm = np.zeros(max(xu.size, 1)), np.zeros(max(xm.size, 1))
        if self.kind == "port":
            port().orc_gradient(C.byref(R.s), n_f, _nonempty(xu), _nonempty(xm), lam,
                                n_workers, gu, gm)
        else:
            ref().ref_gradient(R.ref_handle(), n_f, _nonempty(xu), _nonempty(xm), lam,
                               n_workers, gu, gm)
        return np.concatenate([gu[: xu.size], gm[: xm.size]])

    def quartic(self, R, n_f, x, p, lam, n_chunks=1, n_workers=1):
        xu, xm = _split(x, n_f, R.n_u)
        pu, pm = _split(p, n_f, R.n_u)
        c = np.zeros(5)
        args = (n_f, _nonempty(xu), _nonempty(xm), _nonempty(pu), _nonempty(pm), lam,
                n_chunks, n_workers, c)
        if self.kind == "port":
            port().orc_quartic(C.byref(R.s), *args)
        else:
            ref().ref_quartic(R.ref_handle(), *args)
        return c

    def backtracking(self, c, slope, alpha0=10.0, cc=0.5, tau=0.9, max_bt=100):
        a, k = C.c_double(0), C.c_int(0)
        f = port().orc_backtracking if self.kind == "port" else ref().ref_backtracking
        st = f(np.ascontiguousarray(c, dtype=np.float64), slope, alpha0, cc, tau, max_bt,
               C.byref(a), C.byref(k))
        return st, a.value, k.value

    def half_sweep(self, R, users, n_f, src, lam, n_blocks=1, n_workers=1):
        src = np.ascontiguousarray(src, dtype=np.float64)
        n_dest = R.n_u if users else R.n_m
        out = np.zeros(max(n_f * n_dest, 1))
        fb = C.c_int(0)
        if self.kind == "port":
            f = port().orc_update_users if users else port().orc_update_items
            f(C.byref(R.s), n_f, _nonempty(src), lam, n_workers, out, C.byref(fb))
        else:
            ref().ref_half_sweep(R.ref_handle(), int(users), n_f, _nonempty(src), lam,
                                 n_blocks, n_workers, out, C.byref(fb))
        return out[: n_f * n_dest], fb.value

    def als_sweep(self, R, n_f, x, lam):
        nu = n_f * R.n_u
        users, _ = self.half_sweep(R, True, n_f, x[nu:], lam)
        items, _ = self.half_sweep(R, False, n_f, users, lam)
        return np.concatenate([users, items])

    def routing_totals(self, R, n_blocks):
        tu, tm = C.c_int64(0), C.c_int64(0)
        if self.kind == "port":
            port().orc_routing_totals(C.byref(R.s), n_blocks, C.byref(tu), C.byref(tm))
        else:
            ref().ref_routing_totals(R.ref_handle(), n_blocks, C.byref(tu), C.byref(tm))
        return tu.value, tm.value

    def _solve(self, which, R, cfg):
        n_f = cfg.n_f
        mu = np.zeros(max(n_f * R.n_u, 1))
        mm = np.zeros(max(n_f * R.n_m, 1))
        cap = cfg.max_iters + 2
        trace = (TraceRec * cap)()
        ln = C.c_int(0)
        res = Result()
        if self.kind == "port":
            f = port().orc_ncg_solve if which == "ncg" else port().orc_als_solve
            st = f(C.byref(R.s), C.byref(cfg), mu, mm, trace, cap, C.byref(ln), C.byref(res))
        else:
            f = ref().ref_ncg_solve if which == "ncg" else ref().ref_als_solve
            st = f(R.ref_handle(), C.byref(cfg), mu, mm, trace, cap, C.byref(ln), C.byref(res))
        if st != 0:
            raise ValueError("invalid SolverConfig")
        recs = [dict(iter=t.iter, loss=t.loss, grad_norm=t.grad_norm,
                     elapsed_seconds=t.elapsed_seconds, backtracks=t.backtracks,
                     shuffled_columns=t.shuffled_columns, restarted=bool(t.restarted))
                for t in trace[: min(ln.value, cap)]]
        x = np.concatenate([mu[: n_f * R.n_u], mm[: n_f * R.n_m]])
        return x, recs, dict(converged=bool(res.converged), iterations=res.iterations,
                             final_loss=res.final_loss, final_grad_norm=res.final_grad_norm,
                             restarts=res.restarts, fallback_steps=res.fallback_steps,
                             fallback_columns=res.fallback_columns)

    def ncg_solve(self, R, cfg):
        return self._solve("ncg", R, cfg)

    def als_solve(self, R, cfg):
        return self._solve("als", R, cfg)


# BASELINE.json workloads, restated on the oracle side (same table as the
# product's synth.CONFIGS; tests/test_golden.py pins the two generators
# bitwise) so that the reference arm never loads the product library.
# index -> (n_users, n_items, nnz, n_f, lambda, data seed)
CONFIGS = {
    0: dict(n_u=1_000, n_m=500, nnz=20_000, n_f=10, lam=0.1, seed=1000),
    1: dict(n_u=138_493, n_m=26_744, nnz=20_000_263, n_f=100, lam=0.01, seed=1001),
    2: dict(n_u=138_493, n_m=26_744, nnz=20_000_263, n_f=(10, 25, 50, 100, 200), lam=0.01,
            seed=1001),
    3: dict(n_u=1_000_000, n_m=100_000, nnz=100_000_000, n_f=50, lam=0.05, seed=1003),
    4: dict(n_u=8_000_000, n_m=800_000, nnz=960_000_000, n_f=25, lam=0.05, seed=1004),
}


def synth_triples(n_u, n_m, nnz, seed, min_per_user=20):
    """orc_synth_generate: the BASELINE workload recipe."""
    users = np.empty(nnz, np.int32)
    items = np.empty(nnz, np.int32)
    values = np.empty(nnz, np.float64)
    if port().orc_synth_generate(n_u, n_m, nnz, min_per_user, seed, users, items, values):
        raise ValueError("orc_synth_generate: bad dimensions or unreachable nnz")
    return users, items, values


def generate(config_index, scale_users=None):
    """OracleRatings of BASELINE config `config_index` (optionally only the
    first `scale_users` users' ratings, for bounded CPU samples)."""
    c = CONFIGS[config_index]
    users, items, values = synth_triples(c["n_u"], c["n_m"], c["nnz"], c["seed"])
    n_u = c["n_u"]
    if scale_users is not None and scale_users < n_u:
        keep = users < scale_users
        users, items, values = users[keep], items[keep], values[keep]
        n_u = scale_users
    return OracleRatings(n_u, c["n_m"], users, items, values)


def dot(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    e = np.zeros(1)
    return port().orc_dot(x.size, 0, _nonempty(x), e, _nonempty(y), e)


def beta_bar(gn, gp, bn, bp):
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (gn, gp, bn, bp)]
    e = np.zeros(1)
    return port().orc_beta_bar(arrs[0].size, 0, _nonempty(arrs[0]), e, _nonempty(arrs[1]), e,
                               _nonempty(arrs[2]), e, _nonempty(arrs[3]), e)


def ref_mean_ranking_accuracy(n_f, n_u, n_m, user_k, item_k, user_f, item_f, t, n_workers=1):
    """The reference's ranking::mean_ranking_accuracy (oracle/_ref)."""
    L = ref()
    L.ref_mean_ranking_accuracy.restype = C.c_double
    L.ref_mean_ranking_accuracy.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_int,
                                            C.c_int]
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (user_k, item_k, user_f, item_f)]
    return L.ref_mean_ranking_accuracy(n_f, n_u, n_m, *a, t, n_workers)
