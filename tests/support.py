"""Seeded generators and independent oracles shared by the test suites.

Python restatement of the reference's tests/support.hpp (the generators draw
from the oracle's mt19937_64 ``Rng``, so the instances are the reference
tests' own instances, draw for draw).  Test infrastructure only.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.pyoracle import Rng  # noqa: E402


class Triples:
    def __init__(self, n_u, n_m, users, items, values):
        self.n_u, self.n_m = n_u, n_m
        self.users = np.asarray(users, dtype=np.int32)
        self.items = np.asarray(items, dtype=np.int32)
        self.values = np.asarray(values, dtype=np.float64)

    def __len__(self):
        return len(self.users)


def random_ratings(n_u, n_m, density, seed, lo=0.5, hi=5.0):
    """support.hpp:42-52: Bernoulli(density) pattern, values U[lo,hi]."""
    rng = Rng(seed)
    us, its, vs = [], [], []
    for i in range(n_u):
        for j in range(n_m):
            if rng.uniform() < density:
                us.append(i)
                its.append(j)
                vs.append(lo + (hi - lo) * rng.uniform())
    if not us:
        us, its, vs = [0], [0], [lo]
    return Triples(n_u, n_m, us, its, vs)


def rank_one_ratings(n_u, n_m, seed):
    """support.hpp:55-64."""
    rng = Rng(seed)
    u = [0.5 + rng.uniform() for _ in range(n_u)]
    m = [0.5 + rng.uniform() for _ in range(n_m)]
    us, its, vs = [], [], []
    for i in range(n_u):
        for j in range(n_m):
            us.append(i)
            its.append(j)
            vs.append(u[i] * m[j])
    return Triples(n_u, n_m, us, its, vs)


def _round_half_away(x):
    return math.floor(x + 0.5) if x >= 0 else -math.floor(-x + 0.5)


def movielens_like(n_u, n_m, density, seed, latent_rank=10):
    """support.hpp:70-109."""
    from oracle.pyoracle import port
    rng = Rng(seed)
    a = [rng.uniform() for _ in range(n_u * latent_rank)]
    b = [rng.uniform() for _ in range(n_m * latent_rank)]
    cum = np.zeros(n_m)
    run = 0.0
    for j in range(n_m):
        run += math.pow(float(j + 1), -0.7)
        cum[j] = run
    stamp = [-1] * n_m
    us, its, vs = [], [], []
    lib = port()
    for i in range(n_u):
        spread = math.exp(0.35 * rng.normal())
        count = int(_round_half_away(density * n_m * spread))
        count = min(max(count, 1), n_m)
        drawn = 0
        while drawn < count:
            j = lib.orc_sample_cumulative(cum, n_m, rng.uniform())
            if stamp[j] == i:
                continue
            stamp[j] = i
            drawn += 1
            score = 0.0
            for k in range(latent_rank):
                score += a[i * latent_rank + k] * b[j * latent_rank + k]
            value = 0.5 + 4.5 * score / latent_rank + 0.35 * rng.normal()
            value = min(max(_round_half_away(value * 2.0) / 2.0, 0.5), 5.0)
            us.append(i)
            its.append(j)
            vs.append(value)
    return Triples(n_u, n_m, us, its, vs)


def random_flat(n_f, n_u, n_m, seed, lo=-1.0, hi=1.0):
    """support.hpp:111-118 (user part then item part)."""
    rng = Rng(seed)
    n = n_f * (n_u + n_m)
    return np.array([lo + (hi - lo) * rng.uniform() for _ in range(n)])


def random_model(n_f, n_u, n_m, seed, lo=-1.0, hi=1.0):
    """support.hpp:120-127 -> (user_data, item_data)."""
    x = random_flat(n_f, n_u, n_m, seed, lo, hi)
    return x[: n_f * n_u].copy(), x[n_f * n_u:].copy()


def naive_loss(x, T, n_f, lam, dtype=np.float64):
    """support.hpp:131-159 (dtype=np.longdouble gives naive_loss_ld)."""
    x = np.asarray(x, dtype=dtype)
    U = x[: n_f * T.n_u].reshape(T.n_u, n_f)
    M = x[n_f * T.n_u:].reshape(T.n_m, n_f)
    pred = np.einsum("ij,ij->i", U[T.users], M[T.items])
    e = T.values.astype(dtype) - pred
    total = np.sum(e * e)
    cu = np.bincount(T.users, minlength=T.n_u).astype(dtype)
    cm = np.bincount(T.items, minlength=T.n_m).astype(dtype)
    total += dtype(lam) * np.sum(cu * np.sum(U * U, axis=1))
    total += dtype(lam) * np.sum(cm * np.sum(M * M, axis=1))
    return total


def fd_gradient(x, T, n_f, lam):
    """support.hpp:198-213: central differences on the long-double loss."""
    g = np.zeros_like(x)
    probe = np.array(x, dtype=np.float64)
    for k in range(x.size):
        xk = x[k]
        h = 1e-6 * (1.0 + abs(xk))
        probe[k] = xk + h
        up = naive_loss(probe, T, n_f, lam, np.longdouble)
        probe[k] = xk - h
        down = naive_loss(probe, T, n_f, lam, np.longdouble)
        probe[k] = xk
        g[k] = float((up - down) / (np.longdouble(2.0) * np.longdouble(h)))
    return g


def ulps_between(a, b):
    """support.hpp:216-224."""
    if a == b:
        return 0

    def ordered(v):
        bits = int(np.array(v, dtype=np.float64).view(np.int64))
        return bits if bits >= 0 else -(2 ** 63) - bits

    return abs(ordered(a) - ordered(b))
