"""BASELINE.json workloads (seeded synthetic stand-ins).

Config 1 has MovieLens-20M's shape; the dataset itself is not available, so
the generator (alsncg_synth_generate: rank-10 truth, Zipf(1) items, >= 20
ratings per user, half-star values) produces a matrix of that shape.
"""
from __future__ import annotations

import numpy as np

from ._lib import check, lib, ptr
from .ratings import RatingsMatrix

# index -> (n_users, n_items, nnz, n_f, lambda, data seed)
CONFIGS = {
    0: dict(n_u=1_000, n_m=500, nnz=20_000, n_f=10, lam=0.1, seed=1000),
    1: dict(n_u=138_493, n_m=26_744, nnz=20_000_263, n_f=100, lam=0.01, seed=1001),
    2: dict(n_u=138_493, n_m=26_744, nnz=20_000_263, n_f=(10, 25, 50, 100, 200), lam=0.01,
            seed=1001),
    3: dict(n_u=1_000_000, n_m=100_000, nnz=100_000_000, n_f=50, lam=0.05, seed=1003),
    4: dict(n_u=8_000_000, n_m=800_000, nnz=960_000_000, n_f=25, lam=0.05, seed=1004),
}


def generate_triples(n_u, n_m, nnz, seed, min_per_user=20):
    users = np.empty(nnz, np.int32)
    items = np.empty(nnz, np.int32)
    values = np.empty(nnz, np.float64)
    check(lib().alsncg_synth_generate(n_u, n_m, nnz, min_per_user, seed, ptr(users), ptr(items),
                                      ptr(values)))
    return users, items, values


def generate(config_index, scale_users=None):
    """RatingsMatrix of BASELINE config `config_index` (optionally only the
    first `scale_users` users' worth of ratings, for bounded CPU samples)."""
    c = CONFIGS[config_index]
    users, items, values = generate_triples(c["n_u"], c["n_m"], c["nnz"], c["seed"])
    n_u = c["n_u"]
    if scale_users is not None and scale_users < n_u:
        keep = users < scale_users
        users, items, values = users[keep], items[keep], values[keep]
        n_u = scale_users
    return RatingsMatrix.from_triples(n_u, c["n_m"], users=users, items=items, values=values)
