"""RatingsMatrix (ratings.hpp:50-105): immutable dual CSR/CSC store.

Construction goes through the product's C-ABI build (alsncg_csr_build),
bit-identical to RatingsMatrix::from_triples (ratings.cpp:28-89).  The device
copy is uploaded lazily, once per context.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import lib, ptr


class DataError(RuntimeError):
    """ratings.hpp:31-35."""


class DuplicateRatingError(DataError):
    """ratings.hpp:37-43."""

    def __init__(self, user, item):
        super().__init__(f"duplicate rating for user {user}, item {item}")
        self.user, self.item = user, item


@dataclass
class Rating:
    user: int = 0
    item: int = 0
    value: float = 0.0


class RatingsMatrix:
    def __init__(self):
        self._n_u = self._n_m = self._nnz = 0
        self._single = False
        self.uptr = np.zeros(1, np.int64)
        self.iptr = np.zeros(1, np.int64)
        self.uidx = np.zeros(0, np.int32)
        self.iidx = np.zeros(0, np.int32)
        self.uval = np.zeros(0)
        self.ival = np.zeros(0)
        self._dev = {}

    @staticmethod
    def from_triples(n_users, n_items, triples=None, single_precision_storage=False, *,
                     users=None, items=None, values=None):
        """triples: iterable of Rating / (user, item, value), or the three
        parallel arrays users/items/values."""
        if triples is not None:
            t = [(r.user, r.item, r.value) if isinstance(r, Rating) else tuple(r) for r in triples]
            users = np.array([a for a, _, _ in t], dtype=np.int32)
            items = np.array([b for _, b, _ in t], dtype=np.int32)
            values = np.array([c for _, _, c in t], dtype=np.float64)
        users = np.ascontiguousarray(users, dtype=np.int32)
        items = np.ascontiguousarray(items, dtype=np.int32)
        values = np.ascontiguousarray(values, dtype=np.float64)
        nnz = users.size
        if n_users < 0 or n_items < 0:
            raise DataError("negative matrix dimensions")
        r = RatingsMatrix()
        r._n_u, r._n_m, r._nnz, r._single = n_users, n_items, nnz, bool(single_precision_storage)
        r.uptr = np.zeros(n_users + 1, np.int64)
        r.iptr = np.zeros(n_items + 1, np.int64)
        r.uidx = np.zeros(nnz, np.int32)
        r.iidx = np.zeros(nnz, np.int32)
        r.uval = np.zeros(nnz)
        r.ival = np.zeros(nnz)
        du, di = C.c_int(-1), C.c_int(-1)
        st = lib().alsncg_csr_build(n_users, n_items, nnz, ptr(users), ptr(items), ptr(values),
                                    int(single_precision_storage), ptr(r.uptr), ptr(r.uidx),
                                    ptr(r.uval), ptr(r.iptr), ptr(r.iidx), ptr(r.ival),
                                    C.byref(du), C.byref(di))
        if st == _lib.EDUP:
            raise DuplicateRatingError(du.value, di.value)
        _lib.check(st)
        return r

    # -- accessors (ratings.hpp:62-90)
    def n_users(self):
        return self._n_u

    def n_items(self):
        return self._n_m

    def nnz(self):
        return self._nnz

    def user_count(self, i):
        return int(self.uptr[i + 1] - self.uptr[i])

    def item_count(self, j):
        return int(self.iptr[j + 1] - self.iptr[j])

    def user_items(self, i):
        return self.uidx[self.uptr[i]:self.uptr[i + 1]]

    def user_values(self, i):
        return self.uval[self.uptr[i]:self.uptr[i + 1]]

    def item_users(self, j):
        return self.iidx[self.iptr[j]:self.iptr[j + 1]]

    def item_values(self, j):
        return self.ival[self.iptr[j]:self.iptr[j + 1]]

    def single_precision_storage(self):
        return self._single

    def to_triples(self):
        users = np.repeat(np.arange(self._n_u, dtype=np.int32), np.diff(self.uptr))
        return [Rating(int(u), int(i), float(v)) for u, i, v in zip(users, self.uidx, self.uval)]

    def check_consistent(self):
        """ratings.cpp:103-132 (test support)."""
        if self.uptr[-1] != self._nnz or self.iptr[-1] != self._nnz:
            raise AssertionError("nnz mismatch")
        users = np.repeat(np.arange(self._n_u, dtype=np.int64), np.diff(self.uptr))
        items = np.repeat(np.arange(self._n_m, dtype=np.int64), np.diff(self.iptr))
        a = sorted(zip(users.tolist(), self.uidx.tolist(), self.uval.tolist()))
        b = sorted(zip(self.iidx.tolist(), items.tolist(), self.ival.tolist()))
        if a != b:
            raise AssertionError("views disagree")
        for i in range(self._n_u):
            if np.any(np.diff(self.user_items(i)) <= 0):
                raise AssertionError("user adjacency not sorted")
        for j in range(self._n_m):
            if np.any(np.diff(self.item_users(j)) <= 0):
                raise AssertionError("item adjacency not sorted")

    # -- device residency
    def device(self, ctx=None):
        """alsncg_ratings handle for ctx (uploaded once)."""
        from .device import default_context
        ctx = ctx or default_context()
        key = id(ctx)
        if key not in self._dev:
            h = C.c_void_p()
            _lib.check(lib().alsncg_ratings_upload(
                ctx.handle, self._n_u, self._n_m, self._nnz, ptr(self.uptr), ptr(self.uidx),
                ptr(self.uval), ptr(self.iptr), ptr(self.iidx), ptr(self.ival), C.byref(h)))
            self._dev[key] = (ctx, h)
        return self._dev[key][1]

    def release_device(self):
        for ctx, h in self._dev.values():
            if ctx.handle:
                lib().alsncg_ratings_free(h)
        self._dev = {}

    def __del__(self):
        try:
            self.release_device()
        except Exception:
            pass
