"""FactorModel / FlatVector and the vector operations (factors.hpp:24-91).

axpby/dot/norm run on the device kernels (k_vec.cu): axpby is bitwise the
reference's a*x + b*y; dot/norm follow the reference's index order bit for bit.
"""
from __future__ import annotations

import math

import numpy as np

from ._lib import check, lib, ptr


class FactorModel:
    """Column-major factors: user_data is n_f x n_u, item_data n_f x n_m."""

    def __init__(self, n_f=0, n_u=0, n_m=0):
        self.n_f, self.n_u, self.n_m = n_f, n_u, n_m
        self.user_data = np.zeros(n_f * n_u)
        self.item_data = np.zeros(n_f * n_m)

    def user_col(self, i):
        return self.user_data[i * self.n_f:(i + 1) * self.n_f]

    def item_col(self, j):
        return self.item_data[j * self.n_f:(j + 1) * self.n_f]


class FlatVector:
    """x = [u_1 .. u_{n_u}, m_1 .. m_{n_m}] stored as two segments."""

    def __init__(self, n_f=0, n_u=0, n_m=0, user_part=None, item_part=None):
        self.n_f, self.n_u, self.n_m = n_f, n_u, n_m
        self.user_part = (np.zeros(n_f * n_u) if user_part is None
                          else np.ascontiguousarray(user_part, dtype=np.float64))
        self.item_part = (np.zeros(n_f * n_m) if item_part is None
                          else np.ascontiguousarray(item_part, dtype=np.float64))

    @staticmethod
    def zeros(n_f, n_u, n_m):
        return FlatVector(n_f, n_u, n_m)

    @staticmethod
    def from_array(x, n_f, n_u, n_m):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return FlatVector(n_f, n_u, n_m, x[:n_f * n_u].copy(), x[n_f * n_u:].copy())

    def size(self):
        return self.n_f * (self.n_u + self.n_m)

    def same_shape(self, o):
        return (self.n_f, self.n_u, self.n_m) == (o.n_f, o.n_u, o.n_m)

    def array(self):
        return np.concatenate([self.user_part, self.item_part])

    def user_col(self, i):
        return self.user_part[i * self.n_f:(i + 1) * self.n_f]

    def item_col(self, j):
        return self.item_part[j * self.n_f:(j + 1) * self.n_f]

    def at(self, k):
        split = self.n_f * self.n_u
        if k < 0 or k >= self.size():
            raise IndexError("FlatVector::at")
        return self.user_part[k] if k < split else self.item_part[k - split]

    def set(self, k, v):
        split = self.n_f * self.n_u
        if k < 0 or k >= self.size():
            raise IndexError("FlatVector::set")
        if k < split:
            self.user_part[k] = v
        else:
            self.item_part[k - split] = v


def random_init(n_f, n_u, n_m, seed):
    """factors.cpp:24-32 (host mt19937_64 stream, items first)."""
    if n_f < 1:
        raise ValueError("random_init: n_f must be >= 1")
    m = FactorModel(n_f, n_u, n_m)
    u = np.zeros(max(n_f * n_u, 1))
    it = np.zeros(max(n_f * n_m, 1))
    check(lib().alsncg_random_init(n_f, n_u, n_m, seed, ptr(u), ptr(it)))
    m.user_data, m.item_data = u[:n_f * n_u].copy(), it[:n_f * n_m].copy()
    return m


def flatten(model):
    return FlatVector(model.n_f, model.n_u, model.n_m, model.user_data.copy(),
                      model.item_data.copy())


def unflatten(x):
    m = FactorModel()
    m.n_f, m.n_u, m.n_m = x.n_f, x.n_u, x.n_m
    m.user_data, m.item_data = x.user_part.copy(), x.item_part.copy()
    return m


def _dev_pair(x, y, ctx):
    from .device import DeviceBuffer
    return DeviceBuffer.from_array(ctx, x.array()), DeviceBuffer.from_array(ctx, y.array())


def axpby(a, x, b, y, ctx=None):
    """a*x + b*y componentwise on the device (factors.cpp:80-93)."""
    from .device import DeviceBuffer, default_context
    if not x.same_shape(y):
        raise ValueError("axpby: shape mismatch")
    ctx = ctx or default_context()
    dx, dy = _dev_pair(x, y, ctx)
    out = DeviceBuffer(ctx, x.size())
    check(lib().alsncg_dev_axpby(ctx.handle, x.size(), a, dx.ptr, b, dy.ptr, out.ptr))
    return FlatVector.from_array(out.to_array(), x.n_f, x.n_u, x.n_m)


def dot(x, y, ctx=None):
    """Euclidean inner product in the reference's index order (factors.cpp:95-103,
    bit-identical; the fused driver uses the compensated k_vec reductions)."""
    import ctypes as C
    from .device import default_context
    if not x.same_shape(y):
        raise ValueError("dot: shape mismatch")
    ctx = ctx or default_context()
    dx, dy = _dev_pair(x, y, ctx)
    out = C.c_double()
    check(lib().alsncg_dev_dot_seq(ctx.handle, x.size(), dx.ptr, dy.ptr, C.byref(out)))
    return out.value


def norm(x, ctx=None):
    return math.sqrt(dot(x, x, ctx))
