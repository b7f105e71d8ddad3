"""Device context (one per GPU per process) and device buffers."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._lib import check, lib, ptr


class Context:
    """alsncg_ctx: device, CUDA stream, optional NCCL communicator."""

    def __init__(self, device=0, rank=0, world=1, nccl_id=None):
        h = C.c_void_p()
        if world > 1:
            buf = (C.c_ubyte * 128).from_buffer_copy(bytes(nccl_id))
            check(lib().alsncg_ctx_create_dist(device, rank, world, buf, C.byref(h)))
        else:
            check(lib().alsncg_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device, self.rank, self.world = device, rank, world

    @classmethod
    def loopback(cls, device, rank, group):
        """Rank `rank` of an in-process LoopGroup (testing aid: the sharded
        path on one GPU, one host thread per rank)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        check(lib().alsncg_ctx_create_loopback(device, rank, group.handle, C.byref(h)))
        self.handle = h
        self.device, self.rank, self.world = device, rank, group.world
        self._group = group  # keep the group alive as long as its ranks
        return self

    @staticmethod
    def nccl_unique_id():
        buf = (C.c_ubyte * 128)()
        check(lib().alsncg_nccl_unique_id(buf))
        return bytes(buf)

    @property
    def stream(self):
        return lib().alsncg_ctx_stream(self.handle)

    def synchronize(self):
        check(lib().alsncg_ctx_synchronize(self.handle))

    def set_profiling(self, on):
        check(lib().alsncg_ctx_set_profiling(self.handle, int(on)))

    def reset_stats(self):
        check(lib().alsncg_ctx_reset_stats(self.handle))

    def launches(self):
        return lib().alsncg_ctx_launches(self.handle)

    def kernel_stats(self):
        """{kernel name: (launches, total ms)} from per-launch CUDA events."""
        out = {}
        n = lib().alsncg_ctx_stat_count(self.handle)
        for k in range(max(n, 0)):
            name, cnt, ms = C.c_char_p(), C.c_int64(), C.c_double()
            check(lib().alsncg_ctx_stat(self.handle, k, C.byref(name), C.byref(cnt), C.byref(ms)))
            out[name.value.decode()] = (cnt.value, ms.value)
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib().alsncg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopGroup:
    """alsncg_loopgroup: in-process stand-in for an NCCL communicator (tests)."""

    def __init__(self, world):
        h = C.c_void_p()
        check(lib().alsncg_loopgroup_create(world, C.byref(h)))
        self.handle, self.world = h, world

    def __del__(self):
        try:
            if self.handle:
                lib().alsncg_loopgroup_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class DeviceBuffer:
    """Raw device allocation owned by a Context (float64 elements)."""

    def __init__(self, ctx, n):
        self.ctx, self.n = ctx, int(n)
        p = C.c_void_p()
        check(lib().alsncg_dev_malloc(ctx.handle, max(self.n, 1) * 8, C.byref(p)))
        self.ptr = p

    @classmethod
    def from_array(cls, ctx, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = cls(ctx, a.size)
        if a.size:
            check(lib().alsncg_memcpy_h2d(ctx.handle, b.ptr, ptr(a), a.nbytes))
        return b

    def to_array(self):
        out = np.empty(self.n)
        if self.n:
            check(lib().alsncg_memcpy_d2h(self.ctx.handle, ptr(out), self.ptr, out.nbytes))
        return out

    def free(self):
        if getattr(self, "ptr", None) is not None and self.ctx.handle:
            lib().alsncg_dev_free(self.ctx.handle, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


_default = {}


def default_context():
    """Process-wide context on ALSNCG_DEVICE (default 0)."""
    dev = int(os.environ.get("ALSNCG_DEVICE", "0"))
    if dev not in _default:
        _default[dev] = Context(dev)
    return _default[dev]


def row_stride(n_f):
    return lib().alsncg_row_stride(n_f)
