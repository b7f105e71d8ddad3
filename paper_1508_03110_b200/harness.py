"""alsncg::harness trace CSV (harness.hpp:68-72, harness.cpp:80-127) -- the
file cmd_train writes per run and speedup / rank-eval read back.  Host-only
(no device); the rest of the reference harness is out of scope."""
from __future__ import annotations

import ctypes as C

from ._lib import TraceRecordC, check, lib
from .config import ConvergenceTrace, TraceRecord


def write_trace_csv(path, trace):
    recs = trace.records if isinstance(trace, ConvergenceTrace) else list(trace)
    arr = (TraceRecordC * max(len(recs), 1))()
    for i, r in enumerate(recs):
        arr[i] = TraceRecordC(r.iter, r.loss, r.grad_norm, r.elapsed_seconds, r.backtracks,
                              r.shuffled_columns, int(r.restarted))
    check(lib().alsncg_write_trace_csv(str(path).encode(), C.cast(arr, C.c_void_p), len(recs)))


def read_trace_csv(path):
    n = C.c_int(0)
    check(lib().alsncg_read_trace_csv(str(path).encode(), None, 0, C.byref(n)))
    arr = (TraceRecordC * max(n.value, 1))()
    check(lib().alsncg_read_trace_csv(str(path).encode(), C.cast(arr, C.c_void_p), n.value, C.byref(n)))
    t = ConvergenceTrace()
    for r in arr[: n.value]:
        t.append(TraceRecord(iter=r.iter, loss=r.loss, grad_norm=r.grad_norm,
                             elapsed_seconds=r.elapsed_seconds, backtracks=r.backtracks,
                             shuffled_columns=r.shuffled_columns, restarted=bool(r.restarted)))
    return t


def mean_iteration_seconds(trace):
    """harness.cpp:120-127."""
    if not len(trace):
        from .ratings import DataError
        raise DataError("mean_iteration_seconds: empty trace")
    a, b = trace.records[0], trace.records[-1]
    if a.iter == b.iter:
        return 0.0
    return (b.elapsed_seconds - a.elapsed_seconds) / (b.iter - a.iter)
