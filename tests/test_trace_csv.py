"""Trace CSV (harness.cpp:80-127): the product's
writer is byte-identical to the reference's own write_trace_csv (oracle/_ref),
the reader round-trips every double exactly, and malformed files raise the
reference's DataError / logic_error.  Host-only (no GPU)."""
import ctypes as C

import numpy as np
import pytest

import paper_1508_03110_b200 as P
from oracle.pyoracle import ref, ref_available


def sample_trace(n=25, seed=3):
    rng = np.random.default_rng(seed)
    t = P.ConvergenceTrace()
    el = 0.0
    for i in range(n):
        el += float(rng.exponential(0.3))
        t.append(P.TraceRecord(iter=i, loss=float(rng.lognormal(8, 2)), grad_norm=float(rng.lognormal(-8, 3)),
                               elapsed_seconds=el, backtracks=int(rng.integers(0, 101)),
                               shuffled_columns=int(rng.integers(0, 2**40)), restarted=bool(i % 7 == 3)))
    return t


def test_roundtrip_exact(tmp_path):
    t = sample_trace()
    p = tmp_path / "trace.csv"
    P.harness.write_trace_csv(p, t)
    back = P.harness.read_trace_csv(p)
    assert len(back) == len(t)
    for a, b in zip(back.records, t.records):
        assert (a.iter, a.loss, a.grad_norm, a.elapsed_seconds, a.backtracks, a.shuffled_columns) == \
            (b.iter, b.loss, b.grad_norm, b.elapsed_seconds, b.backtracks, b.shuffled_columns)
    want = (t.records[-1].elapsed_seconds - t.records[0].elapsed_seconds) / (len(t) - 1)
    assert P.harness.mean_iteration_seconds(back) == want


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_bytes_equal_reference_writer(tmp_path):
    t = sample_trace(40, 9)
    mine, theirs = tmp_path / "mine.csv", tmp_path / "ref.csv"
    P.harness.write_trace_csv(mine, t)
    R = t.records
    L = ref()
    L.ref_write_trace_csv.argtypes = [C.c_char_p, C.c_int] + [C.c_void_p] * 6
    arrs = [np.array([r.iter for r in R], np.int32), np.array([r.loss for r in R]),
            np.array([r.grad_norm for r in R]), np.array([r.elapsed_seconds for r in R]),
            np.array([r.backtracks for r in R], np.int32),
            np.array([r.shuffled_columns for r in R], np.int64)]
    assert L.ref_write_trace_csv(str(theirs).encode(), len(R), *[a.ctypes.data for a in arrs]) == 0
    assert mine.read_bytes() == theirs.read_bytes()


def test_errors(tmp_path):
    with pytest.raises(P.DataError):
        P.harness.read_trace_csv(tmp_path / "missing.csv")
    bad = tmp_path / "bad.csv"
    bad.write_text("iter,loss,grad_norm,elapsed_s,backtracks,shuffled_columns\n0,1.0,2.0,0.0,0\n")
    with pytest.raises(P.DataError):
        P.harness.read_trace_csv(bad)
    bad.write_text("iter,loss,grad_norm,elapsed_s,backtracks,shuffled_columns\n0,1.0,x,0.0,0,0\n")
    with pytest.raises(P.DataError):
        P.harness.read_trace_csv(bad)
    bad.write_text("iter,loss,grad_norm,elapsed_s,backtracks,shuffled_columns\r\n\r\n")
    with pytest.raises(P.DataError):
        P.harness.read_trace_csv(bad)  # empty trace
    bad.write_text("iter,loss,grad_norm,elapsed_s,backtracks,shuffled_columns\n1,1,1,0,0,0\n1,1,1,0,0,0\n")
    with pytest.raises(AssertionError):
        P.harness.read_trace_csv(bad)  # ConvergenceTrace::append: iterations must increase
    with pytest.raises(P.DataError):
        P.harness.mean_iteration_seconds(P.ConvergenceTrace())
