"""SolverConfig, trace and result types (config.hpp:29-98, config.cpp)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

from . import _lib
from .factors import FactorModel


@dataclass
class SolverConfig:
    lambda_: float = 0.1
    n_f: int = 10
    max_iters: int = 10000
    tol: float = 1e-6
    seed: int = 0
    alpha0: float = 10.0
    armijo_c: float = 0.5
    tau: float = 0.9
    max_backtracks: int = 100
    n_blocks: int = 0
    n_workers: int = 1
    trace_every: int = 1
    snapshot_every: int = 0
    paper_timing: bool = False

    def validate(self):  # config.cpp:21-34
        def bad(what):
            raise ValueError("SolverConfig: " + what)
        if self.lambda_ < 0.0:
            bad("lambda must be >= 0")
        if self.n_f < 1:
            bad("n_f must be >= 1")
        if self.max_iters < 0:
            bad("max_iters must be >= 0")
        if self.alpha0 <= 0.0:
            bad("alpha0 must be > 0")
        if not (0.0 < self.armijo_c < 1.0):
            bad("armijo_c must be in (0,1)")
        if not (0.0 < self.tau < 1.0):
            bad("tau must be in (0,1)")
        if self.max_backtracks < 0:
            bad("max_backtracks must be >= 0")
        if self.n_blocks < 0:
            bad("n_blocks must be >= 0 (0 = use n_workers)")
        if self.n_workers < 1:
            bad("n_workers must be >= 1")
        if self.trace_every < 1:
            bad("trace_every must be >= 1")
        if self.snapshot_every < 0:
            bad("snapshot_every must be >= 0")

    def resolved_blocks(self):
        return self.n_blocks if self.n_blocks > 0 else (self.n_workers if self.n_workers > 0 else 1)

    def to_c(self, fixed_alpha=None, force_beta_zero=False):
        c = _lib.Config()
        c.lambda_, c.n_f, c.max_iters, c.tol, c.seed = (self.lambda_, self.n_f, self.max_iters,
                                                        self.tol, self.seed)
        c.alpha0, c.armijo_c, c.tau = self.alpha0, self.armijo_c, self.tau
        c.max_backtracks, c.n_blocks, c.n_workers = (self.max_backtracks, self.n_blocks,
                                                     self.n_workers)
        c.trace_every, c.snapshot_every = self.trace_every, self.snapshot_every
        c.paper_timing = int(bool(self.paper_timing))
        c.has_fixed_alpha = int(fixed_alpha is not None)
        c.fixed_alpha = float(fixed_alpha or 0.0)
        c.force_beta_zero = int(bool(force_beta_zero))
        return c


@dataclass
class TraceRecord:
    iter: int = 0
    loss: float = 0.0
    grad_norm: float = 0.0
    elapsed_seconds: float = 0.0
    backtracks: int = 0
    shuffled_columns: int = 0
    restarted: bool = False


@dataclass
class ConvergenceTrace:
    records: List[TraceRecord] = field(default_factory=list)

    def append(self, rec):  # config.cpp:36-44
        if self.records:
            if rec.iter <= self.records[-1].iter:
                raise AssertionError("ConvergenceTrace: iterations must be strictly increasing")
            if rec.elapsed_seconds < self.records[-1].elapsed_seconds:
                raise AssertionError("ConvergenceTrace: elapsed time must be non-decreasing")
        self.records.append(rec)

    def __len__(self):
        return len(self.records)

    def __getitem__(self, k):
        return self.records[k]

    def back(self):
        return self.records[-1]


@dataclass
class QuarticPoly:
    c: List[float] = field(default_factory=lambda: [0.0] * 5)

    def __call__(self, alpha):  # config.hpp:79-81 (Horner)
        c = self.c
        return (((c[4] * alpha + c[3]) * alpha + c[2]) * alpha + c[1]) * alpha + c[0]


@dataclass
class SolveResult:
    model: Optional[FactorModel] = None
    trace: ConvergenceTrace = field(default_factory=ConvergenceTrace)
    converged: bool = False
    iterations: int = 0
    final_loss: float = 0.0
    final_grad_norm: float = 0.0
    restarts: int = 0
    fallback_steps: int = 0
    fallback_columns: int = 0
