"""B200-native ALS-NCG core (arXiv 1508.03110): the data-parallel hot path
(ALS half-sweep, objective gradient, one-pass quartic line search, fused NCG
vector work) as sm_100a CUDA kernels behind the reference's solver API.

Python mirror of /root/reference/proj/include/alsncg (module per header);
every compute call goes through the C-ABI in include/alsncg_capi.h.
"""
from . import als, config, factors, harness, linesearch, ncg, ranking, ratings  # noqa: F401
from ._lib import LIB_PATH, AlsncgError, lib  # noqa: F401
from .config import ConvergenceTrace, QuarticPoly, SolveResult, SolverConfig, TraceRecord  # noqa: F401
from .device import Context, DeviceBuffer, LoopGroup, default_context, row_stride  # noqa: F401
from .factors import FactorModel, FlatVector, axpby, dot, flatten, norm, random_init, unflatten  # noqa: F401
from .ratings import DataError, DuplicateRatingError, Rating, RatingsMatrix  # noqa: F401
from .synth import CONFIGS, generate  # noqa: F401
