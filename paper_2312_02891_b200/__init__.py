"""B200-native inner-solve hot path of inexact low-rank Sylvester ADI
(arXiv 2312.02891), behind the reference package's (``sylvadi``) API.

The product path is CUDA only (libsylvadi_b200.so, sm_100a); there is no CPU
fallback.  Importing this package does not touch the GPU.
"""

from . import _lib
from .adi import (C_BOUND, CSV_HEADER, AdiConfig, AdiState, DeviceAdi, LowRankSolution,
                  SolveReport, StepRecord, Strategy, SylvesterProblem, ToleranceDecision,
                  block_norm, choose_tolerances, computed_residual_norm, gamma, run,
                  run_with_state, tolB_from_tolA, tolerance_budget)
from .device import DeviceMatrix, DeviceOperator, GmresWorkspace, axpy, gram
from .krylov import (DeviceSolveResult, GpuGmresBinding, InnerSolveResult, SolverBindings,
                     make_gpu_bindings)
from .shifts import ShiftSequence

__version__ = "0.1.0"


def library_path():
    return _lib.LIB_PATH
