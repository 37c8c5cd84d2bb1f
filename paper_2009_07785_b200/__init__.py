"""B200-native domain propagation (arXiv 2009.07785, GPU-atomic algorithm).

Drop-in for the reference `propgate` propagator API (propagate_parallel /
propagate_round_parallel, with propagate_sequential's verdicts); the compute
runs in hand-written sm_100a CUDA kernels behind the C-ABI in
include/propgate_b200.h.
"""
from .model import (EngineConfig, LoopMode, PropagationResult, PropagationStatus,  # noqa: F401
                    ProblemInstance, ScalarMode, SparseMatrix, VariableBounds, kInf)
