"""B200-native (sm_100a) dual-domain convolutional sparse coding hot path.

The product is the in-tree CUDA library lib/libdcsc_cuda.so (C-ABI in
include/dcsc_cuda.h); dcsc.py mirrors the reference solver API over it.
"""
from .dcsc import (CodingDualState, Context, LearningDualState, SolverConfig, evaluate_objective,
                   forward_dft2, inverse_dft2, run_csc, solve_coding, solve_learning, synth_generate)

__all__ = ["CodingDualState", "Context", "LearningDualState", "SolverConfig", "evaluate_objective",
           "forward_dft2", "inverse_dft2", "run_csc", "solve_coding", "solve_learning", "synth_generate"]
