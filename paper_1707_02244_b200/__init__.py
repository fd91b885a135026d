"""paper_1707_02244_b200 — B200-native circulant LASSO recovery engine.

A from-scratch sm_100a implementation of the ISTA and circulant-ADMM solvers
of arxiv 1707.02244 behind the reference ``circlasso`` solver API.  The
compute lives in ``_lib/libcirclasso_b200.so`` (C-ABI: include/circlasso_b200.h);
this package binds it with ctypes and mirrors the reference names.
"""
from .api import (  # noqa: F401
    AdmmState, ShardedSolve, read_pgm, write_pgm, admm_dense_run, admm_setup, admm_step, CadmmState, CapacityError, DeblurResult, GrayImage, deblur_recover, make_image, run_deblur_experiment, CirculantMatrix, CommError, ConsistencyError, CudaError, DiagonalOperator,
    DimensionError, DivergenceError, Error, FootprintKind, FormatError, IstaState, ParameterError, PartialCirculantOperator,
    PhaseError, RecoveryReport, SensingProblem, SingularityError, SolverConfig, SparseSignal, StopMetric,
    SubsamplingMask, ThresholdPairing, TracePoint, analytic_footprint, blur_matrix, cadmm_run, cadmm_setup,
    cadmm_step, circ_matvec, circ_transpose_matvec, compose_sensing, device_count, ffma_peak_tflops,
    gen_circulant_sensing, gen_sparse_signal, gen_star_field, ista_run, ista_setup, ista_step, make_problem,
    mask_gram_inverse, measure, mse, partial_matvec, partial_transpose_matvec, regularized_gram_inverse,
    soft_threshold, spectral_norm)
from ._native import LIB_PATH  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
