"""flowfem_b200: B200-native adaptive-alpha Horn-Schunck + illumination optical-flow solver
(arXiv 1508.02977), P1 FEM on the pixel triangulation, additive-Schwarz-preconditioned CG
with batched banded-Cholesky subdomain solves in hand-written sm_100a CUDA.

The C-ABI (include/flowfem_b200.h) is the drop-in boundary; ``flowfem`` mirrors the
reference's ``flowfem::`` API on top of it.
"""
from .flowfem import (AdaptConfig, Context, DataTerms, DerivativeField, FlowfemError,
                      FlowState, IndicatorField, Partition, RegField, RunConfig, RunResult,
                      SchwarzOptions, SchwarzSolver, SchwarzStats, SplitChoice, assemble_apply, assign_workers,
                      build_data_terms, build_partition, choose_split, compute_derivatives,
                      default_context, enumerate_splits, error_indicator, frames_to_terms,
                      gaussian_smooth, kernel_launches, run_on_frames, run_on_frames_device,
                      schwarz_solve, SolveMethod, SolverConfig, SolveReport, SparseSystem,
                      spmv, rcm_order, cg_solve, solve, load_image, save_pgm, FloField,
                      read_flo, write_flo, to_flo, FlowMetrics, compute_metrics,
                      PipelineConfig, PipelineResult, run_pipeline,
                      uniform_reg, update_alpha)

__all__ = [n for n in dir() if not n.startswith("_")]
