"""B200-native Gaussian belief propagation: the synchronous sweep path of the
reference ``gabp`` package (arXiv 0810.1119), on hand-written sm_100a CUDA kernels.

Public names mirror the reference package (/root/reference/pkg/src/gabp/__init__.py)
for the path this package covers; see DESIGN.md for scope.
"""

from .graph import (DegenerateProductError, GaussianGraph, ScalarGaussian, build_graph,
                    gaussian_product)
from .linalg import (MatrixMarketError, RectMatrix, SingularMatrixError, SymSystem,
                     ZeroDiagonalError, dominance_class, parse_matrix_market, parse_vector,
                     residual_norm_per_eq, spectral_radius_gabp_test, system_from_matrix_market,
                     write_matrix_market, write_vector)
from .problems import (CONFIGS, ProblemInstance, decorrelator_detect, gen_cdma,
                       gen_cdma_detection, gen_nonpsd3, gen_poisson, gen_poisson2d,
                       gen_poisson3d, gen_random, gen_random_sparse, gen_toy3, load_instance)
from .solver import (SCHEDULES, MeansHistory, MessageState, SingularSubgraphError,
                     SolveOptions, SolveReport, broadcast_sweep, compute_message,
                     compute_message_max_product, infer_marginals, initial_state, solve,
                     solve_graph, sweep)

__all__ = [name for name in dir() if not name.startswith("_")]
