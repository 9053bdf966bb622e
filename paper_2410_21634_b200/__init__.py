"""B200-native local diffusion (arXiv 2410.21634): LocalGD / LocalCH /
LocalSOR / heat-kernel push / warm-started repair on sm_100a, plus batched
multi-seed solves.  Drop-in for the reference package's solver entry points.
"""

from .graph import (CsrGraph, EdgeEvent, apply_event, apply_events, csr_from_pairs,
                    from_edges, load_edge_list, spectral_norm_estimate, volume)
from .systems import (DiffusionSystem, OperatorQ, SystemError, dense_solve,
                      make_generalized_system, make_hk_system, make_katz_system,
                      make_ppr_system, series_oracle)
from .reports import LocalReport, SolveReport, SolverState
from .metrics import error_norms, sample_sources
from .local_solvers import (local_ch, local_gd, local_gs, local_hb, local_hk, local_sor, optimal_omega,
                            push_sweeps)
from .global_solvers import GlobalConfig, gradient_descent
from .dynamic import PprPair, event_adjust, make_pair, parse_events, repair, run_snapshots
from .batch import BatchOutput, BatchSolver, local_gd_batch, local_sor_batch

__version__ = "0.1.0"
