"""B200-native lagged, graph-ordered upwind-DG S_N transport sweep
(arXiv 1810.11080), behind the reference's SweepSolver interface.

The product is ``lib/libhosweep_b200.so`` (CUDA sm_100a kernels + C++ host
setup, C ABI in ``include/hosweep_b200.h``); this package is its host-side
Python mirror (``SweepSolver``) and the synthetic-config input construction.
"""
from .problem import Problem, config, CONFIG_NAMES  # noqa: F401
from .solver import (  # noqa: F401
    SolveOptions, SweepOrdering, SolverState, ConvergenceHistory, BalanceReport, SweepSolver,
    balance_report, SolverError, MeshError, GeometryError, AssemblyError, HswError,
)
from .mesh_io import read_mesh, write_mesh, mesh_from_json, mesh_to_json, problem_from_mesh  # noqa: F401

__version__ = "0.1.0"
