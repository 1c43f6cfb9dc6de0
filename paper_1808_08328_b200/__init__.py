"""B200-native (sm_100a, FP64) DPP assemble + field-split GMRES solver.

Drop-in for the hot path of the reference package `dppflow` (arXiv
1808.08328): the same public names (reference src/dppflow/__init__.py:4-38)
for meshes, assembly, the PETSc-style split options and the solver, backed by
hand-written CUDA kernels in libdpp.so (csrc/, C ABI in include/dpp.h).
There is no CPU fallback: without libdpp.so or a CUDA device the compute
entry points raise DeviceUnavailable.
"""

from ._native import DeviceUnavailable, ZeroPivotError
from .assembly import BlockSystem, DiscreteField, assemble, monolithic_view, solution_fields
from .blocksolve import (
    FIELD_SPLIT_OPTIONS,
    SCALE_SPLIT_OPTIONS,
    OptionError,
    SolveReport,
    SolverConfig,
    build_field_split,
    build_preconditioner,
    build_scale_split,
    method_config,
    parse_options,
    solve,
)
from .elements import ElementFamily, Formulation, dof_count, eval_basis, quadrature_rule
from .linalg import (
    KrylovStats,
    amg_setup,
    strength_aggregates,
    amg_vcycle,
    apply_ilu0,
    diag_lump,
    gmres,
    ilu0,
    schur_selfp,
    spmv,
)
from .mesh import CellKind, Mesh, cell_geometry, facet_adjacency, generate_unit_mesh
from .problem import (
    BoundarySpec,
    DppParameters,
    boundary_data,
    constant_mms,
    eta,
    exact_solution_2d,
    exact_solution_3d,
    manufactured_solution,
    mms_2d,
    mms_3d,
    paper_2d_parameters,
    paper_3d_parameters,
)
from .spectrum import (
    CSV_COLUMNS,
    EfficiencySeries,
    SpectrumRecord,
    StaticScalingError,
    convergence_slope,
    doa,
    doe,
    dos,
    field_errors,
    l2_error,
    parallel_efficiency,
    read_csv,
    run_case,
    static_scaling_run,
    write_csv,
)

__version__ = "0.1.0"
