"""B200-native Swarm-Gen safety filter (arXiv 2501.19042).

Drop-in for the reference's ``swarmfilter`` safety-filter path: same problem
types, ``SafetyFilter`` call signature and result types, running the whole
alternating-minimisation loop in one persistent sm_100a kernel per batch
(``csrc/``, C ABI in ``include/sgsf.h``).  Importing this package does not
touch the GPU; the native library loads on first use and there is no CPU
fallback.
"""
from .basis import BasisMatrices, Trajectory, bernstein_matrices, build_basis, coeffs_to_axis_major
from .errors import (
    DegreeTooLow,
    DimensionMismatch,
    EndpointCollision,
    GoalOutsideWorkspace,
    NonPositiveGeometry,
    ProblemValidationError,
    RankDeficient,
    SchemaMismatch,
    SingularKKT,
    StartOutsideWorkspace,
    SwarmFilterError,
    TooFewSamples,
)
from .precompute import EqualitySystem, build_equality, device_constants
from .problem import (
    EndpointState,
    RobotBoundary,
    RobotShape,
    SwarmProblem,
    Workspace,
    load_problem,
    pair_margin,
    validate_problem,
    workspace_margin,
)
from .proposals import (
    ProposalBatch,
    WarmStart,
    load_proposals,
    load_warmstart,
    project_to_boundary,
    sample_proposals,
    save_proposals,
    save_warmstarts,
    straight_line_coeffs,
)
from .solver import (
    BatchResult,
    DeviceBatch,
    Operator,
    SafetyFilter,
    SolveResult,
    SolverConfig,
    SphericalVars,
    batch_solve,
    coefficient_step,
    multiplier_update,
    solve,
    spherical_step,
    write_residuals_csv,
)
from .metrics import (
    DIVERSITY_DEFINITION,
    BatchReport,
    BenchmarkGrid,
    benchmark,
    build_batch_report,
    build_spherical_rhs,
    diversity_cosine,
    mean_pairwise_cosine,
    primal_residual,
    save_report_json,
    spherical_targets,
    write_csv,
)
from .generative import (
    CVAEDecoder,
    PipelineGraph,
    VQVAEDecoder,
    calibrate_batchnorm,
    decode_proposals,
    generate_and_filter,
    make_decoder,
)
from .unrolled import UnrolledIterates, boundary_projection, fixed_point_loss, unrolled_solve
from .verdict import (
    ViolationReport,
    check_coefficients,
    check_original_constraints,
    coeffs_to_trajectory,
    feasible_fraction,
    feasible_results,
    verdict_batched,
)

__version__ = "0.1.0"
