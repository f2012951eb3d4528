"""paper_1008_1371_b200 -- B200-native one-sided Jacobi hyperbolic SVD.

Drop-in for the hot path of the reference package ``hjsvd``:
``drive(G, J, cfg) -> HsvdResult`` with the same names, fields, defaults and
exceptions (/root/reference/pkg/src/hjsvd/__init__.py:9-81, solver part).
All numerics run in hand-written sm_100a CUDA (lib/libhsvd_b200.so, C ABI
in include/hsvd_b200.h); there is no CPU fallback.
"""

from .errors import (
    DefinitenessLostError,
    HsvdCudaError,
    NumericalSingularityError,
    RankDeficiencyError,
    ShapeError,
)
from .linalg import (
    DEFAULT_CHUNK,
    EPS,
    SignatureVector,
    as_factor,
    dot_chunked,
    fused_pair_update,
    orthonormality_distance,
)
from .factory import (
    ALPHA,
    GAP,
    FactorPair,
    SpectrumSpec,
    TestBundle,
    bunch_parlett_factor,
    bunch_parlett_factor_device,
    draw_spectrum,
    eigvalsh,
    generate_factor_pair,
    generate_symmetric,
    qr_shorten,
)
from .matio import read_csv_matrix, read_gjh, write_csv_matrix, write_gjh
from .rotation import (
    CODE_BIG,
    CODE_NONE,
    CODE_SMALL,
    TEPS,
    PivotGram,
    Rotation,
    compute_rotation,
    convergence_code,
    diagonal_update_predicted,
    relatively_orthogonal,
    rotation_params_batch,
)
from .solver import (
    BorderInfo,
    DiagonalPackageVector,
    HsvdResult,
    SolverConfig,
    border,
    check_convergence,
    drive,
    drive_device,
    jacobi_step,
    precompute,
    recover_V,
    sort_diagonal,
    strip_bordered,
)
from .sharded import (
    ShardComm,
    ShardedResult,
    drive_local_shards,
    drive_sharded,
    drive_sharded_device,
    gather_result,
)
from .strategies import (
    StepperState,
    schedule_table,
    stepper_advance,
    stepper_advance_all,
    stepper_init,
)

__version__ = "0.1.0"
