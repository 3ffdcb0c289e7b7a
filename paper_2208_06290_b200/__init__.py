"""B200-native HODLR factorize/solve engine (arXiv 2208.06290 hot path).

Public API mirrors the reference package ``hodlr`` (tree + batched kernel
layer) and its SPEC factorization/solver contracts; all arithmetic runs in
hand-written sm_100a CUDA kernels behind the C ABI in ``include/hodlr_b200.h``.
"""

from .tree import ClusterTree, IndexRange, build_tree, sibling_pairs  # noqa: F401
from .backend import (  # noqa: F401
    SERIAL,
    BlockBatch,
    BlockRef,
    LuPivots,
    SingularBlockError,
    ThreadedExecutor,
    as_stack,
    batched_gemm,
    batched_lu_factor_inplace,
    batched_lu_solve_inplace,
    gemm_stacks,
    grouped_gemm_large,
    lu_solve_stacks,
    parse_executor,
)
from .hodlr import (  # noqa: F401
    FactorPlan,
    HodlrFactorization,
    HodlrMatrix,
    HodlrSingularError,
    LevelPanel,
    RefinementResult,
    factorize,
    factorize_from_host,
    flop_report,
    logdet,
    pad_level_panels,
    truncate_ranks,
    random_hodlr,
    solve,
    solve_flops,
    solve_with_refinement,
)
from .construct import (  # noqa: F401
    CompressionConfig,
    GaussianPoints,
    LaplaceDoubleLayer,
    assemble,
    assemble_dense,
    contour_default,
    gaussian_hodlr,
    kd_points,
    laplace_dl_geometry,
    laplace_dl_hodlr,
    schur_surrogate_hodlr,
    separator_grid,
)
from ._lib import HodlrNativeError, LIB_PATH  # noqa: F401
from .io import dump, load  # noqa: F401
from .krylov import GmresResult, gmres, gmres_hodlr  # noqa: F401

__version__ = "0.1.0"
