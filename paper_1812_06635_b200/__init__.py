"""B200-native FastL1 hot path (arXiv 1812.06635): FISTA/ISTA + stable GAP Safe
screening + dictionary switching as one persistent sm_100a kernel behind a
C-ABI (include/fl1cuda.h). See DESIGN.md.
"""
from .fastl1 import (  # noqa: F401
    ApproxDictionary,
    ApproxSequence,
    Backend,
    DenseDictionary,
    InvalidArgument,
    RunOptions,
    SolveResult,
    SukroDictionary,
    SwitchConfig,
    fastl1_solve,
    lambda_max,
    lipschitz_bound,
    make_exact_approx,
    recompute_flops,
    run_lasso,
    RULE_DYNAMIC,
    RULE_GAP,
    SOLVER_FISTA,
    SOLVER_ISTA,
    VARIANT_MULTI_DICT,
    VARIANT_PLAIN,
    VARIANT_SCREENED,
)
