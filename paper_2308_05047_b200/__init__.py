"""shorsim_b200: B200-native iterative-Shor simulator (arXiv 2308.05047 hot path).

The stage loop of the reference's ``IterativeShorEngine``
(/root/reference/proj/src/statevector.cpp:323-412) on hand-written sm_100a
kernels behind the C ABI of ``include/shorsim_b200.h``.
"""
from .engine import (  # noqa: F401
    BitString,
    BudgetExceededError,
    CeilingExceededError,
    ConfigError,
    CudaError,
    DegenerateBranchError,
    Error,
    ErrorConfig,
    ErrorEvent,
    ErrorKind,
    FactoringProblem,
    FactorizationTimeoutError,
    IterativeShorEngine,
    NotInvertibleError,
    PauliProbs,
    RunResult,
    SimulatorOptions,
    StageTrace,
    bit_length,
    build_info,
    exhaustive_joint_distribution,
    parse_error_config,
    recommended_t,
    run_iterative_shor,
    sample_measurement,
)
from .postprocess import (  # noqa: F401
    Classification,
    EkeraOutcome,
    EkeraParams,
    ekera_postprocess,
    ekera_postprocess_array,
    factorize,
    PostProcessOutcome,
    ProblemResult,
    multiplicative_order,
    run_problem,
    shor_postprocess_array,
    shor_standard_procedure,
)
from .sharded import DistGroup, LocalGroup, Shard, ShardedShorEngine, digits_to_probs  # noqa: F401
from .state import (  # noqa: F401
    ExchangePlan,
    ShardedState,
    ShardIndexList,
    ShardLayout,
    apply_hadamard_top,
    apply_oracle,
    apply_phase,
    build_permutation_plan,
    init_state,
    make_shard_layout,
    measure_top,
    plan_receive_lists,
    plan_send_lists,
    reset_top,
    stage_phase,
)
