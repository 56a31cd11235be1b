"""B200-native engine for the data-parallel core of arXiv 2504.15303.

Drop-in for the reference package's hot path (hetserve):

* deployment search -- ``search_optimal_config``, ``estimate_system_throughput``
  (GPU kernels K1 table build + K2 exhaustive argmax / ranking);
* scheduler replay -- ``run_continuous``, ``run_scenario``,
  ``run_policy_comparison`` (GPU kernel K3, one warp per trace).

Types and exceptions carry the reference's names and fields.  The compute
path is the CUDA library ``libhetserve_b200.so`` (include/hetserve_b200.h);
there is no CPU fallback.
"""

from .domain import (
    RunningTokens,
    kv_usage,
    ClusterSpec,
    DeploymentConfig,
    EngineOverheads,
    FeasibilityVerdict,
    FitError,
    HetserveError,
    InfeasibleConfigError,
    InfeasibleError,
    InfeasibleRequestError,
    KvBudget,
    LatencyParams,
    MachinePlacement,
    MachineSpec,
    ModelSpec,
    RankDeficientError,
    Request,
    SchedulingError,
    SpecError,
    TraceError,
    WorkloadLimits,
    check_memory_constraint,
    decode_iteration_time,
    decode_time,
    deployment_for,
    enumerate_tp_degrees,
    kv_budget,
    kv_bytes_per_token,
    prefill_time,
)
from .planner import (
    BatchPlan,
    MachineEstimate,
    SearchOutcome,
    SearchTables,
    ThroughputEstimate,
    best_config,
    build_tables,
    deployment_of,
    estimate_batch_time,
    estimate_instance_throughput,
    merge_topk,
    estimate_system_throughput,
    plan_static_batches,
    time_batches,
    search_best,
    search_optimal_config,
    search_topk,
)
from .scheduling import (
    POLICIES,
    InstanceHandle,
    OutputLengthPredictor,
    PolicyConfig,
    PredictorConfig,
    Scheduler,
    ideal_batch_size,
    per_request_cost,
    request_oversized,
    workload,
)
from .simulator import (
    InstanceMetrics,
    ReplayBatchResult,
    Scenario,
    SimMetrics,
    build_instances,
    generate_arrivals,
    replay_candidates,
    replay_deployments,
    replay_traces,
    run_continuous,
    run_policy_comparison,
    run_scenario,
    run_static,
)
from ._native import EngineError, EngineUnavailable

__version__ = "0.1.0"
