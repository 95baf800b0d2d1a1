"""B200-native AERO-MPPI plan-cycle hot path (arXiv 2509.17340).

build_snapshot + plan_step as hand-written sm_100a CUDA kernels behind a
C ABI (include/amppi_b200.h); this package is the thin host-side mirror of
the reference planner's interface.  See DESIGN.md.
"""
from .planner import (  # noqa: F401
    Anchor,
    AnchorGrid,
    ClosedLoop,
    AmppiError,
    CollisionParams,
    ControlInput,
    CostBreakdown,
    CostWeights,
    DynamicsParams,
    EnsembleConfig,
    GoalSpec,
    InstanceRecord,
    MppiConfig,
    PerceptionSnapshot,
    PlanResult,
    Planner,
    PlanningFailed,
    PointCloudBuffer,
    State,
    apply_velocity_cap,
)
from ._abi import LIB_PATH, load  # noqa: F401
