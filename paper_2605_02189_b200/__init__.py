"""B200-native PipeMax decode hot path.

Import surface mirrors the reference package ``pipemax`` (REF
pkg/src/pipemax/__init__.py:9-73) for the decode path: the control plane
(``model_core``, ``scheduler``) and the engine types (``trace``) import
without a GPU; ``run_decode`` / ``simulate_decode`` (the B200 engine) load
torch and the sm_100a library on first use.
"""

from .model_core import (
    CalibrationWarning,
    ClusterConfig,
    DegenerateSamples,
    EstimatorParams,
    NoKvHeadroom,
    PrefillInstance,
    Request,
    blocks_for_tokens,
    calibrate_estimator,
    capacity_blocks,
    estimate_decode_time,
    kv_footprint,
    per_batch_token_budget,
    prefill_makespan_closed_form,
    system_token_capacity,
)
from .scheduler import (
    EmptySystem,
    SchedulerState,
    StepPlan,
    batch_indices,
    commit_plan,
    detect_steady,
    initial_partition,
    prefetch_budget,
    residual_set,
    schedule_step,
    select_prefetch_steady,
    select_prefetch_warmup,
)
from .trace import (
    CapacityError,
    ConfigError,
    EpisodeMetrics,
    EventTrace,
    GpuState,
    NoiseSpec,
    OutOfMemory,
)


def run_decode(*args, **kwargs):
    """B200 decode engine with ``simulate_decode``'s shape (see engine.py)."""
    from .engine import run_decode as _run
    return _run(*args, **kwargs)


simulate_decode = run_decode

__version__ = "0.1.0"
