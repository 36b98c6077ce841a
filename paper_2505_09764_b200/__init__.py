"""B200-native FAST All-to-All(v) hot path (arXiv 2505.09764).

A drop-in for the scheduler/executor path of the reference package
``tiersched``: the names below mirror ``tiersched.__all__``
(/root/reference/pkg/src/tiersched/__init__.py:76-129) for everything on the
hot path.  Synthesis runs as batched sm_100a kernels (csrc/synth.cu), the
executor as P2P copy kernels over NVSwitch (csrc/exec.cu), the MoE front-end
as histogram/scan and 16-byte pack/unpack kernels (csrc/moe.cu).  All of it is
reached through the C-ABI in include/fastb200.h; there is no CPU fallback.
"""

from .model import (
    MAX_SAFE_TOTAL,
    load_matrix,
    save_matrix,
    DemandMatrix,
    InternalInvariantError,
    ServerMatrix,
    TileView,
    Topology,
    ValidationError,
    max_rc,
    reduce_to_server_level,
    tile,
    validate_topology,
)
from .schedule import (
    BalancePlan,
    Decomposition,
    IntraMove,
    PackedSchedule,
    PermutationStage,
    Schedule,
    dumps_canonical,
    schedule_from_json,
    schedule_to_json,
)
from .workloads import gen_adversarial, gen_hotspot, gen_uniform, gen_zipf, load_trace


def algorithmic_bandwidth(total_bytes: int, gpu_count: int, completion_s: float) -> float:
    """Total bytes per GPU per second of completion (bounds.py:90-98)."""
    if gpu_count <= 0:
        raise ValidationError("gpu_count must be positive")
    if completion_s <= 0:
        raise ValidationError("completion time must be positive")
    return total_bytes / (gpu_count * completion_s)


_LAZY = {
    # GPU synthesis (needs torch + libfastb200.so)
    "synthesize_fast": "synth", "synthesize_fast_batch": "synth",
    "synthesize_packed": "synth", "SynthBuffers": "synth",
    "build_balance_plan": "synth", "decompose_server_matrix": "synth",
    "embed_doubly_stochastic": "synth", "decompose": "synth",
    "balance_senders": "synth", "merge_peer": "synth", "find_perfect_matching": "synth",
    "strip_auxiliary": "synth", "sort_stages_ascending": "synth",
    # executor
    "FastComm": "executor", "execute_fast": "executor", "all_to_all_fast": "executor",
    # analytical cost model + baseline + bounds (device kernel csrc/sim.cu)
    "Timeline": "simulate", "simulate_fast": "simulate", "simulate_batch": "simulate",
    "simulate_spreadout": "simulate", "SimBuffers": "simulate", "step_cost": "simulate",
    "intra_phase_time": "simulate", "split_deliveries": "simulate",
    "stage_redistribution": "simulate", "spreadout_stages": "simulate",
    "spreadout_completion_units": "simulate", "spreadout_intra": "simulate",
    "synthesize_spreadout": "simulate", "SpreadoutSchedule": "simulate",
    "BoundsReport": "simulate", "bounds_report": "simulate", "optimal_time": "simulate",
    "fast_worstcase_time": "simulate", "ratio_bound": "simulate",
    "intra_assumption_holds": "simulate",
    # MoE front-end
    "MoEDispatch": "moe",
}


def __getattr__(name: str):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = [
    "BalancePlan", "Decomposition", "DemandMatrix", "InternalInvariantError", "IntraMove",
    "MAX_SAFE_TOTAL", "PackedSchedule", "PermutationStage", "Schedule", "ServerMatrix",
    "TileView", "Topology", "ValidationError", "algorithmic_bandwidth", "dumps_canonical",
    "gen_adversarial", "gen_hotspot", "gen_uniform", "gen_zipf", "load_matrix", "load_trace",
    "max_rc", "save_matrix",
    "reduce_to_server_level", "schedule_from_json", "schedule_to_json", "tile",
    "validate_topology", *_LAZY,
]
__version__ = "0.1.0"
