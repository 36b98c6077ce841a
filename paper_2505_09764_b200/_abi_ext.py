"""ctypes signatures of the executor and MoE front-end entry points."""

from __future__ import annotations

import ctypes

from ._lib import FastPlan, FastSchedBufs

V = ctypes.c_void_p
I = ctypes.c_int
I64 = ctypes.c_int64
P_SCHED = ctypes.POINTER(FastSchedBufs)
P_PLAN = ctypes.POINTER(FastPlan)


class FastSimTopo(ctypes.Structure):
    """fast_sim_topo (include/fastb200.h)."""

    _fields_ = [("scaleup_bw", ctypes.c_double), ("scaleout_bw", ctypes.c_double),
                ("wakeup_delay", ctypes.c_double)]


class FastSimIn(ctypes.Structure):
    """fast_sim_in: packed schedules to evaluate."""

    _fields_ = [(name, ctypes.c_void_p) for name in (
        "balanced", "server", "common_sum", "move_count", "moves", "n_stages", "stage_order",
        "stage_weight", "stage_perm", "stage_bytes", "status", "demand")] + [
        ("move_slots", ctypes.c_int), ("stage_stride", ctypes.c_int)]


class FastSimOut(ctypes.Structure):
    """fast_sim_out: per-schedule model outputs."""

    _fields_ = [(name, ctypes.c_void_p) for name in (
        "t_balance", "t_intra", "scale_out", "redistribution", "total", "t_optimal",
        "t_worstcase", "assumption_ok", "so_weight", "so_server", "so_demand", "so_total",
        "status", "workspace")]

SIGNATURES: list[tuple[str, object, list]] = [
    # executor: plan compile (exec.cu / plan.cuh)
    ("fast_plan_workspace_bytes", ctypes.c_size_t, [I, I]),
    ("fast_plan_op_capacity", I64, [I, I]),
    ("fast_plan_compile", I, [V, V, I, I, P_SCHED, I64, I64, I64, P_PLAN, V]),
    ("fast_plan_compile_ex", I, [V, V, I, I, P_SCHED, I64, I64, I64, P_PLAN, I, V]),
    ("fast_plan_compile_host", I, [V, V, I, I, I, V, V, V, I64, I64, I64, V, I64, V, V, V]),
    # communicator + P2P execution
    ("fast_comm_create", I, [I, I, I, I64, I64, ctypes.POINTER(V)]),
    ("fast_comm_ipc_handle", I, [V, V]),
    ("fast_comm_open_peers", I, [V, ctypes.c_char_p]),
    ("fast_comm_destroy", I, [V]),
    ("fast_comm_recv_ptr", V, [V]),
    ("fast_comm_staging_ptr", V, [V]),
    ("fast_comm_demand_ptr", V, [V, I64]),
    ("fast_comm_recv_capacity", I64, [V]),
    ("fast_comm_staging_capacity", I64, [V]),
    ("fast_gather_demand", I, [V, V, I64, V]),
    ("fast_exec", I, [V, P_PLAN, V, I64, I, I64, V, V]),
    ("fast_comm_status", I, [V, ctypes.POINTER(ctypes.c_int32)]),
    ("fast_comm_peer_ptr", V, [V, I]),
    ("fast_alltoallv", I, [V, V, V, I, I, P_SCHED, P_PLAN, I, I64, V, V]),
    ("fast_comm_epoch", I64, [V]),
    ("fast_comm_set_epoch", I, [V, I64]),
    ("fast_comm_set_fused", I, [V, I]),
    ("fast_comm_set_send_rows", I, [V, V, V, I64, I64]),
    ("fast_comm_set_send_capacity", I, [V, I64]),
    ("fast_comm_set_pdl", I, [V, I]),
    ("fast_comm_set_copy_self", I, [V, I]),
    ("fast_debug_copy", I, [V, V, I64, I, I64, I, V]),
    ("fast_debug_memcpy", I, [V, V, I64, V]),
    ("fast_comm_create_group", I, [I, I64, I64, ctypes.POINTER(V)]),
    ("fast_exec_group", I, [ctypes.POINTER(V), I, P_PLAN, ctypes.POINTER(V), I64, I, I64, V, V]),
    # stage-level building blocks (stages.cu)
    ("fast_match_batch", I, [V, I, I, V, V, V]),
    ("fast_strip_sort_workspace_bytes", ctypes.c_size_t, [I, I]),
    ("fast_strip_sort", I, [V, V, V, V, I, I, I, V, V, V, V, V, V]),
    # analytical cost model (sim.cu)
    ("fast_sim_workspace_bytes", ctypes.c_size_t, [I, I, I, I]),
    ("fast_simulate_batch", I, [ctypes.POINTER(FastSimIn), I, I, I, ctypes.POINTER(FastSimTopo),
                                ctypes.POINTER(FastSimOut), V]),
    # MoE front-end (moe.cu)
    ("fast_moe_gate", I, [I, ctypes.c_uint64, I, V, V, V, V]),
    ("fast_moe_route_workspace_bytes", ctypes.c_size_t, [I, I, I]),
    ("fast_moe_route", I, [V, I, I, I, I64, V, V, V, V, V, V]),
    ("fast_moe_pack", I, [V, I, I, I64, V, V, V, I, V, V, V]),
    ("fast_moe_unpack_self", I, [V, V, I, I, V, V, V]),
    ("fast_moe_rowmap", I, [I, I, V, V, V, I, V, V, V]),
    ("fast_moe_unpack_self_rows", I, [V, V, I, I, V, V, I64, V, V]),
    ("fast_moe_combine", I, [V, V, V, I, I, I, I, I64, V, V, V, I, V, V, V, V]),
    ("fast_moe_route_ex", I, [V, I, I, I, I, I64, V, V, V, V, V, V]),
    ("fast_moe_combine_ex", I, [V, V, V, I, I, I, I, I64, V, V, V, I, I, V, V, V, V]),
]
