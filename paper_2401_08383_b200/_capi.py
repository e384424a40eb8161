"""ctypes binding of include/exflow_c.h (libexflow_b200.so, built in-tree).

There is deliberately no fallback: if the shared library is missing or was
built without sm_100a kernels every call raises, so a GPU run can never
silently go through a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libexflow_b200.so")

EXF_OK, EXF_RUNTIME, EXF_INVALID, EXF_CUDA, EXF_COMM = 0, 1, 2, 3, 4


class ExflowError(RuntimeError):
    """EXF_RUNTIME: mirrors std::runtime_error / ParseError (CLI exit 1)."""


class ExflowInvalidArgument(ValueError):
    """EXF_INVALID: mirrors std::invalid_argument (CLI exit 2)."""


class ExflowCudaError(RuntimeError):
    """EXF_CUDA: CUDA runtime, launch or kernel fault."""


class ExflowCommError(RuntimeError):
    """EXF_COMM: peer exchange failure or barrier timeout."""


_ERRORS = {EXF_RUNTIME: ExflowError, EXF_INVALID: ExflowInvalidArgument,
           EXF_CUDA: ExflowCudaError, EXF_COMM: ExflowCommError}


class SimCounters(C.Structure):
    _fields_ = [("gpu_local_events", C.c_int64), ("node_local_events", C.c_int64),
                ("away_from_home_events", C.c_int64), ("coherent_moves", C.c_int64),
                ("hops_intra_node", C.c_int64), ("hops_inter_node", C.c_int64)]


class SimReportC(C.Structure):
    _fields_ = [("hops_intra_node", C.c_int64), ("hops_inter_node", C.c_int64),
                ("locality_gpu", C.c_double), ("locality_node", C.c_double),
                ("p", C.c_double), ("p_star", C.c_double),
                ("alltoall_count", C.c_int64), ("allgather_count", C.c_int64),
                ("setup_allgather_count", C.c_int64), ("volume_units", C.c_double),
                ("estimated_latency", C.c_double)]


class AnnealParamsC(C.Structure):
    _fields_ = [("restarts", C.c_int32), ("max_iters", C.c_int64),
                ("initial_temperature", C.c_double), ("cooling", C.c_double),
                ("seed", C.c_uint64)]


class SolveReportC(C.Structure):
    _fields_ = [("solver", C.c_char * 32), ("objective", C.c_double), ("seed", C.c_uint64),
                ("iterations", C.c_int64), ("restarts", C.c_int32),
                ("has_optimality_gap", C.c_int32), ("optimality_gap", C.c_double),
                ("has_tiers", C.c_int32), ("inter_node_crossings", C.c_double),
                ("intra_node_crossings", C.c_double), ("weighted_cost", C.c_double)]


_VP = C.c_void_p
_I32, _I64, _D = C.c_int32, C.c_int64, C.c_double

# name -> (restype, argtypes); every symbol declared in include/exflow_c.h
SIGNATURES = {
    "exf_last_error": (C.c_char_p, []),
    "exf_version": (_I32, []),
    "exf_device_ok": (_I32, []),
    "exf_count_transitions_workspace_bytes": (_I64, [_I64, _I32, _I32, _I32]),
    "exf_count_transitions": (C.c_int, [_VP, _I64, _I32, _I32, _I32, _VP, _VP, _VP, _VP]),
    "exf_count_transitions_host": (C.c_int, [_VP, _I64, _I32, _I32, _I32, _VP, _VP]),
    "exf_route_replay": (C.c_int, [_VP, _VP, _VP, _I64, _I32, _I32, _I32, _I32, _I32, _VP,
                                   _VP]),
    "exf_sim_report_from_counters": (C.c_int, [_VP, _I64, _I32, _I32, _I32, _D, _D, _I32, _I32,
                                               _VP]),
    "exf_simulate_host": (C.c_int, [_VP, _I64, _I32, _I32, _VP, _I32, _I32, _D, _D, _I32, _I32,
                                    _VP, _VP]),
    "exf_token_hops": (C.c_int, [_VP, _I32, _I32, _VP, _I32, _I32, _I32, _I32, _VP, _VP, _VP]),
    "exf_contiguous_placement": (C.c_int, [_I32, _I32, _I32, _I32, _VP]),
    "exf_random_placement": (C.c_int, [_I32, _I32, _I32, _I32, C.c_uint64, _VP]),
    "exf_validate_placement": (C.c_int, [_VP, _I32, _I32, _I32, _I32]),
    "exf_objective_crossings": (C.c_int, [_VP, _I32, _I32, _I32, _VP, _I32, _I32, _I32, _VP]),
    "exf_balanced_assignment_count": (_I64, [_I32, _I32, _I64]),
    "exf_solve_exact_dp": (C.c_int, [_VP, _I32, _I32, _I32, _I64, _VP, _VP]),
    "exf_solve_local_search": (C.c_int, [_VP, _I32, _I32, _I32, _VP, _VP, _VP]),
    "exf_solve_staged": (C.c_int, [_VP, _I32, _I32, _I32, _I32, _D, _D, _VP, _I64, _VP, _VP]),
    "exf_generate_markov_trace": (C.c_int, [_I32, _I32, _I64, _D, _I32, C.c_uint64, _VP]),
    "exf_model_create": (C.c_int, [_VP, _VP, _VP]),
    "exf_model_destroy": (C.c_int, [_VP]),
    "exf_model_ipc_handle": (C.c_int, [_VP, _VP]),
    "exf_model_connect": (C.c_int, [_VP, _VP]),
    "exf_model_connect_local": (C.c_int, [_VP, _I32]),
    "exf_model_step": (C.c_int, [_VP, _VP, _VP]),
    "exf_model_step_phase": (C.c_int, [_VP, _I32, _I32, _VP, _VP]),
    "exf_model_output": (C.c_int, [_VP, _VP]),
    "exf_model_context_setup": (C.c_int, [_VP, _VP]),
    "exf_model_context_setup_phase": (C.c_int, [_VP, _I32, _VP]),
    "exf_model_read_kv": (C.c_int, [_VP, _I32, _I32, _I32, _I32, _VP, _VP]),
    "exf_model_read_kv_len": (C.c_int, [_VP, _I32, _VP]),
    "exf_model_read_attn": (C.c_int, [_VP, _I32, _VP, _VP, _VP, _VP]),
    "exf_model_set_forced_routes": (C.c_int, [_VP, _VP]),
    "exf_model_read_routes": (C.c_int, [_VP, _VP]),
    "exf_model_read_crossed": (C.c_int, [_VP, _VP]),
    "exf_affinity_snapshot": (C.c_int, [_VP, _VP]),
    "exf_model_reset_stats": (C.c_int, [_VP]),
    "exf_model_check": (C.c_int, [_VP]),
    "exf_model_read_expert": (C.c_int, [_VP, _I32, _I32, _VP, _VP, _VP, _VP]),
    "exf_model_read_gate": (C.c_int, [_VP, _I32, _VP]),
    "exf_model_read_resident": (C.c_int, [_VP, _I32, _VP, _VP, _VP]),
    "exf_model_capture": (C.c_int, [_VP, _VP, _VP]),
    "exf_model_replay": (C.c_int, [_VP, _VP]),
    "exf_model_launches_per_step": (_I32, [_VP]),
    "exf_model_describe": (C.c_int, [_VP, _VP, _I32]),
    "exf_model_read_ffn_timeline": (C.c_int, [_VP, _VP, _I32]),
    "exf_debug_last_timeout": (C.c_int32, [_VP]),
    "exf_model_expert_storage": (C.c_int, [_VP, _I32, _I32, _VP, _VP, _VP, _VP]),
    "exf_model_set_placement": (C.c_int, [_VP, _VP]),
    "exf_model_read_step_timeline": (C.c_int, [_VP, _VP, _I32]),
    "exf_coherent_attention_workspace_bytes": (_I64, [_I64, _I32, _I32, _I32]),
    "exf_coherent_attention": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _I64, _I32, _I32, _I32, _I32,
                                         C.c_float, _VP, _VP, _VP]),
    "exf_kv_append": (C.c_int, [_VP, _VP, _VP, _I64, _I32, _I32, _I32, _I32, _I32, _VP, _VP, _VP,
                                _VP, _VP]),
    "exf_ipc_export": (C.c_int, [_VP, _VP, _VP]),
    "exf_ipc_import": (C.c_int, [_VP, _I64, _VP]),
    "exf_ipc_close": (C.c_int, [_VP, _I64]),
}


class ModelConfigC(C.Structure):
    _fields_ = [("num_experts", C.c_int32), ("num_layers", C.c_int32), ("d_model", C.c_int32),
                ("d_ffn", C.c_int32), ("top_k", C.c_int32), ("tokens_per_gpu", C.c_int32),
                ("world_size", C.c_int32), ("rank", C.c_int32), ("seed", C.c_uint64),
                ("init_std", C.c_float), ("gate_affinity", C.c_float), ("ep_mode", C.c_int32),
                ("dtype", C.c_int32), ("attn_heads", C.c_int32), ("context_len", C.c_int32),
                ("context_prefix", C.c_int32)]

_lib = None


def load():
    """Load libexflow_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: run __graft_entry__.build() (make -C "
                "paper_2401_08383_b200/csrc); there is no CPU fallback")
        lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc != EXF_OK:
        msg = load().exf_last_error().decode()
        raise _ERRORS.get(rc, ExflowError)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
