"""ctypes binding of libshorsim_b200.so (the C ABI of include/shorsim_b200.h).

The product path always goes through this library: if it is missing the import
fails loudly — there is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SHS_LIB overrides the library path (build variants for A/B measurements)
LIB_PATH = os.environ.get("SHS_LIB") or os.path.join(HERE, "libshorsim_b200.so")

u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int32
dbl = C.c_double
vp = C.c_void_p

SHS_OK = 0
SHS_ERROR = 1
SHS_CONFIG_ERROR = 2
SHS_CEILING_EXCEEDED = 3
SHS_DEGENERATE_BRANCH = 4
SHS_BUDGET_EXCEEDED = 5
SHS_NOT_INVERTIBLE = 6
SHS_INVALID_ARGUMENT = 7
SHS_CUDA_ERROR = 8
SHS_FACTORIZATION_TIMEOUT = 9

COMBINE = {"auto": 0, "kahan": 1, "exact": 2}
SHS_DIGITS = 80
SHS_SHARD_IPC_BYTES = 1088
MAX_SHARDS = 16
TILING = {"auto": 0, "force": 1, "off": 2}


class shs_problem(C.Structure):
    _fields_ = [("N", u64), ("a", u64), ("L", u32), ("t", u32), ("seed", u64)]


class shs_error(C.Structure):
    _fields_ = [("kind", i32), ("delta", dbl), ("px", dbl), ("py", dbl), ("pz", dbl),
                ("has_pauli", i32)]


class shs_options(C.Structure):
    _fields_ = [("shard_count", u32), ("workers", u32), ("qubit_ceiling", u32),
                ("check_norms", i32), ("device", i32), ("combine", i32), ("tiling", i32),
                ("n_devices", i32), ("devices", C.POINTER(i32))]


class shs_stage_trace(C.Structure):
    _fields_ = [("cbit", u32), ("p1", dbl), ("sampled_bit", i32), ("observed_bit", i32),
                ("classical_flip", C.c_uint8), ("quantum_error_branch", C.c_uint8)]


# (name, restype, argtypes) for every symbol include/shorsim_b200.h declares
SIGNATURES = [
    ("shs_default_options", None, [C.POINTER(shs_options)]),
    ("shs_engine_create", C.c_int, [C.POINTER(shs_problem), C.POINTER(shs_error),
                                    C.POINTER(shs_options), C.POINTER(vp)]),
    ("shs_engine_destroy", None, [vp]),
    ("shs_engine_run", C.c_int, [vp, u64, u64, C.POINTER(u64), C.POINTER(u64),
                                 C.POINTER(shs_stage_trace)]),
    ("shs_engine_run_batch", C.c_int, [vp, u64, u64, u32, C.POINTER(u64)]),
    ("shs_engine_run_many", C.c_int, [vp, u64, u64, u32, C.POINTER(u64), C.POINTER(u64),
                                      C.POINTER(dbl), C.POINTER(i32)]),
    ("shs_engine_run_sequential", C.c_int, [vp, u64, u64, u32, C.POINTER(u64)]),
    ("shs_engine_batched", C.c_int, [vp]),
    ("shs_engine_stage_multipliers", C.c_int, [vp, C.POINTER(u64)]),
    ("shs_engine_stages", u32, [vp]),
    ("shs_state_init", C.c_int, [vp]),
    ("shs_stage_probs", C.c_int, [vp, u32, u64, u64, C.POINTER(dbl), C.POINTER(dbl)]),
    ("shs_stage_collapse", C.c_int, [vp, i32, dbl]),
    ("shs_stage_read", C.c_int, [vp, i32, u64, u64, C.POINTER(dbl)]),
    ("shs_state_read", C.c_int, [vp, i32, u64, u64, C.POINTER(dbl)]),
    ("shs_state_gather", C.c_int, [vp, i32, C.POINTER(u64), u64, C.POINTER(dbl)]),
    ("shs_stage_block_sums", C.c_int, [vp, C.POINTER(dbl)]),
    ("shs_num_blocks", u64, [vp]),
    ("shs_index_map", C.c_int, [vp, u32, u64, u64, C.POINTER(u64)]),
    ("shs_sample_measurement", C.c_int, [dbl, u64, u32, u32, C.POINTER(shs_error),
                                         C.POINTER(i32)]),
    ("shs_bitflip", C.c_int, [C.POINTER(u64), u32, dbl, u64, u32]),
    ("shs_engine_set_timing", C.c_int, [vp, i32]),
    ("shs_engine_kernel_times", C.c_int, [vp, C.POINTER(dbl), C.POINTER(u64)]),
    ("shs_stage_tile_plan", C.c_int, [vp, u32, C.POINTER(u64)]),
    ("shs_engine_stream", vp, [vp]),
    ("shs_engine_launch_count", u64, [vp]),
    ("shs_engine_device_bytes", u64, [vp]),
    ("shs_engine_devices", C.c_int, [vp, C.POINTER(i32), i32]),
    ("shs_shard_create", C.c_int, [C.POINTER(shs_problem), C.POINTER(shs_error),
                                   C.POINTER(shs_options), u32, u32, C.POINTER(vp)]),
    ("shs_shard_destroy", None, [vp]),
    ("shs_shard_range", C.c_int, [vp, C.POINTER(u64)]),
    ("shs_shard_buffers", C.c_int, [vp, C.POINTER(vp)]),
    ("shs_shard_ipc_handles", C.c_int, [vp, C.c_void_p]),
    ("shs_shard_attach", C.c_int, [vp, u32, C.POINTER(vp)]),
    ("shs_shard_attach_ipc", C.c_int, [vp, u32, C.c_void_p]),
    ("shs_shard_attach_local", C.c_int, [vp, vp]),
    ("shs_shard_set_barrier", C.c_int, [vp, C.c_char_p]),
    ("shs_shards_run", C.c_int, [C.POINTER(vp), u32, u64, u64, C.POINTER(u64), C.POINTER(u64),
                                 C.POINTER(shs_stage_trace)]),
    ("shs_shard_device_bytes", u64, [vp]),
    ("shs_shard_kahan", C.c_int, [vp]),
    ("shs_shard_set_sparse", C.c_int, [vp, i32]),
    ("shs_shard_sparse_stages", u32, [vp]),
    ("shs_node_barrier_open", C.c_int, [C.c_char_p, u32, i32, C.POINTER(vp)]),
    ("shs_node_barrier_arrive", C.c_int, [vp]),
    ("shs_node_barrier_close", None, [vp]),
    ("shs_shard_kahan_probs", C.c_int, [vp, C.POINTER(dbl), C.POINTER(dbl)]),
    ("shs_shard_init", C.c_int, [vp]),
    ("shs_shard_needs_exchange", C.c_int, [vp, u32]),
    ("shs_shard_exchange", C.c_int, [vp, u32]),
    ("shs_shard_probs", C.c_int, [vp, u32, u64, u64, C.POINTER(u64)]),
    ("shs_shard_collapse", C.c_int, [vp, i32, dbl]),
    ("shs_shard_sync", C.c_int, [vp]),
    ("shs_shard_state_read", C.c_int, [vp, i32, u64, u64, C.POINTER(dbl)]),
    ("shs_shard_stage_read", C.c_int, [vp, i32, u64, u64, C.POINTER(dbl)]),
    ("shs_digits_to_probs", C.c_int, [C.POINTER(u64), C.POINTER(dbl), C.POINTER(dbl)]),
    ("shs_shard_set_timing", C.c_int, [vp, i32]),
    ("shs_shard_kernel_times", C.c_int, [vp, C.POINTER(dbl), C.POINTER(u64)]),
    ("shs_shard_launch_count", u64, [vp]),
    ("shs_shard_set_timeline", C.c_int, [vp, i32]),
    ("shs_shard_timeline", C.c_int64, [vp, C.POINTER(dbl), u64]),
    ("shs_shard_stream", vp, [vp]),
    ("shs_sv_create", C.c_int, [u32, u32, i32, C.POINTER(vp)]),
    ("shs_sv_clone", C.c_int, [vp, C.POINTER(vp)]),
    ("shs_sv_destroy", None, [vp]),
    ("shs_sv_layout", C.c_int, [vp, C.POINTER(u32)]),
    ("shs_sv_read", C.c_int, [vp, u64, u64, C.POINTER(dbl)]),
    ("shs_sv_write", C.c_int, [vp, u64, u64, C.POINTER(dbl)]),
    ("shs_sv_init_state", C.c_int, [vp, C.POINTER(dbl)]),
    ("shs_sv_apply_oracle", C.c_int, [vp, u64, u64]),
    ("shs_sv_apply_phase", C.c_int, [vp, u32, u64, u64]),
    ("shs_sv_apply_hadamard_top", C.c_int, [vp]),
    ("shs_sv_group_norms", C.c_int, [vp, C.POINTER(dbl)]),
    ("shs_sv_reset_top", C.c_int, [vp, i32, i32, C.POINTER(dbl), dbl]),
    ("shs_sv_launch_count", u64, [vp]),
    ("shs_plan_build", C.c_int, [u64, u64, u32, u32, i32, C.POINTER(u64), C.POINTER(i32),
                                 C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    ("shs_plan_lists", C.c_int, [u64, u64, u32, u32, u32, i32, i32, C.POINTER(u64),
                                 C.POINTER(u64)]),
    ("shs_exhaustive_distribution", C.c_int, [C.POINTER(shs_problem), C.POINTER(shs_error), u64,
                                              i32, C.POINTER(dbl)]),
    ("shs_engine_set_sparse", C.c_int, [C.c_void_p, i32]),
    ("shs_engine_sparse_stages", u32, [C.c_void_p]),
    ("shs_engine_set_orbit", C.c_int, [C.c_void_p, i32]),
    ("shs_engine_orbit_info", C.c_int, [C.c_void_p, C.POINTER(u64)]),
    ("shs_engine_orbit_stages", C.c_int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    ("shs_shor_postprocess", C.c_int, [C.POINTER(u64), u32, u32, u64, u64, u64, i32, i32,
                                       C.c_void_p]),
    ("shs_ekera_postprocess", C.c_int, [C.POINTER(u64), u32, u32, u64, u64, C.c_void_p, u64,
                                        u64, u64, i32, i32, C.c_void_p]),
    ("shs_factorize", C.c_int, [u64, u64, i32, C.POINTER(u64), C.POINTER(u32), C.POINTER(u32)]),
    ("shs_last_error", C.c_char_p, []),
    ("shs_build_info", C.c_char_p, []),
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the engine library (once). Raises ImportError when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_2308_05047_b200/csrc`). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
