"""ctypes binding of the product library ``lib/liboffsim.so.0``.

The library is the drop-in boundary: the reference's C ABI
(``include/offsim/offsim_c.h``) plus the B200 executor ABI
(``include/fuyou/fy_adam.h``). This module only declares signatures; it
never falls back to anything when the library is missing — importing the
package on a machine without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = LIB_DIR / "liboffsim.so.0"

# fy_status / offsim_status share the numbering of proj/include/offsim/offsim_c.h:16-22
FY_OK, FY_ERR_CONFIG, FY_ERR_INFEASIBLE, FY_ERR_INVARIANT, FY_ERR_INTERNAL, FY_ERR_DEVICE = (
    0, 2, 3, 4, 5, 6)
FY_BF16, FY_FP16, FY_FP32 = 0, 1, 2


class FyError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"status {status}: {message}")
        self.status = status


class AdamHparams(C.Structure):
    _fields_ = [
        ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
        ("weight_decay", C.c_float), ("step", C.c_uint64), ("adamw_mode", C.c_int),
        ("bias_correction", C.c_int), ("grad_scale", C.c_float), ("beta_t_given", C.c_int),
        ("beta1_t", C.c_float), ("beta2_t", C.c_float),
    ]


class AdamCounter(C.Structure):
    _fields_ = [("step", C.c_uint64), ("beta1", C.c_float), ("beta2", C.c_float),
                ("beta1_t", C.c_float), ("beta2_t", C.c_float), ("constructed", C.c_int)]


class AdamwArgs(C.Structure):
    _fields_ = [
        ("master", C.c_void_p), ("exp_avg", C.c_void_p), ("exp_avg_sq", C.c_void_p),
        ("grad", C.c_void_p), ("grad_dtype", C.c_int), ("param_out", C.c_void_p),
        ("param_dtype", C.c_int), ("n", C.c_uint64), ("hp", AdamHparams),
        ("grad_sq_sum", C.c_void_p), ("accumulate_sq", C.c_int), ("workspace", C.c_void_p),
        ("nonfinite_flag", C.c_void_p), ("grad_scale_dev", C.c_void_p), ("skip_if_set", C.c_void_p),
    ]


class PipelineConfig(C.Structure):
    _fields_ = [
        ("device", C.c_int), ("max_chunk_elems", C.c_uint64), ("slots", C.c_uint32),
        ("grad_dtype", C.c_int), ("param_dtype", C.c_int), ("grads_on_host", C.c_int),
        ("params_to_host", C.c_int), ("keep_params_on_device", C.c_int),
        ("states_on_device", C.c_int), ("no_step_counter", C.c_int),
    ]


class Chunk(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("h_states", C.c_void_p), ("grad", C.c_void_p),
        ("h_param", C.c_void_p), ("d_param", C.c_void_p), ("grad_ready", C.c_void_p),
        ("states_stride", C.c_uint64), ("update_done", C.c_void_p), ("flags", C.c_uint32),
    ]


class SwapConfig(C.Structure):
    _fields_ = [
        ("device", C.c_int), ("slot_bytes", C.c_uint64), ("slots", C.c_uint32),
        ("file_dir", C.c_char_p), ("direct_io", C.c_int),
    ]


FY_GATHER_NONE, FY_GATHER_NCCL, FY_GATHER_PEER = 0, 1, 2
FY_TIER_DEVICE, FY_TIER_HOST = 0, 1
FY_NCCL_ID_BYTES = 128
FY_IPC_HANDLE_BYTES = 64


class ShardConfig(C.Structure):
    _fields_ = [
        ("device", C.c_int), ("world", C.c_uint32), ("rank", C.c_uint32), ("gather", C.c_int),
        ("nccl_id", C.c_void_p), ("tier", C.c_int), ("chunk_count", C.c_uint32),
        ("chunk_elems", C.POINTER(C.c_uint64)), ("grad_dtype", C.c_int), ("param_dtype", C.c_int),
        ("slots", C.c_uint32), ("piece_elems", C.c_uint64), ("params_to_host", C.c_int),
        ("no_step_counter", C.c_int), ("grads_on_host", C.c_int),
    ]


class ShardSlice(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("count", C.c_uint64), ("stride", C.c_uint64),
                ("params", C.c_void_p)]


class ShardIo(C.Structure):
    _fields_ = [("states", C.c_void_p), ("grad", C.c_void_p), ("h_param", C.c_void_p),
                ("grad_ready", C.c_void_p)]


class ShardStats(C.Structure):
    _fields_ = [("step_ms", C.c_double), ("gather_bytes", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("world", C.c_uint32), ("rank", C.c_uint32),
                ("gather", C.c_int), ("stages", C.c_int), ("consumer_warps", C.c_int)]


FY_SWAP_CPU, FY_SWAP_SSD = 0, 1
FY_CHUNK_STATES_ON_DEVICE = 1


class ChunkTiming(C.Structure):
    _fields_ = [
        ("h2d_start_ns", C.c_uint64), ("h2d_end_ns", C.c_uint64),
        ("upd_start_ns", C.c_uint64), ("upd_end_ns", C.c_uint64),
        ("d2h_start_ns", C.c_uint64), ("d2h_end_ns", C.c_uint64),
    ]


def _load(path: Path = LIB_PATH) -> C.CDLL:
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (or `make`). There is no fallback implementation.")
    lib = C.CDLL(str(path), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    st = C.c_int
    sig = {
        "fy_version": (C.c_char_p, []),
        "fy_last_error": (C.c_char_p, []),
        "fy_adamw_workspace_floats": (C.c_uint32, []),
        "fy_adamw_chunk": (st, [C.POINTER(AdamwArgs), C.c_void_p]),
        "fy_adamw_chunk_gather": (st, [C.POINTER(AdamwArgs), C.POINTER(C.c_void_p), C.c_uint32,
                                       C.c_void_p]),
        "fy_grad_stats": (st, [C.c_void_p, C.c_int, C.c_uint64, C.c_float, C.c_void_p, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_void_p]),
        "fy_adamw_tune": (st, [C.c_int, C.c_int, C.c_int]),
        "fy_adam_counter_init": (st, [C.POINTER(AdamCounter), C.c_float, C.c_float]),
        "fy_adam_counter_next": (st, [C.POINTER(AdamCounter), C.POINTER(AdamHparams)]),
        "fy_nccl_unique_id": (st, [C.c_void_p]),
        "fy_shard_create": (st, [C.POINTER(ShardConfig), C.POINTER(C.c_void_p)]),
        "fy_shard_destroy": (None, [C.c_void_p]),
        "fy_shard_slice_info": (st, [C.c_void_p, C.c_uint32, C.POINTER(ShardSlice)]),
        "fy_shard_ipc_handle": (st, [C.c_void_p, C.c_void_p]),
        "fy_shard_arena": (st, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
        "fy_shard_connect": (st, [C.c_void_p, C.c_void_p]),
        "fy_shard_connect_ptrs": (st, [C.c_void_p, C.POINTER(C.c_void_p)]),
        "fy_shard_step": (st, [C.c_void_p, C.POINTER(ShardIo), C.POINTER(AdamHparams), C.c_int,
                               C.c_void_p]),
        "fy_shard_wait": (st, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
        "fy_shard_get_stats": (st, [C.c_void_p, C.POINTER(ShardStats)]),
        "fy_shard_update_ms": (st, [C.c_void_p, C.POINTER(C.c_double), C.c_uint32]),
        "fy_adamw_sm_budget": (st, [C.c_int]),
        "fy_adamw_chunks": (st, [C.POINTER(AdamwArgs), C.c_uint32, C.c_void_p]),
        "fy_clip_coef": (st, [C.c_void_p, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p]),
        "fy_pipeline_set_controls": (st, [C.c_void_p, C.c_void_p, C.c_void_p]),
        "fy_device_info": (st, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]),
        "fy_shard_range": (st, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "fy_pipeline_create": (st, [C.POINTER(PipelineConfig), C.POINTER(C.c_void_p)]),
        "fy_pipeline_destroy": (None, [C.c_void_p]),
        "fy_pipeline_step": (st, [C.c_void_p, C.POINTER(Chunk), C.c_uint32,
                                  C.POINTER(AdamHparams), C.c_int]),
        "fy_pipeline_wait": (st, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
        "fy_pipeline_timings": (st, [C.c_void_p, C.POINTER(ChunkTiming), C.c_uint32,
                                     C.POINTER(C.c_uint64)]),
        "fy_host_alloc": (st, [C.c_uint64, C.POINTER(C.c_void_p)]),
        "fy_host_free": (st, [C.c_void_p]),
        "fy_ipc_alloc": (st, [C.c_uint64, C.POINTER(C.c_void_p), C.c_void_p]),
        "fy_ipc_open": (st, [C.c_void_p, C.POINTER(C.c_void_p)]),
        "fy_ipc_close": (st, [C.c_void_p]),
        "fy_ipc_free": (st, [C.c_void_p]),
        "fy_swapper_create": (st, [C.POINTER(SwapConfig), C.POINTER(C.c_void_p)]),
        "fy_swapper_destroy": (None, [C.c_void_p]),
        "fy_swap_out": (st, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                             C.POINTER(C.c_uint64)]),
        "fy_swap_in": (st, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
        "fy_swap_release": (st, [C.c_void_p, C.c_uint64]),
        "fy_swapper_sync": (st, [C.c_void_p]),
        "fy_swapper_stats": (st, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_char_p)]),
        "fy_host_alloc_on": (st, [C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]),
        "fy_device_numa_node": (st, [C.c_int, C.POINTER(C.c_int)]),
        "fy_host_numa_node": (st, [C.c_void_p, C.POINTER(C.c_int)]),
    }
    if path != LIB_PATH:  # the sweep build (build/sweep) adds the variant selector
        sig["fy_adamw_tune_bulk"] = (st, [C.c_int, C.c_int, C.c_int])
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()

SWEEP_LIB_PATH = LIB_DIR.parent.parent / "build" / "sweep" / "liboffsim_sweep.so"


def load_sweep_lib() -> C.CDLL:
    """The sweep-only build (make sweep): same ABI plus fy_adamw_tune_bulk's
    experimental TMA variants. Bench / test tooling only; never the product."""
    return _load(SWEEP_LIB_PATH)


def check(status: int) -> None:
    if status != FY_OK:
        raise FyError(status, LIB.fy_last_error().decode())
