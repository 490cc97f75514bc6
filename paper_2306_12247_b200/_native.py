"""ctypes binding of libcapsim_b200.so (include/capsim_b200.h).

There is no fallback: if the shared library is missing or was not built for this machine,
importing the product's accelerated entry points raises ``NativeLibraryError`` — the drop-in
never silently runs a CPU path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path


LIB_PATH = Path(os.environ.get("CAPSIM_B200_LIB") or Path(__file__).resolve().parent / "_lib" / "libcapsim_b200.so")

CS_OK = 0
CS_E_INVALID = -1
CS_E_CUDA = -2
CS_E_NODEVICE = -3
CS_E_UNSUPPORTED = -4

CS_CAP_F32 = 0
CS_CAP_F64 = 1

CS_FLAG_CHECK_VIOLATIONS = 1
CS_FLAG_ACCUMULATE_HIST = 2
CS_FLAG_SEGMENT_EPILOGUE = 4
CS_FLAG_PREPARED = 8

CS_CTRL_TIME_MAJOR = 256

CS_SWEEP_WORDS = 12

CS_QUERY_BINS = 0
CS_QUERY_SELECT = 1
CS_QUERY_FEASIBLE = 2

TRACE_KINDS = {"solar": 0, "wind": 1, "mixed": 2, "iid": 3}

# Every symbol declared in include/capsim_b200.h (checked by tests/test_native_abi.py).
EXPORTS = (
    "cs_last_error", "cs_abi_version", "cs_device_query",
    "cs_tables_create", "cs_tables_destroy", "cs_tables_get_info", "cs_tables_grid_bins",
    "cs_tables_union_map", "cs_tables_lookup_host", "cs_tables_lookup_host_lut", "cs_tables_upload",
    "cs_eval_workspace_size", "cs_eval", "cs_eval_last_kernel_ms", "cs_eval_last_launches", "cs_eval_last_plan",
    "cs_select_caps", "cs_feasible_caps", "cs_query_host",
    "cs_engine_create", "cs_engine_destroy", "cs_engine_eval_host",
    "cs_sweep_totals", "cs_replay", "cs_generate_traces", "cs_select_sampling", "cs_entries_aggregate",
    "cs_traces_parse_files", "cs_traces_parse_text", "cs_traces_info", "cs_traces_copy", "cs_traces_pack",
    "cs_traces_destroy", "cs_comm_init_all", "cs_comm_size", "cs_comm_allreduce_i64", "cs_comm_destroy",
)


class NativeLibraryError(RuntimeError):
    """libcapsim_b200.so is missing or unusable (build it: python -m paper_2306_12247_b200.build)."""


class CudaError(RuntimeError):
    pass


class GridDesc(C.Structure):
    _fields_ = [
        ("n_entries", C.c_int32),
        ("mtl", C.POINTER(C.c_int32)),
        ("bs", C.POINTER(C.c_int32)),
        ("throughput_ips", C.POINTER(C.c_double)),
        ("power_w", C.POINTER(C.c_double)),
        ("idle_power_w", C.c_double),
    ]


class Agg(C.Structure):
    _fields_ = [
        ("avg_throughput_ips", C.c_double),
        ("energy_proxy_wh", C.c_double),
        ("idle_steps", C.c_int64),
        ("switches", C.c_int64),
        ("violations", C.c_int64),
        ("num_steps", C.c_int64),
    ]


AGG_FIELDS = [f[0] for f in Agg._fields_]


class TablesInfo(C.Structure):
    _fields_ = [
        ("cap_dtype", C.c_int32),
        ("n_grids", C.c_int32),
        ("n_union_bins", C.c_int32),
        ("max_grid_bins", C.c_int32),
        ("lut_entries", C.c_int32),
        ("lut_shift", C.c_int32),
        ("lut_level1", C.c_int32),
        ("lut_subtables", C.c_int32),
        ("device_bytes", C.c_int64),
        ("lut_unsafe_leaves", C.c_int32),
        ("n_segments", C.c_int32),
        ("lut_big_entries", C.c_int32),
        ("lut_big_shift", C.c_int32),
        ("lut_big_unsafe_leaves", C.c_int32),
        ("lut_huge_entries", C.c_int32),
        ("lut_huge_shift", C.c_int32),
        ("lut_huge_unsafe_leaves", C.c_int32),
    ]


class EvalArgs(C.Structure):
    _fields_ = [
        ("caps", C.c_void_p),
        ("n_traces", C.c_int64),
        ("n_steps", C.c_int64),
        ("ld", C.c_int64),
        ("step_seconds", C.c_int32),
        ("switch_penalty_s", C.c_double),
        ("flags", C.c_uint32),
        ("step_bins", C.c_void_p),
        ("ld_bins", C.c_int64),
        ("agg", C.c_void_p),
        ("hist", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
    ]


class EvalPlan(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("ctas", "threads", "warps_per_group", "smem_bytes", "trace_segments",
                                         "lut_entries", "lut_shift", "epilogue", "redirect_uniform")]


class TraceInfo(C.Structure):
    _fields_ = [("n_values", C.c_int64), ("start_unix_us", C.c_int64), ("status", C.c_int32), ("line", C.c_int32)]


class ReplayStep(C.Structure):
    _fields_ = [("measured_power_w", C.c_double), ("bin_reactive", C.c_uint16), ("bin_final", C.c_uint16),
                ("kind_bits", C.c_uint8), ("pad", C.c_uint8 * 3)]


class ReplayAgg(C.Structure):
    _fields_ = [("violations", C.c_int64), ("reconfigs", C.c_int64), ("violation_fraction", C.c_double),
                ("avg_throughput_ips", C.c_double), ("num_steps", C.c_int64)]


_lib = None
_lock = threading.Lock()


def _declare(L: C.CDLL) -> None:
    vp, i32, i64, u32, dbl, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double, C.c_size_t
    P = C.POINTER
    sig = {
        "cs_last_error": ([], C.c_char_p),
        "cs_abi_version": ([], C.c_int),
        "cs_device_query": ([i32, P(i32), P(i32), P(i32)], C.c_int),
        "cs_tables_create": ([P(GridDesc), i32, i32, i32, i32, P(vp)], C.c_int),
        "cs_tables_destroy": ([vp], C.c_int),
        "cs_tables_get_info": ([vp, P(TablesInfo)], C.c_int),
        "cs_tables_grid_bins": ([vp, i32, i32, vp, vp, P(i32)], C.c_int),
        "cs_tables_union_map": ([vp, i32, vp], C.c_int),
        "cs_tables_lookup_host": ([vp, vp, i64, vp], C.c_int),
        "cs_tables_lookup_host_lut": ([vp, vp, i64, C.c_int32, vp], C.c_int),
        "cs_tables_upload": ([vp, i32], C.c_int),
        "cs_eval_workspace_size": ([vp, P(EvalArgs), P(sz)], C.c_int),
        "cs_eval": ([vp, P(EvalArgs), vp], C.c_int),
        "cs_eval_last_kernel_ms": ([P(C.c_float)], C.c_int),
        "cs_eval_last_launches": ([P(i32)], C.c_int),
        "cs_eval_last_plan": ([P(EvalPlan)], C.c_int),
        "cs_select_caps": ([vp, i32, i32, vp, i64, vp, vp, vp], C.c_int),
        "cs_feasible_caps": ([vp, i32, i32, vp, i64, vp, vp], C.c_int),
        "cs_engine_create": ([i32, i64, i64, i32, P(vp)], C.c_int),
        "cs_engine_destroy": ([vp], C.c_int),
        "cs_comm_init_all": ([i32, vp, P(vp)], C.c_int),
        "cs_comm_size": ([vp, P(i32)], C.c_int),
        "cs_comm_allreduce_i64": ([vp, vp, i64, vp], C.c_int),
        "cs_comm_destroy": ([vp], C.c_int),
        "cs_engine_eval_host": ([vp, vp, vp, i64, i64, i64, i32, dbl, u32, vp, vp, P(i64), P(i64)], C.c_int),
        "cs_generate_traces": ([vp, i64, i64, i64, i64, i32, i32, C.c_float, C.c_uint64, vp], C.c_int),
        "cs_replay": ([vp, i32, vp, i64, i64, i64, i32, i32, vp, dbl, vp, vp, i32, C.c_uint64, vp, vp, vp], C.c_int),
        "cs_select_sampling": ([vp, i32, vp, i64, i64, i64, i64, i64, C.c_uint64, i64, vp, vp, vp], C.c_int),
        "cs_query_host": ([vp, i32, i32, i32, vp, i64, vp, vp], C.c_int),
        "cs_sweep_totals": ([vp, i64, i32, vp, u32, vp], C.c_int),
        "cs_entries_aggregate": ([vp, i64, i64, i64, vp, i32, dbl, vp, vp, vp, vp], C.c_int),
        "cs_traces_parse_files": ([P(C.c_char_p), i32, i64, i32, i32, P(vp)], C.c_int),
        "cs_traces_parse_text": ([C.c_char_p, i64, i64, i32, P(vp)], C.c_int),
        "cs_traces_info": ([vp, i32, P(TraceInfo)], C.c_int),
        "cs_traces_copy": ([vp, i32, vp], C.c_int),
        "cs_traces_pack": ([vp, i32, i64, i64, vp, i32], C.c_int),
        "cs_traces_destroy": ([vp], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> C.CDLL:
    """Load (once) the in-tree shared library; raises NativeLibraryError if it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise NativeLibraryError(
                        f"{LIB_PATH} not found: build it with `python -m paper_2306_12247_b200.build` "
                        "(there is no CPU fallback)")
                try:
                    L = C.CDLL(str(LIB_PATH))
                except OSError as exc:  # pragma: no cover - depends on the host
                    raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
                _declare(L)
                if L.cs_abi_version() != 1:
                    raise NativeLibraryError("libcapsim_b200.so ABI version mismatch; rebuild it")
                _lib = L
    return _lib


def last_error() -> str:
    return lib().cs_last_error().decode("utf-8", "replace")


def check(rc: int, invalid: type[Exception] = ValueError) -> None:
    """Map a C status to an exception. The Python layer validates arguments first with the
    reference's own messages (errors.py:4-22, policy.py:137-138, sim.py:147-150), so a C-side
    CS_E_INVALID is raised as ``invalid`` (ValidationError for table staging)."""
    if rc == CS_OK:
        return
    msg = lib().cs_last_error().decode("utf-8", "replace")
    if rc == CS_E_INVALID:
        raise invalid(msg)
    if rc == CS_E_NODEVICE:
        raise NativeLibraryError(msg)
    if rc == CS_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise CudaError(msg)
