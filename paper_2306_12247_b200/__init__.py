"""paper_2306_12247_b200 — B200-native engine for the trace-driven policy-evaluation path of
capsim (arXiv 2306.12247, "Opportunities of Renewable Energy Powered DNN Inference").

A drop-in for the reference's hot path: same names, signatures and records as
capsim/__init__.py:8-116 for profile tables, power traces, the batching / multi-tenant /
combination policies and simulate(); every decision runs in hand-written sm_100a kernels
(libcapsim_b200.so via ctypes). Use it as ``import paper_2306_12247_b200 as capsim``.

Also on the GPU: the online controller replay (controller.py) and the
sampling selector (select_sampling / simulate with sampling_policy, §8(f) rank 2). Trace CSVs
load through a native parser (load_trace / load_traces / load_trace_matrix, rank 3) and sweeps
serialise as Parquet tables (columnar.py, rank 4). Out of scope: the CLI.
"""

from .controller import (
    REACTIVE,
    ControlEvent,
    ControllerReport,
    ControllerState,
    ControlMode,
    EventKind,
    event_log_csv_text,
    moving_average_prediction,
    proactive,
    replay,
    replay_many,
    step_proactive,
    step_reactive,
)
from .columnar import (
    ColumnarRun,
    eval_table,
    histogram_table,
    load_columnar,
    reports_table,
    save_columnar,
    steps_table,
    table_to_reports,
)
from .engine import EvalResult, HostEngine, Tables, generate_traces
from .shard import (DeviceComm, MultiDeviceResult, ShardedResult, SweepTotals, evaluate_devices, evaluate_sharded,
                    shard_range, sweep_words)
from .errors import CapsimError, ParseError, ValidationError
from .policy import (
    BATCHING,
    COMBINATION,
    IDLE_SELECTION,
    MULTI_TENANT,
    PolicyIndex,
    PolicyKind,
    PolicyTag,
    Selection,
    feasible_set,
    improvement_pct,
    sampling_policy,
    sampling_steps,
    select_config,
    select_configs,
    select_sampling,
)
from .profile import (
    Config,
    ProfileEntry,
    ProfileGrid,
    SynthParams,
    compute_throughput,
    grid_csv_text,
    load_grid,
    profiling_cost,
    save_grid,
    synthesize_grid,
)
from .sim import (
    REPORT_SCHEMA,
    ComparisonRow,
    ComparisonTable,
    SimReport,
    StepRecord,
    compare,
    comparison_csv_text,
    load_report,
    report_from_dict,
    report_json_text,
    report_to_dict,
    save_report,
    simulate,
    simulate_many,
    slice_report,
)
from .trace import (
    PowerTrace,
    TraceMatrix,
    TraceStats,
    load_trace,
    load_trace_matrix,
    load_traces,
    normalize_display,
    normalize_trace,
    save_trace,
    trace_array,
    trace_csv_text,
    trace_stats,
)

__version__ = "0.1.0"

__all__ = [
    "BATCHING", "COMBINATION", "MULTI_TENANT", "IDLE_SELECTION",
    "CapsimError", "ParseError", "ValidationError",
    "ComparisonRow", "ComparisonTable", "Config", "PolicyIndex", "PolicyKind", "PolicyTag", "PowerTrace",
    "ProfileEntry", "ProfileGrid", "Selection", "SimReport", "StepRecord", "SynthParams", "TraceStats",
    "REPORT_SCHEMA",
    "compare", "comparison_csv_text", "compute_throughput", "feasible_set", "grid_csv_text", "improvement_pct",
    "load_grid", "load_report", "load_trace", "normalize_display", "normalize_trace", "profiling_cost",
    "report_from_dict", "report_json_text", "report_to_dict", "sampling_policy", "sampling_steps", "save_grid", "save_report",
    "save_trace", "select_config", "select_configs", "select_sampling", "simulate", "simulate_many",
    "slice_report", "synthesize_grid", "trace_array", "trace_csv_text", "trace_stats",
    "Tables", "EvalResult", "HostEngine", "generate_traces", "TraceMatrix",
    "ShardedResult", "SweepTotals", "evaluate_sharded", "evaluate_devices", "DeviceComm", "MultiDeviceResult", "shard_range", "sweep_words", "load_traces", "load_trace_matrix",
    "ColumnarRun", "eval_table", "histogram_table", "load_columnar", "reports_table", "save_columnar", "steps_table",
    "table_to_reports",
    "REACTIVE", "ControlEvent", "ControllerReport", "ControllerState", "ControlMode", "EventKind",
    "event_log_csv_text", "moving_average_prediction", "proactive", "replay", "replay_many", "step_proactive",
    "step_reactive",
]
