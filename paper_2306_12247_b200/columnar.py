"""Columnar results: the sweep's reports as Parquet tables.

The reference serialises one SimReport per JSON document (schema v1, sim.py:258-431) with an
optional per-step array — fine for one run, infeasible for 10^6 traces x grids x policies. This
module writes the same fields column-wise, one row per (trace, grid, policy), plus the global
config histogram and, for small runs, the per-step records. A directory holds:

    manifest.json              format name/version, report schema version, run parameters
    summary.parquet            report_to_dict(summary_only=True) fields, one row per report
    config_histogram.parquet   steps per (grid, policy, config) (idle = null config)
    steps.parquet (optional)   the per-step records of report_to_dict's "steps" array

Row i of summary.parquet and report_to_dict(report_i, summary_only=True) hold the same values
(tests/test_columnar.py); table_to_reports() rebuilds summary-only SimReports.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import ValidationError
from .policy import BATCHING, COMBINATION, MULTI_TENANT, PolicyKind, PolicyTag
from .sim import REPORT_SCHEMA_VERSION, SimReport

COLUMNAR_FORMAT = "capsim-columnar"
COLUMNAR_VERSION = 1
_EXHAUSTIVE = (BATCHING, MULTI_TENANT, COMBINATION)  # the engine's policy axis order


def _pa():
    import pyarrow as pa

    return pa


def _summary_schema():
    pa = _pa()
    d = pa.dictionary(pa.int32(), pa.string())
    return pa.schema([
        ("trace", pa.int64()), ("trace_label", d), ("model_name", d), ("policy_tag", d),
        ("budget_m", pa.int32()), ("rounds_r", pa.int32()), ("step_seconds", pa.int32()),
        ("idle_power_w", pa.float64()), ("num_steps", pa.int64()), ("avg_throughput_ips", pa.float64()),
        ("idle_steps", pa.int64()), ("energy_proxy_wh", pa.float64()), ("switches", pa.int64()),
        ("violations", pa.int64()),
    ])


def _dict_col(codes: np.ndarray, values: Sequence[str]):
    pa = _pa()
    return pa.DictionaryArray.from_arrays(pa.array(codes.astype(np.int32)), pa.array(list(values), pa.string()))


def reports_table(reports: Sequence[SimReport], trace_index: Sequence[int] | None = None):
    """Summary table of existing SimReports (any policy, sampling included)."""
    pa = _pa()
    n = len(reports)
    labels = sorted({r.trace_label for r in reports})
    models = sorted({r.model_name for r in reports})
    tags = [t.value for t in PolicyTag]
    li, mi, ti = ({v: i for i, v in enumerate(x)} for x in (labels, models, tags))
    cols = {
        "trace": pa.array(np.arange(n) if trace_index is None else np.asarray(trace_index), pa.int64()),
        "trace_label": _dict_col(np.array([li[r.trace_label] for r in reports]), labels),
        "model_name": _dict_col(np.array([mi[r.model_name] for r in reports]), models),
        "policy_tag": _dict_col(np.array([ti[r.policy.tag.value] for r in reports]), tags),
        "budget_m": pa.array([r.policy.budget_m for r in reports], pa.int32()),
        "rounds_r": pa.array([r.policy.rounds_r for r in reports], pa.int32()),
        "step_seconds": pa.array([r.step_seconds for r in reports], pa.int32()),
        "idle_power_w": pa.array([r.idle_power_w for r in reports], pa.float64()),
        "num_steps": pa.array([r.num_steps for r in reports], pa.int64()),
        "avg_throughput_ips": pa.array([r.avg_throughput_ips for r in reports], pa.float64()),
        "idle_steps": pa.array([r.idle_steps for r in reports], pa.int64()),
        "energy_proxy_wh": pa.array([r.energy_proxy_wh for r in reports], pa.float64()),
        "switches": pa.nulls(n, pa.int64()),
        "violations": pa.array(np.zeros(n, np.int64)),
    }
    return pa.table(cols, schema=_summary_schema())


def eval_table(result, *, trace_labels: Sequence[str], step_seconds: int, first_trace: int = 0):
    """Summary table straight from a batched evaluation (engine.EvalResult): T x M x 3 rows in
    (trace, grid, policy) order, built vectorised from the device aggregates — no per-report
    Python objects, so 10^6-trace sweeps serialise in seconds."""
    pa = _pa()
    agg = result.agg.cpu().numpy() if hasattr(result.agg, "cpu") else np.asarray(result.agg)
    T, M, P, _ = agg.shape
    ints = agg.view(np.int64)
    if len(trace_labels) != T:
        raise ValueError(f"need {T} trace labels, got {len(trace_labels)}")
    grids = result.tables.grids
    n = T * M * P
    labels = list(trace_labels)
    uniq, inv = np.unique(np.array(labels, dtype=object), return_inverse=True)
    idle_pw = np.array([g.gpu_idle_power_w if g.gpu_idle_power_w is not None else 0.0 for g in grids])
    cols = {
        "trace": pa.array(np.repeat(np.arange(first_trace, first_trace + T, dtype=np.int64), M * P)),
        "trace_label": _dict_col(np.repeat(inv, M * P), [str(u) for u in uniq]),
        "model_name": _dict_col(np.tile(np.repeat(np.arange(M), P), T), [g.model_name for g in grids]),
        "policy_tag": _dict_col(np.tile(np.arange(P), T * M), [k.tag.value for k in _EXHAUSTIVE]),
        "budget_m": pa.array(np.zeros(n, np.int32)),
        "rounds_r": pa.array(np.zeros(n, np.int32)),
        "step_seconds": pa.array(np.full(n, step_seconds, np.int32)),
        "idle_power_w": pa.array(np.tile(np.repeat(idle_pw, P), T)),
        "num_steps": pa.array(ints[..., 5].reshape(-1)),
        "avg_throughput_ips": pa.array(agg[..., 0].reshape(-1)),
        "idle_steps": pa.array(ints[..., 2].reshape(-1)),
        "energy_proxy_wh": pa.array(agg[..., 1].reshape(-1)),
        "switches": pa.array(ints[..., 3].reshape(-1)),
        "violations": pa.array(ints[..., 4].reshape(-1)),
    }
    return pa.table(cols, schema=_summary_schema())


def histogram_table(tables, hist):
    """Global config histogram: steps per (grid, exhaustive policy, config); idle rows have null
    mtl / bs. Integer-exact (Tables.config_histograms). ``hist`` may also be the EvalResult
    itself (required for grid-chunked runs, whose union-bin histograms are per chunk)."""
    pa = _pa()
    model, tag, mtl, bs, steps = [], [], [], [], []
    rows = hist.config_histograms() if hasattr(hist, "config_histograms") else tables.config_histograms(hist)
    for m, row in enumerate(rows):
        for p, d in enumerate(row):
            for cfg, c in sorted(d.items(), key=lambda kv: (kv[0] is not None, kv[0] or (0, 0))):
                model.append(tables.grids[m].model_name)
                tag.append(_EXHAUSTIVE[p].tag.value)
                mtl.append(None if cfg is None else cfg.mtl)
                bs.append(None if cfg is None else cfg.bs)
                steps.append(c)
    return pa.table({"model_name": pa.array(model, pa.string()), "policy_tag": pa.array(tag, pa.string()),
                     "mtl": pa.array(mtl, pa.int32()), "bs": pa.array(bs, pa.int32()),
                     "steps": pa.array(steps, pa.int64())})


def steps_table(reports: Sequence[SimReport], trace_index: Sequence[int] | None = None):
    """The per-step records of reports that carry them (report_to_dict's "steps"), long format."""
    pa = _pa()
    cols: dict[str, list] = {k: [] for k in ("report", "trace", "step_index", "cap_w", "idle", "mtl", "bs",
                                             "throughput_ips", "power_w", "feasible_count")}
    for i, r in enumerate(reports):
        if r.steps is None:
            continue
        t = i if trace_index is None else trace_index[i]
        for s in r.steps:
            c = s.selection.config
            cols["report"].append(i)
            cols["trace"].append(t)
            cols["step_index"].append(s.step_index)
            cols["cap_w"].append(s.cap_w)
            cols["idle"].append(s.idle)
            cols["mtl"].append(None if c is None else c.mtl)
            cols["bs"].append(None if c is None else c.bs)
            cols["throughput_ips"].append(s.selection.throughput_ips)
            cols["power_w"].append(s.selection.power_w)
            cols["feasible_count"].append(s.selection.feasible_count)
    types = {"report": pa.int64(), "trace": pa.int64(), "step_index": pa.int64(), "cap_w": pa.float64(),
             "idle": pa.bool_(), "mtl": pa.int32(), "bs": pa.int32(), "throughput_ips": pa.float64(),
             "power_w": pa.float64(), "feasible_count": pa.int64()}
    return pa.table({k: pa.array(v, types[k]) for k, v in cols.items()})


@dataclass
class ColumnarRun:
    manifest: dict
    summary: object            # pyarrow.Table
    histogram: object = None   # pyarrow.Table or None
    steps: object = None       # pyarrow.Table or None


def save_columnar(path: str | Path, summary, *, histogram=None, steps=None, params: dict | None = None) -> Path:
    """Write a columnar run directory (manifest + Parquet tables); files are replaced atomically."""
    import os

    import pyarrow.parquet as pq

    out = Path(path)
    out.mkdir(parents=True, exist_ok=True)
    manifest = {"format": COLUMNAR_FORMAT, "version": COLUMNAR_VERSION, "report_schema_version": REPORT_SCHEMA_VERSION,
                "rows": summary.num_rows, "tables": ["summary"] + (["config_histogram"] if histogram is not None else [])
                + (["steps"] if steps is not None else []), "params": params or {}}
    for name, tab in (("summary", summary), ("config_histogram", histogram), ("steps", steps)):
        if tab is None:
            continue
        tmp = out / f".{name}.parquet.tmp"
        pq.write_table(tab, tmp, compression="zstd")
        os.replace(tmp, out / f"{name}.parquet")
    tmp = out / ".manifest.json.tmp"
    tmp.write_text(json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    os.replace(tmp, out / "manifest.json")
    return out


def load_columnar(path: str | Path) -> ColumnarRun:
    import pyarrow.parquet as pq

    d = Path(path)
    manifest = json.loads((d / "manifest.json").read_text())
    if manifest.get("format") != COLUMNAR_FORMAT:
        raise ValidationError(f"not a {COLUMNAR_FORMAT} directory", path=str(d))
    if manifest.get("version") != COLUMNAR_VERSION:
        raise ValidationError(f"unsupported {COLUMNAR_FORMAT} version {manifest.get('version')}", path=str(d))
    tabs = {n: pq.read_table(d / f"{n}.parquet") if (d / f"{n}.parquet").exists() else None
            for n in ("summary", "config_histogram", "steps")}
    if tabs["summary"] is None:
        raise ValidationError("summary.parquet missing", path=str(d))
    return ColumnarRun(manifest, tabs["summary"], tabs["config_histogram"], tabs["steps"])


def row_dicts(summary) -> list[dict]:
    """report_to_dict(..., summary_only=True) of every row."""
    cols = summary.to_pydict()
    out = []
    for i in range(summary.num_rows):
        out.append({
            "schema_version": REPORT_SCHEMA_VERSION,
            "model_name": cols["model_name"][i],
            "trace_label": cols["trace_label"][i],
            "policy": {"tag": cols["policy_tag"][i], "budget_m": cols["budget_m"][i], "rounds_r": cols["rounds_r"][i]},
            "step_seconds": cols["step_seconds"][i],
            "idle_power_w": cols["idle_power_w"][i],
            "num_steps": cols["num_steps"][i],
            "avg_throughput_ips": cols["avg_throughput_ips"][i],
            "idle_steps": cols["idle_steps"][i],
            "energy_proxy_wh": cols["energy_proxy_wh"][i],
        })
    return out


def table_to_reports(summary) -> list[SimReport]:
    """Summary-only SimReports (steps=None) of every row, as simulate_many returns them."""
    out = []
    for d in row_dicts(summary):
        p = d["policy"]
        kind = PolicyKind(PolicyTag(p["tag"]), p["budget_m"], p["rounds_r"])
        out.append(SimReport(model_name=d["model_name"], policy=kind, trace_label=d["trace_label"],
                             step_seconds=d["step_seconds"], idle_power_w=d["idle_power_w"],
                             num_steps=d["num_steps"], avg_throughput_ips=d["avg_throughput_ips"],
                             idle_steps=d["idle_steps"], energy_proxy_wh=d["energy_proxy_wh"], steps=None))
    return out
