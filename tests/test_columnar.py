"""Columnar results: Parquet rows == the reference's schema-v1 report fields.

CPU: reports with per-step records (built from the oracle, itself pinned to the reference's
golden vectors) round-trip through summary / steps tables; each summary row equals
report_to_dict(report, summary_only=True) and each steps row equals an entry of its "steps"."""

from __future__ import annotations

import datetime as dt

import numpy as np
import pytest

import paper_2306_12247_b200 as cs
from paper_2306_12247_b200 import columnar as col

REGIMES = {"batching": cs.BATCHING, "multi-tenant": cs.MULTI_TENANT, "combination": cs.COMBINATION}


def oracle_reports():
    from oracle import oracle

    grids = [cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=16, model_name="tiny-a")),
             cs.synthesize_grid(cs.SynthParams(mtl_cap=3, bs_cap=8, t_max_ips=5000.0, model_name="tiny-b",
                                               p_idle_w=80.0))]
    rng = np.random.default_rng(3)
    reports, tix = [], []
    for t in range(3):
        caps = np.clip(np.cumsum(rng.normal(0, 30, 200)) + 200, 0, 350)
        caps[:7] = 0.0
        for g in grids:
            cfgs, mtl, bs, thr, pw = g.columns()
            og = oracle.GridArrays(np.array(mtl, np.int32), np.array(bs, np.int32), np.array(thr), np.array(pw),
                                   float(g.gpu_idle_power_w or 0.0))
            for name, kind in REGIMES.items():
                r = oracle.simulate(og, caps, name, 60, 0.0)
                steps = []
                for i, (cap, s, c) in enumerate(zip(caps, r.sel, r.count)):
                    sel = (cs.Selection(None, 0.0, 0.0, 0) if s < 0 else
                           cs.Selection(cfgs[s], thr[s], pw[s], int(c)))
                    steps.append(cs.StepRecord(i, float(cap), sel, s < 0))
                reports.append(cs.SimReport(g.model_name, kind, f"trace-{t}", 60, float(g.gpu_idle_power_w or 0.0),
                                            len(caps), r.avg_throughput_ips, r.idle_steps, r.energy_proxy_wh,
                                            tuple(steps)))
                tix.append(t)
    samp = cs.sampling_policy(4, 2)
    reports.append(cs.SimReport("tiny-a", samp, "trace-0", 60, 60.0, 5, 123.5, 1, 9.75, None))
    tix.append(0)
    return reports, tix


def test_summary_rows_equal_schema_v1_fields(tmp_path):
    reports, tix = oracle_reports()
    summ = col.reports_table(reports, tix)
    assert summ.num_rows == len(reports)
    assert col.row_dicts(summ) == [cs.report_to_dict(r, summary_only=True) for r in reports]
    steps = col.steps_table(reports, tix)
    assert steps.num_rows == sum(r.num_steps for r in reports if r.steps is not None)
    out = col.save_columnar(tmp_path / "run", summ, steps=steps, params={"switch_penalty_s": 0.0})
    run = col.load_columnar(out)
    assert run.manifest["format"] == col.COLUMNAR_FORMAT and run.manifest["rows"] == len(reports)
    assert run.summary.equals(summ) and run.steps.equals(steps) and run.histogram is None
    back = col.table_to_reports(run.summary)
    assert back == [cs.SimReport(r.model_name, r.policy, r.trace_label, r.step_seconds, r.idle_power_w,
                                 r.num_steps, r.avg_throughput_ips, r.idle_steps, r.energy_proxy_wh, None)
                    for r in reports]
    # steps rows == report_to_dict(...)["steps"] entries
    sd = run.steps.to_pydict()
    want = [s for r in reports if r.steps is not None for s in cs.report_to_dict(r)["steps"]]
    for i in (0, 1, 50, len(want) - 1):
        got = {"step_index": sd["step_index"][i], "cap_w": sd["cap_w"][i], "idle": sd["idle"][i],
               "config": None if sd["mtl"][i] is None else {"mtl": sd["mtl"][i], "bs": sd["bs"][i]},
               "throughput_ips": sd["throughput_ips"][i], "power_w": sd["power_w"][i],
               "feasible_count": sd["feasible_count"][i]}
        assert got == want[i]


def test_rejects_foreign_directories(tmp_path):
    (tmp_path / "manifest.json").write_text('{"format": "other", "version": 1}')
    with pytest.raises(cs.ValidationError):
        col.load_columnar(tmp_path)


def test_reports_table_is_columnar_not_json(tmp_path):
    """10^5 summary rows write and read back in well under a second per 10^5 (no JSON docs)."""
    import time

    n = 100_000
    rep = cs.SimReport("m", cs.COMBINATION, "t", 60, 0.0, 10, 1.0, 0, 1.0, None)
    summ = col.reports_table([rep] * 1000)
    import pyarrow as pa

    big = pa.concat_tables([summ] * (n // 1000))
    t = time.perf_counter()
    col.save_columnar(tmp_path / "big", big)
    assert col.load_columnar(tmp_path / "big").summary.num_rows == n
    assert time.perf_counter() - t < 10
