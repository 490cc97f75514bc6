"""GPU: columnar results straight from a batched evaluation (eval_table / histogram_table) hold
the same values as simulate_many's SimReports (report_to_dict, schema v1) and the oracle."""

from __future__ import annotations

import datetime as dt

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_eval_table_matches_reports_and_oracle(cuda_ok, tmp_path):
    import torch

    import paper_2306_12247_b200 as cs
    from oracle import oracle
    from paper_2306_12247_b200 import columnar as col

    grids = [cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=32, model_name="m-a")),
             cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=64, t_max_ips=7000.0, p_idle_w=40.0,
                                               model_name="m-b"))]
    rng = np.random.default_rng(9)
    T, S = 6, 999
    caps = np.clip(np.cumsum(rng.normal(0, 20, (T, S)), axis=1) + 150, 0, 350)
    traces = [cs.PowerTrace(f"tr{t}", 60, dt.datetime(2020, 1, 1), tuple(caps[t].tolist())) for t in range(T)]
    reports = cs.simulate_many(grids, traces, switch_penalty_s=7.0)
    tables = cs.Tables.stage(grids, "f64")
    host = np.zeros((T, S + 1))
    host[:, :S] = caps
    res = tables.evaluate(torch.from_numpy(host).cuda(), S, step_seconds=60, switch_penalty_s=7.0)
    summ = col.eval_table(res, trace_labels=[t.source_label for t in traces], step_seconds=60)
    assert summ.num_rows == T * len(grids) * 3
    flat = [reports[t][m][p] for t in range(T) for m in range(len(grids)) for p in range(3)]
    assert col.row_dicts(summ) == [cs.report_to_dict(r, summary_only=True) for r in flat]
    d = summ.to_pydict()
    for i, r in enumerate(flat):  # and the oracle (reference algorithm) for every row
        g = grids[i // 3 % len(grids)]
        cfgs, mtl, bs, thr, pw = g.columns()
        og = oracle.GridArrays(np.array(mtl, np.int32), np.array(bs, np.int32), np.array(thr), np.array(pw),
                               float(g.gpu_idle_power_w or 0.0))
        o = oracle.simulate(og, caps[i // (3 * len(grids))], r.policy.tag.value, 60, 7.0)
        assert d["idle_steps"][i] == o.idle_steps and d["violations"][i] == 0
        assert abs(d["avg_throughput_ips"][i] - o.avg_throughput_ips) <= 1e-6 * abs(o.avg_throughput_ips)
        assert abs(d["energy_proxy_wh"][i] - o.energy_proxy_wh) <= 1e-6 * abs(o.energy_proxy_wh)
    hist = col.histogram_table(tables, res.hist)
    h = hist.to_pydict()
    for m, g in enumerate(grids):
        for tag in ("batching", "multi-tenant", "combination"):
            tot = sum(s for mn, tg, s in zip(h["model_name"], h["policy_tag"], h["steps"]) if mn == g.model_name
                      and tg == tag)
            assert tot == T * S
    run = col.load_columnar(col.save_columnar(tmp_path / "sweep", summ, histogram=hist,
                                              params={"switch_penalty_s": 7.0}))
    assert run.summary.equals(summ) and run.histogram.equals(hist)
    assert col.table_to_reports(run.summary) == flat
