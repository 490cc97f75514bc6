"""GPU sampling selector (sampling kernel, policy.py:191-273 / sim.py:159-163) vs the reference's
own outputs (tests/golden/sampling_golden.json) and the pinned oracle at larger sizes: entries
and feasible counts bit-exact, aggregates bit-exact (math.fsum on both sides)."""

from __future__ import annotations

from datetime import datetime

import numpy as np
import pytest

from conftest import golden
from test_gpu_parity import oracle_grid
from test_staging_host import grid_from_doc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cs(cuda_ok):
    import paper_2306_12247_b200 as m

    return m


def _doc(sel):
    if sel.config is None:
        return [0, 0, 0.0, 0.0, sel.feasible_count]
    return [sel.config.mtl, sel.config.bs, sel.throughput_ips, sel.power_w, sel.feasible_count]


def test_select_sampling_matches_reference_golden(cs):
    n = 0
    for case in golden("sampling_golden.json")["cases"]:
        grid = grid_from_doc(case["grid"])
        for cap, budget, rounds, seed, want in case["queries"]:
            assert _doc(cs.select_sampling(grid, budget, rounds, cap, seed)) == want, (case["name"], cap, budget,
                                                                                       rounds, seed)
            n += 1
    assert n > 3000


def test_simulate_sampling_matches_reference_golden(cs):
    sim = golden("sampling_golden.json")["sim"]
    for run in sim["runs"]:
        grid = grid_from_doc(sim["grids"][run["name"]])
        tr = cs.PowerTrace(run["name"], 3600, datetime(2020, 1, 1), tuple(sim["traces"][run["name"]]))
        rep = cs.simulate(grid, tr, cs.sampling_policy(run["budget_m"], run["rounds_r"]), seed=run["seed"],
                          switch_penalty_s=run["switch_penalty_s"])
        key = (run["name"], run["budget_m"], run["rounds_r"], run["seed"], run["switch_penalty_s"])
        assert rep.avg_throughput_ips == run["avg_throughput_ips"], key
        assert rep.idle_steps == run["idle_steps"], key
        assert rep.energy_proxy_wh == run["energy_proxy_wh"], key
        assert [None if s.selection.config is None else _doc(s.selection) for s in rep.steps] == run["steps"], key


def test_sampling_steps_match_oracle_fine_grid(cs):
    """4096-entry grid: both random.sample branches, budgets past 227 MT outputs (the lazy twist
    catches up) and past the in-register maximum (scratch-pool variant), negative and >64-bit
    seeds, long hill climbs."""
    from oracle import oracle

    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    og = oracle_grid(g)
    rng = np.random.default_rng(5)
    caps = np.concatenate([[0.0, -0.0, 60.0, 350.0, 1e9], rng.uniform(0.0, 350.0, 250)])
    for budget, rounds, seed_base in ((1, 0, 0), (5, 3, -12345), (6, 1, 2**40), (37, 2, 99), (256, 0, 2**70 + 5),
                                      (256, 4, -(2**90)), (300, 1, 11), (1000, 0, -3), (4096, 1, 7)):
        sels = cs.sampling_steps(g, budget, rounds, caps.tolist(), seed_base)
        cfgs = g.columns()[0]
        for i, (cap, sel) in enumerate(zip(caps, sels)):
            idx, cnt = oracle.select_sampling(og, budget, rounds, float(cap), seed_base + i)
            want = None if idx < 0 else cfgs[idx]
            assert (sel.config, sel.feasible_count) == (want, cnt), (budget, rounds, seed_base, i, float(cap))


def test_simulate_many_sampling_matches_oracle(cs):
    from oracle import oracle

    grids = [cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=64, seed=s, noise_pct=2.0)) for s in (1, 2)]
    rng = np.random.default_rng(3)
    vals = np.clip(np.cumsum(rng.normal(0, 20, (6, 300)), axis=1) + 180, 0, 350)
    traces = [cs.PowerTrace(f"t{i}", 60, datetime(2020, 1, 1), tuple(v.tolist())) for i, v in enumerate(vals)]
    kinds = [cs.sampling_policy(3, 1), cs.COMBINATION, cs.sampling_policy(9, 0)]
    reps = cs.simulate_many(grids, traces, kinds=kinds, seed=4, switch_penalty_s=20.0)
    for t in range(len(traces)):
        for m, g in enumerate(grids):
            og = oracle_grid(g)
            for k, kind in enumerate(kinds):
                if kind.tag is cs.PolicyTag.SAMPLING:
                    want = oracle.simulate_sampling(og, vals[t], kind.budget_m, kind.rounds_r, 4, 60, 20.0)
                else:
                    want = oracle.simulate(og, vals[t], "combination", 60, 20.0)
                r = reps[t][m][k]
                assert r.avg_throughput_ips == want.avg_throughput_ips
                assert r.idle_steps == want.idle_steps
                assert r.energy_proxy_wh == want.energy_proxy_wh


def test_sampling_errors(cs):
    g1 = grid_from_doc(golden("sim_golden.json")["grids"]["g1"])
    with pytest.raises(ValueError, match="budget_m"):
        cs.select_sampling(g1, 0, 0, 200.0, 0)
    with pytest.raises(ValueError, match="rounds_r"):
        cs.select_sampling(g1, 1, -1, 200.0, 0)
    with pytest.raises(ValueError, match="cap_w"):
        cs.select_sampling(g1, 1, 0, -1.0, 0)
    assert cs.select_sampling(g1, 4, 2, float("nan"), 0).config is None
    big = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    assert cs.select_sampling(big, 5000, 0, 200.0, 0) == cs.select_config(big, cs.COMBINATION, 200.0)


def test_device_entry_aggregate_matches_fsum(cs):
    """cs_entries_aggregate (simulate_many's sampling summaries) vs the reference's _aggregate
    restated on the host with math.fsum, over random per-step selections and penalties."""
    import torch

    from paper_2306_12247_b200.sim import _sampling_aggregate

    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128, noise_pct=2.0, seed=9))
    tables = cs.Tables.stage([g], "f64")
    rng = np.random.default_rng(17)
    n = len(g.entries)
    for S, pen, step in ((1, 0.0, 60), (777, 0.0, 60), (10080, 20.0, 60), (5000, 7200.0, 3600)):
        ent = rng.integers(-1, n, size=(64, S)).astype(np.int32)
        ent[:8] = np.repeat(rng.integers(-1, n, size=(8, 1)), S, axis=1)  # constant rows
        avg, en, idle = tables.aggregate_entries(0, torch.from_numpy(ent).cuda(), S, step_seconds=step,
                                                 switch_penalty_s=pen)
        avg, en, idle = avg.cpu().numpy(), en.cpu().numpy(), idle.cpu().numpy()
        want = [_sampling_aggregate(g, ent[t], step, float(g.gpu_idle_power_w or 0.0), pen) for t in range(64)]
        wa = np.array([w[0] for w in want])
        we = np.array([w[2] for w in want])
        assert np.array_equal(idle, [w[1] for w in want])
        assert np.allclose(avg, wa, rtol=1e-12, atol=0) and np.allclose(en, we, rtol=1e-12, atol=0)
        assert np.mean(avg == wa) >= 0.95 and np.mean(en == we) >= 0.95
