"""The sampling-selector restatement (oracle ora_select_sampling: CPython's Random.sample on the
MT19937 stream + the neighbour hill climb) pinned to the reference's own outputs
(tests/golden/sampling_golden.json, policy.py:191-273 and sim.py:159-163)."""

from __future__ import annotations

from conftest import golden, grid_arrays
from oracle import oracle


def _doc(grid_doc, idx, cnt):
    if idx < 0:
        return [0, 0, 0.0, 0.0, cnt]
    m, b, t, p = grid_doc["entries"][idx]
    return [m, b, t, p, cnt]


def test_select_sampling_matches_reference():
    doc = golden("sampling_golden.json")
    n = 0
    for case in doc["cases"]:
        g = grid_arrays(case["grid"])
        for cap, budget, rounds, seed, want in case["queries"]:
            idx, cnt = oracle.select_sampling(g, budget, rounds, cap, seed)
            assert _doc(case["grid"], idx, cnt) == want, (case["name"], cap, budget, rounds, seed)
            n += 1
    assert n > 3000


def test_simulate_sampling_matches_reference():
    sim = golden("sampling_golden.json")["sim"]
    for run in sim["runs"]:
        gdoc = sim["grids"][run["name"]]
        g = grid_arrays(gdoc)
        caps = sim["traces"][run["name"]]
        res = oracle.simulate_sampling(g, caps, run["budget_m"], run["rounds_r"], run["seed"], 3600,
                                       run["switch_penalty_s"])
        assert res.avg_throughput_ips == run["avg_throughput_ips"]
        assert res.idle_steps == run["idle_steps"]
        assert res.energy_proxy_wh == run["energy_proxy_wh"]
        got = [None if i < 0 else _doc(gdoc, int(i), int(c)) for i, c in zip(res.sel, res.count)]
        assert got == run["steps"]
