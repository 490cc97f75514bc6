"""GPU controller replay vs the reference's own replays (golden) and the pinned oracle."""

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


def _sel_doc(sel):
    if sel.config is None:
        return None
    return [sel.config.mtl, sel.config.bs, sel.throughput_ips, sel.power_w, sel.feasible_count]


def test_replay_matches_reference_golden(cs):
    for case in golden("controller_golden.json")["cases"]:
        grid = grid_from_doc(case["grid"])
        mode = cs.REACTIVE if case["mode"] == "reactive" else cs.proactive(case["window_k"])
        init = None if case["initial"] is None else cs.Config(*case["initial"])
        trace = cs.PowerTrace(case["name"], 60, datetime(2020, 1, 1), tuple(case["caps"]))
        rep = cs.replay(grid, trace, mode, initial_config=init, noise_pct=case["noise_pct"], seed=case["seed"])
        key = case["name"]
        assert rep.violations == case["violations"], key
        assert rep.reconfigs == case["reconfigs"], key
        assert rep.violation_fraction == case["violation_fraction"], key
        assert rep.avg_throughput_ips == pytest.approx(case["avg_throughput_ips"], rel=1e-12, abs=0), key
        assert [[e.step_index, e.kind.value, e.cap_w, e.power_w] for e in rep.events] == case["events"], key
        assert [_sel_doc(s) for s in rep.selections] == case["selections"], key


def test_replay_fixtures_from_reference_tests(cs):
    g1 = grid_from_doc(golden("sim_golden.json")["grids"]["g1"])
    tr = cs.PowerTrace("t", 3600, datetime(2020, 1, 1), (250.0, 150.0))
    rep = cs.replay(g1, tr, cs.REACTIVE, initial_config=cs.Config(2, 2))
    assert rep.avg_throughput_ips == pytest.approx((300.0 + 180.0) / 2)
    lines = cs.event_log_csv_text(rep).splitlines()
    assert lines[0] == "step,kind,cap_w,power_w,mtl,bs,throughput_ips"
    assert lines[1].startswith("0,no_action,250.000000,220.000000,2,2,")
    with pytest.raises(cs.ValidationError, match="not present"):
        cs.replay(g1, cs.PowerTrace("t", 60, datetime(2020, 1, 1), (200.0,)), cs.REACTIVE,
                  initial_config=cs.Config(9, 9))


def test_replay_many_matches_oracle(cs):
    from oracle import oracle

    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=32, noise_pct=1.0, seed=3))
    rng = np.random.default_rng(8)
    caps = np.clip(np.cumsum(rng.normal(0, 15, (40, 700)), axis=1) + 200, 0, 350)
    og = oracle_grid(g)
    # windows beyond the old 256-sample history buffer: any window_k >= 1 works
    for mode, k, noise, seed in ((cs.REACTIVE, 1, 0.0, 0), (cs.proactive(4), 4, 3.0, 77),
                                 (cs.ControlMode(cs.REACTIVE.tag, window_k=300), 300, 2.0, 5),
                                 (cs.proactive(300), 300, 1.0, 9), (cs.proactive(1000), 1000, 0.0, 1)):
        s = cs.replay_many(g, caps, mode, noise_pct=noise, seed=seed)
        for t in range(caps.shape[0]):
            proactive = mode.tag is not cs.REACTIVE.tag
            r = oracle.replay(og, caps[t], "proactive" if proactive else "reactive", k, -1, noise, seed + t)
            assert s.violations[t] == r.violations and s.reconfigs[t] == r.reconfigs
            assert s.avg_throughput_ips[t] == pytest.approx(r.avg_throughput_ips, rel=1e-12, abs=0)
