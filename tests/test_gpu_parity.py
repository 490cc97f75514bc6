"""GPU parity: the CUDA path (through libcapsim_b200.so) against the reference's golden
vectors and the pinned CPU oracle. Bar: bit-exact selections, feasible counts, idle counts and
histograms; averages / energies equal (the kernel's double-double epilogue reproduces
math.fsum) and in any case within the north star's 1e-6 relative tolerance."""

from __future__ import annotations

import hashlib
import math
import struct

import numpy as np
import pytest

from conftest import REGIMES, golden, sel_tuple
from test_staging_host import grid_from_doc

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6  # north star tolerance for fp64 sums; the kernel is expected to be exact


@pytest.fixture(scope="module")
def torch(cuda_ok):
    import torch as T

    return T


@pytest.fixture(scope="module")
def cs(cuda_ok):
    import paper_2306_12247_b200 as m

    return m


def oracle_grid(grid):
    from oracle import oracle

    cfgs, mtl, bs, thr, pw = grid.columns()
    return oracle.GridArrays(np.array(mtl, np.int32), np.array(bs, np.int32), np.array(thr, np.float64),
                             np.array(pw, np.float64),
                             0.0 if grid.gpu_idle_power_w is None else float(grid.gpu_idle_power_w))


def sel_doc(sel):
    if sel.config is None:
        return None
    return [sel.config.mtl, sel.config.bs, sel.throughput_ips, sel.power_w, sel.feasible_count]


# ---------------------------------------------------------------------------------------------
# per-cap API (select_config / PolicyIndex / feasible_set) vs the reference


def test_select_config_golden(cs):
    doc = golden("policy_golden.json")
    kinds = {"batching": cs.BATCHING, "multi-tenant": cs.MULTI_TENANT, "combination": cs.COMBINATION}
    for case in doc["cases"]:
        grid = grid_from_doc(case["grid"])
        kw = dict(batching_mtl=case["batching_mtl"], multi_tenant_bs=case["multi_tenant_bs"])
        for regime in REGIMES:
            got = [sel_doc(s) for s in cs.select_configs(grid, kinds[regime], case["caps"], **kw)]
            assert got == case["select"][regime], (case["name"], regime)
            idx = cs.PolicyIndex(grid, kinds[regime], **kw)
            got = [sel_doc(s) for s in idx.select_many(case["caps"])]
            assert got == case["select"][regime], (case["name"], regime, "index")
            for cap, want in zip(case["feasible_caps"], case["feasible_set"][regime]):
                fs = cs.feasible_set(grid, kinds[regime], cap, **kw)
                assert sorted([c.mtl, c.bs] for c in fs) == want


def test_policy_index_of_sampling_kind_is_combination(cs):
    """PolicyIndex(grid, sampling_policy(m, r)) indexes every entry like the combination regime
    (reference policy.py:100-107, 118-134); only select_config rejects sampling kinds."""
    doc = golden("policy_golden.json")
    by_name = {c["name"]: c for c in doc["cases"]}
    for name, want in doc["sampling_index"].items():
        case = by_name[name]
        grid = grid_from_doc(case["grid"])
        idx = cs.PolicyIndex(grid, cs.sampling_policy(4, 2))
        assert [sel_doc(s) for s in idx.select_many(case["caps"])] == want, name
        assert want == case["select"]["combination"], name


def test_select_config_quirks(cs):
    doc = golden("policy_golden.json")
    g1 = grid_from_doc(doc["cases"][0]["grid"])
    kinds = {"batching": cs.BATCHING, "multi-tenant": cs.MULTI_TENANT, "combination": cs.COMBINATION}
    for regime in REGIMES:
        for key, cap in (("inf", math.inf), ("nan", math.nan)):
            assert sel_doc(cs.select_config(g1, kinds[regime], cap)) == doc["g1_quirks"][regime][key]
            assert sel_doc(cs.PolicyIndex(g1, kinds[regime]).select(cap)) == doc["g1_quirks"][regime][key]
    with pytest.raises(ValueError, match="select_sampling"):
        cs.select_config(g1, cs.sampling_policy(2), 200.0)
    with pytest.raises(ValueError):
        cs.select_config(g1, cs.COMBINATION, -1.0)
    assert cs.feasible_set(g1, cs.COMBINATION, math.nan) == set()


# ---------------------------------------------------------------------------------------------
# simulate() vs the reference's own reports


def _digest(report):
    order = [-1 if s.selection.config is None else s.selection.config.mtl * 100000 + s.selection.config.bs
             for s in report.steps]
    counts = [s.selection.feasible_count for s in report.steps]
    raw = struct.pack(f"<{len(order)}q", *order) + struct.pack(f"<{len(counts)}q", *counts)
    return hashlib.sha256(raw).hexdigest()


def test_simulate_golden_bit_exact(cs):
    doc = golden("sim_golden.json")
    kinds = {"batching": cs.BATCHING, "multi-tenant": cs.MULTI_TENANT, "combination": cs.COMBINATION}
    grids = {k: grid_from_doc(v) for k, v in doc["grids"].items()}
    import warnings

    for run in doc["runs"]:
        trace = cs.PowerTrace(run["trace"], run["step_seconds"], __import__("datetime").datetime(2020, 1, 1),
                              tuple(doc["traces"][run["trace"]]))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = cs.simulate(grids[run["grid"]], trace, kinds[run["policy"]],
                              switch_penalty_s=run["switch_penalty_s"])
        key = (run["name"], run["policy"], run["switch_penalty_s"])
        assert rep.idle_steps == run["idle_steps"], key
        assert rep.avg_throughput_ips == pytest.approx(run["avg_throughput_ips"], rel=REL_TOL, abs=0), key
        assert rep.energy_proxy_wh == pytest.approx(run["energy_proxy_wh"], rel=REL_TOL, abs=0), key
        # the double-double epilogue reproduces the exactly rounded math.fsum
        assert rep.avg_throughput_ips == run["avg_throughput_ips"], key
        assert rep.energy_proxy_wh == run["energy_proxy_wh"], key
        assert _digest(rep) == run["digest"]["sha256"], key
        if "steps" in run:
            assert [sel_doc(s.selection) for s in rep.steps] == run["steps"], key


def test_simulate_behaviour_matches_reference_tests(cs):
    """The reference's own behavioural checks (pkg/tests/test_sim.py) on the drop-in."""
    from datetime import datetime

    g1 = grid_from_doc(golden("sim_golden.json")["grids"]["g1"])
    tr = cs.PowerTrace("fixture", 3600, datetime(2020, 1, 1), (200.0, 100.0, 250.0))
    rep = cs.simulate(g1, tr, cs.COMBINATION)
    assert [s.selection.throughput_ips for s in rep.steps] == [190.0, 100.0, 300.0]
    assert cs.slice_report(rep, 0, 3) == rep
    assert cs.slice_report(rep, 0, 2).avg_throughput_ips == pytest.approx(145.0)
    pen = cs.simulate(g1, tr, cs.COMBINATION, switch_penalty_s=1800.0)
    assert pen.avg_throughput_ips == pytest.approx((190.0 + 100.0 * 0.5 + 300.0 * 0.5) / 3)
    with pytest.warns(UserWarning, match="normalize"):
        cs.simulate(g1, cs.PowerTrace("x", 3600, datetime(2020, 1, 1), (400.0, 100.0)), cs.COMBINATION)
    with pytest.raises(ValueError):
        cs.simulate(g1, tr, cs.COMBINATION, switch_penalty_s=-1.0)
    rb = cs.simulate(g1, tr, cs.BATCHING)
    table = cs.compare([rep, rb])
    assert round(next(r for r in table.rows if r.policy_a == "combination").improvement_pct) == 28
    assert cs.load_report.__module__.endswith("sim")
    loaded = cs.report_from_dict(cs.report_to_dict(rep))
    assert loaded == rep


# ---------------------------------------------------------------------------------------------
# batched engine (the benchmarked path) vs the oracle


def _random_caps(rng, T, S, kind):
    if kind == "iid":
        return (rng.random((T, S)) * 360.0).astype(np.float32)
    walk = np.cumsum(rng.normal(0, 6.0, (T, S)), axis=1) + rng.uniform(50, 300, (T, 1))
    c = np.clip(walk, 0, 350).astype(np.float32)
    c[:, ::97] = 0.0
    c[:, 5::89] = -0.0
    return c


def _engine_vs_oracle(cs, torch, grids, caps, step, pen, ld=None):
    from oracle import oracle

    T, S = caps.shape
    ld = ld or (S + 3) // 4 * 4
    host = np.zeros((T, ld), np.float32)
    host[:, :S] = caps
    tables = cs.Tables.stage(grids, "f32")
    res = tables.evaluate(torch.from_numpy(host).cuda(), S, step_seconds=step, switch_penalty_s=pen,
                          per_step=True)
    torch.cuda.synchronize()
    avg, idle, en, _ = oracle.simulate_batch([oracle_grid(g) for g in grids], caps, step, pen, n_threads=8)
    g_avg = res.avg_throughput_ips.cpu().numpy()
    g_en = res.energy_proxy_wh.cpu().numpy()
    assert np.array_equal(res.idle_steps.cpu().numpy(), idle)
    assert np.all(res.violations.cpu().numpy() == 0)
    assert np.allclose(g_avg, avg, rtol=REL_TOL, atol=0)
    assert np.allclose(g_en, en, rtol=REL_TOL, atol=0)
    exact = np.mean(g_avg == avg)
    assert exact > 0.999, f"only {exact:.4f} of averages bit-identical to fsum"
    # per-step union bins -> exact selections and global histogram
    ub = res.step_bins[:, :S].cpu().numpy().view(np.uint16).astype(np.int64)
    hist = np.bincount(ub.ravel(), minlength=tables.n_union_bins)
    assert np.array_equal(res.hist.cpu().numpy(), hist)
    for m, g in enumerate(grids):
        og = oracle_grid(g)
        gb = tables.grid_bins(m)
        for t in range(min(T, 6)):
            for p, regime in enumerate(REGIMES):
                r = oracle.simulate(og, caps[t].astype(np.float64), regime, step, pen)
                b = gb.umap[ub[t]]
                assert np.array_equal(gb.sel[p][b], r.sel), (m, t, regime)
                assert np.array_equal(gb.count[p][b], r.count), (m, t, regime)
                sw = int(np.sum(r.sel[1:] != r.sel[:-1]))
                assert int(res.switches[t, m, p]) == (sw if pen > 0 else 0)
    return res


@pytest.mark.parametrize("kind", ["smooth", "iid"])
@pytest.mark.parametrize("pen", [0.0, 10.0])
def test_engine_single_grid_vs_oracle(cs, torch, kind, pen):
    rng = np.random.default_rng(11)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128, model_name="mobilenet-v1"))
    _engine_vs_oracle(cs, torch, [g], _random_caps(rng, 37, 1441, kind), 60, pen)


def test_engine_bin_epilogue_vs_oracle_and_segments(cs, torch):
    """>= 4M timesteps on one grid without a penalty take the per-bin epilogue (bench path, with
    and without per-step output); it must match the oracle and the segment epilogue."""
    rng = np.random.default_rng(21)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128, model_name="mobilenet-v1"))
    caps = np.concatenate([_random_caps(rng, 300, 10080, "smooth"), _random_caps(rng, 120, 10080, "iid")])
    res = _engine_vs_oracle(cs, torch, [g], caps, 60, 0.0)  # per-step variant
    host = torch.from_numpy(np.ascontiguousarray(caps, np.float32)).cuda()
    tables = cs.Tables.stage([g], "f32")
    fast = tables.evaluate(host, 10080, step_seconds=60)
    seg = tables.evaluate(host, 10080, step_seconds=60, segment_epilogue=True)
    torch.cuda.synchronize()
    for r in (fast, seg):
        assert np.array_equal(r.idle_steps.cpu().numpy(), res.idle_steps.cpu().numpy())
        assert np.array_equal(r.hist.cpu().numpy(), res.hist.cpu().numpy())
        assert np.allclose(r.avg_throughput_ips.cpu().numpy(), res.avg_throughput_ips.cpu().numpy(), rtol=1e-12,
                           atol=0)
        assert np.allclose(r.energy_proxy_wh.cpu().numpy(), res.energy_proxy_wh.cpu().numpy(), rtol=1e-12, atol=0)
    same = np.mean(fast.avg_throughput_ips.cpu().numpy() == seg.avg_throughput_ips.cpu().numpy())
    assert same > 0.999


def test_engine_multi_grid_vs_oracle(cs, torch):
    rng = np.random.default_rng(12)
    grids = [cs.synthesize_grid(cs.SynthParams(t_max_ips=float(rng.uniform(1000, 20000)), tau=float(rng.uniform(8, 128)),
                                               contention=float(rng.uniform(0.7, 1.0)),
                                               gamma=float(rng.uniform(0.5, 1.5)),
                                               p_idle_w=float(rng.uniform(30, 100)), seed=i, noise_pct=1.0,
                                               model_name=f"cnn{i}"))
             for i in range(10)]
    _engine_vs_oracle(cs, torch, grids, _random_caps(rng, 9, 3000, "smooth"), 1, 0.0)
    _engine_vs_oracle(cs, torch, grids[:3], _random_caps(rng, 5, 999, "iid"), 60, 30.0)


def test_engine_split_trace_and_fine_grid(cs, torch):
    """Few long traces take the split-segment path (partials + finalize kernel)."""
    rng = np.random.default_rng(13)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    _engine_vs_oracle(cs, torch, [g], _random_caps(rng, 1, 300_001, "smooth"), 60, 10.0)
    _engine_vs_oracle(cs, torch, [g], _random_caps(rng, 3, 70_000, "iid"), 60, 0.0)


@pytest.mark.parametrize("T,S", [(3000, 300), (4100, 1024)])
def test_fine_grid_multiwarp_groups_many_traces(cs, torch, T, S):
    """Fine 8x512 grid (2,038 bins -> multi-warp worker groups) with several traces per group, so a
    group's warp 0 is still writing trace t's records while its other warps run trace t+1; both
    sizes (plain, and >= 4M timesteps with staged tables) with and without a switching penalty,
    through the bench's kernel (no per-step output): aggregates vs the oracle, switch counts vs
    the selections of a per-step run."""
    from oracle import oracle

    rng = np.random.default_rng(21)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    caps = _random_caps(rng, T, S, "smooth")
    ld = (S + 3) // 4 * 4
    host = np.zeros((T, ld), np.float32)
    host[:, :S] = caps
    dev = torch.from_numpy(host).cuda()
    t = cs.Tables.stage([g], "f32")
    gb = t.grid_bins(0)
    for pen in (0.0, 10.0):
        res = t.evaluate(dev, S, step_seconds=60, switch_penalty_s=pen)
        plan = t.last_plan()
        assert plan["warps_per_group"] > 1 and T > 2 * plan["ctas"] * plan["threads"] // 32 // plan["warps_per_group"]
        avg, idle, en, _ = oracle.simulate_batch([oracle_grid(g)], caps, 60, pen, n_threads=8)
        assert np.array_equal(res.idle_steps.cpu().numpy(), idle)
        assert np.all(res.violations.cpu().numpy() == 0)
        g_avg, g_en = res.avg_throughput_ips.cpu().numpy(), res.energy_proxy_wh.cpu().numpy()
        assert np.allclose(g_avg, avg, rtol=REL_TOL, atol=0) and np.allclose(g_en, en, rtol=REL_TOL, atol=0)
        assert np.mean(g_avg == avg) > 0.999
        ps = t.evaluate(dev, S, step_seconds=60, switch_penalty_s=pen, per_step=True)
        ub = ps.step_bins[:, :S].cpu().numpy().view(np.uint16).astype(np.int64)
        assert np.array_equal(res.hist.cpu().numpy(), np.bincount(ub.ravel(), minlength=t.n_union_bins))
        for p in range(3):
            sel = gb.sel[p][gb.umap[ub]]
            want = np.sum(sel[:, 1:] != sel[:, :-1], axis=1) if pen > 0 else np.zeros(T, np.int64)
            assert np.array_equal(res.switches[:, 0, p].cpu().numpy().astype(np.int64), want), p


def test_fp64_penalty_path_matches_fp32(cs, torch):
    """fp64 caps (the drop-in PowerTrace path) through the penalty loop with multi-warp worker
    groups (fine grid): on f32-representable caps every selection equals the fp32 path's, so
    idle and switch counts are identical and the exact sums agree."""
    rng = np.random.default_rng(22)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    T, S = 1500, 2000
    caps = _random_caps(rng, T, S, "smooth")
    dev32 = torch.from_numpy(caps).cuda()
    t32, t64 = cs.Tables.stage([g], "f32"), cs.Tables.stage([g], "f64")
    for pen in (10.0, 0.0):
        r32 = t32.evaluate(dev32, S, step_seconds=60, switch_penalty_s=pen)
        r64 = t64.evaluate(dev32.double(), S, step_seconds=60, switch_penalty_s=pen)
        assert t64.last_plan()["warps_per_group"] > 1
        assert torch.equal(r32.switches.cpu(), r64.switches.cpu())
        assert torch.equal(r32.idle_steps.cpu(), r64.idle_steps.cpu())
        assert int(r64.violations.sum()) == 0
        for a, b in ((r32.avg_throughput_ips, r64.avg_throughput_ips), (r32.energy_proxy_wh, r64.energy_proxy_wh)):
            a, b = a.cpu().numpy(), b.cpu().numpy()
            assert np.allclose(a, b, rtol=1e-12, atol=0)
        if pen > 0:
            assert int(r64.switches.sum()) > T


def test_engine_random_and_tie_grids(cs, torch):
    doc = golden("policy_golden.json")
    rng = np.random.default_rng(14)
    grids = [grid_from_doc(c["grid"]) for c in doc["cases"] if c["name"].startswith("rand")][:12]
    for g in grids[:6]:
        _engine_vs_oracle(cs, torch, [g], _random_caps(rng, 4, 333, "iid"), 3600, 900.0)
    _engine_vs_oracle(cs, torch, grids[6:], _random_caps(rng, 4, 500, "smooth"), 60, 0.0)


def test_generator_is_shard_invariant(cs, torch):
    a = cs.generate_traces(64, 1000, step_seconds=60, kind="mixed", seed=7)
    b = cs.generate_traces(32, 1000, step_seconds=60, kind="mixed", seed=7, first_trace_id=32)
    torch.cuda.synchronize()
    assert torch.equal(a[32:], b)
    assert float(a.min()) >= 0.0 and float(a.max()) <= 350.0
    assert float(a.std()) > 10.0


@pytest.mark.parametrize("kind", ["solar", "wind", "mixed", "iid"])
@pytest.mark.parametrize("step", [1, 60])
def test_generator_matches_host_port(cs, torch, kind, step):
    """The device generator and its host port (oracle.generate_traces) agree bit for bit, so the
    bench's reference arm and CPU baseline run the reference algorithm on the same caps."""
    from oracle import oracle

    T, S = 70, 9001  # partial warps, three time chunks
    dev = cs.generate_traces(T, S, step_seconds=step, kind=kind, seed=2306, first_trace_id=5)
    host = oracle.generate_traces(T, S, step_seconds=step, kind=kind, seed=2306, first_trace_id=5)
    torch.cuda.synchronize()
    d = dev.cpu().numpy()
    assert d.shape == host.shape
    assert np.array_equal(d.view(np.uint32), host.view(np.uint32))


def test_host_engine_matches_device_path(cs, torch):
    rng = np.random.default_rng(15)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
    caps = _random_caps(rng, 50, 2000, "smooth")
    host = torch.from_numpy(caps).pin_memory()
    t = cs.Tables.stage([g], "f32")
    dev = t.evaluate(host.cuda(), 2000, step_seconds=60)
    eng = cs.HostEngine(t, chunk_traces=16, n_steps_max=2000)
    agg, hist, h2d, d2h = eng.evaluate(host, 2000, step_seconds=60)
    torch.cuda.synchronize()
    assert torch.equal(agg, dev.agg.cpu())
    assert torch.equal(hist, dev.hist.cpu())
    assert h2d == caps.nbytes
    assert d2h == agg.numel() * 8 + hist.numel() * 8


def test_engine_special_caps_match_host_lookup(cs, torch):
    """-0.0, denormals, +inf, NaN and huge caps through the device LUT == host restatement ==
    bisect_right semantics (NaN and +inf bisect to the top, policy.py:139)."""
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    special = np.array([-0.0, 0.0, 1e-45, 1e-38, 59.99, 60.0, 349.9999, 350.0, 350.0001, 3e38,
                        np.inf, np.nan], np.float32)
    rng = np.random.default_rng(5)
    pws = np.array(g.columns()[4], np.float64)
    near = np.concatenate([pws.astype(np.float32), np.nextafter(pws.astype(np.float32), np.float32(0))])
    caps = np.concatenate([special, near, rng.uniform(0, 360, 4000).astype(np.float32)])
    S = caps.shape[0]
    host = np.zeros((1, (S + 3) // 4 * 4), np.float32)
    host[0, :S] = caps
    t = cs.Tables.stage([g], "f32")
    res = t.evaluate(torch.from_numpy(host).cuda(), S, step_seconds=60, per_step=True)
    dev_bins = res.bins_numpy(0)
    assert np.array_equal(dev_bins, t.lookup_host(caps))
    top = t.n_union_bins - 1
    assert dev_bins[0] == 0 and dev_bins[1] == 0 and dev_bins[10] == top and dev_bins[11] == top
    assert int(res.violations.sum()) == 0


@pytest.mark.parametrize("pen", [0.0, 30.0])
def test_graph_replay_matches_evaluate(cs, torch, pen):
    """Tables.capture: a CUDA-graph replay reads the caps buffer at replay time and reproduces
    evaluate() exactly (tiny single-trace plan and split-trace finalize path)."""
    rng = np.random.default_rng(31)
    grids = [cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128, model_name="mobilenet-v1")),
             cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=64, t_max_ips=4000.0, model_name="b"))]
    for T, S in ((1, 1440), (2, 200_000)):
        caps = torch.from_numpy(np.ascontiguousarray(_random_caps(rng, T, S, "smooth"), np.float32)).cuda()
        tables = cs.Tables.stage(grids, "f32")
        g = tables.capture(caps, S, step_seconds=60, switch_penalty_s=pen)
        for _ in range(2):
            r = g.replay()
            torch.cuda.synchronize()
            ref = tables.evaluate(caps, S, step_seconds=60, switch_penalty_s=pen)
            torch.cuda.synchronize()
            assert torch.equal(r.agg, ref.agg) and torch.equal(r.hist, ref.hist)
            caps.mul_(0.75)  # new data in place: the next replay must see it


def test_back_to_back_replays_rearm_item_counter(cs, torch):
    """Traces beyond the first round are handed out from a workspace counter that the last worker
    group of each launch re-arms (graph replays skip the kernel that zeroes it): back-to-back
    replays with more traces than worker groups must each evaluate every trace exactly once."""
    rng = np.random.default_rng(37)
    grid = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128, model_name="mobilenet-v1"))
    T, S = 20_000, 1000  # >> 148 CTAs x 32 one-warp groups
    caps = torch.from_numpy(np.ascontiguousarray(_random_caps(rng, T, S, "smooth"), np.float32)).cuda()
    tables = cs.Tables.stage([grid], "f32")
    ref = tables.evaluate(caps, S, step_seconds=60)
    torch.cuda.synchronize()
    g = tables.capture(caps, S, step_seconds=60)
    for _ in range(4):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(g.result.agg, ref.agg) and torch.equal(g.result.hist, ref.hist)
    assert int(g.result.hist.sum()) == T * S
