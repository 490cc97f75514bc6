"""GPU parity on the exact launch plans the benchmark runs (VERDICT r1 "parity holes").

* C3's plan: the ten bench grids (5,000+ union thresholds), >= 4M timesteps, no per-step output,
  enough traces that no trace is split -> the large-launch plan (finer LUT and segment tables
  staged when they fit), multi-warp worker groups; with week-long traces the huge LUT and
  histograms folded straight into global memory.
* C2's plan: the ten grids over one or two long traces -> traces split across worker groups,
  partial histograms and the per-(trace, grid) finalize kernel (gridDim.y = M).

Each is compared with the pinned CPU oracle (oracle.simulate_batch / oracle.simulate, restating
sim.py:104-188 and policy.py:136-148) on the bench's own generator output: idle counts,
histograms and switch counts exact; sums within 1e-6 and >= 99.9 % bit-identical to fsum.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import REGIMES

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6


@pytest.fixture(scope="module")
def torch(cuda_ok):
    import torch as T

    return T


@pytest.fixture(scope="module")
def cs(cuda_ok):
    import paper_2306_12247_b200 as m

    return m


@pytest.fixture(scope="module")
def ten(cs):
    import bench

    return bench.make_grids("ten")


def _oracle_grids(grids):
    import bench

    return bench.oracle_grids(grids)


def _check_aggs(res, caps_np, grids, step, pen):
    from oracle import oracle

    avg, idle, en, _ = oracle.simulate_batch(_oracle_grids(grids), caps_np, step, pen, n_threads=16)
    g_avg = res.avg_throughput_ips.cpu().numpy()
    g_en = res.energy_proxy_wh.cpu().numpy()
    assert np.array_equal(res.idle_steps.cpu().numpy(), idle)
    assert np.all(res.violations.cpu().numpy() == 0)
    assert np.allclose(g_avg, avg, rtol=REL_TOL, atol=0)
    assert np.allclose(g_en, en, rtol=REL_TOL, atol=0)
    exact = min(np.mean(g_avg == avg), np.mean(g_en == en))
    assert exact > 0.999, f"only {exact:.4f} of sums bit-identical to fsum"


def _check_switches(res, caps_np, grids, step, pen, traces):
    from oracle import oracle

    og = _oracle_grids(grids)
    for t in traces:
        for m in range(len(grids)):
            for p, regime in enumerate(REGIMES):
                r = oracle.simulate(og[m], caps_np[t].astype(np.float64), regime, step, pen)
                want = int(np.sum(r.sel[1:] != r.sel[:-1])) if pen > 0 else 0
                assert int(res.switches[t, m, p]) == want, (t, m, regime)


def _check_hist_and_switches(res, tables, caps, S, step, pen):
    """Histogram and switch counts of ``res`` against a per-step run (bins do not depend on the
    penalty; with a penalty the ten grids' per-step launch would not fit shared memory)."""
    ps = tables.evaluate(caps, S, step_seconds=step, per_step=True)
    ub = ps.step_bins[:, :S].cpu().numpy().view(np.uint16).astype(np.int64)
    hist = np.bincount(ub.ravel(), minlength=tables.n_union_bins)
    if res.hist is not None:
        assert np.array_equal(res.hist.cpu().numpy(), hist)
    else:  # grids evaluated in chunks: per-grid config histograms
        assert res.config_histograms() == tables.config_histograms(hist)
    sw = res.switches.cpu().numpy()
    for m in range(tables.n_grids):
        gb = tables.grid_bins(m)
        for p in range(3):
            sel = gb.sel[p][gb.umap[ub]]
            want = np.sum(sel[:, 1:] != sel[:, :-1], axis=1) if pen > 0 else np.zeros(sel.shape[0], np.int64)
            assert np.array_equal(sw[:, m, p], want), (m, p)


@pytest.mark.parametrize("kind", ["mixed", "iid"])
@pytest.mark.parametrize("pen", [0.0, 10.0])
def test_c3_plan_ten_grids_staged(cs, torch, ten, kind, pen):
    T, S, step = 1536, 4096, 1  # 6.3M timesteps: the large-launch plan, one worker group per trace
    caps = cs.generate_traces(T, S, step_seconds=step, kind=kind, seed=2306)
    torch.cuda.synchronize()
    caps_np = caps[:, :S].cpu().numpy()
    tables = cs.Tables.stage(ten, "f32")
    res = tables.evaluate(caps, S, step_seconds=step, switch_penalty_s=pen, check_violations=True)
    torch.cuda.synchronize()
    plan = tables.last_plan()
    assert plan["trace_segments"] == 1, plan
    assert plan["warps_per_group"] > 1, plan
    _check_aggs(res, caps_np, ten, step, pen)
    _check_hist_and_switches(res, tables, caps, S, step, pen)
    _check_switches(res, caps_np, ten, step, pen, traces=(0, 1, T - 1))


@pytest.mark.parametrize("kind", ["mixed", "iid"])
def test_c3_plan_long_traces_huge_lut_direct_histogram(cs, torch, ten, kind):
    """C3's own plan: week-long 1-s traces (>= 64 steps per union bin) fold each trace's histogram
    straight into global memory, which makes room for the shift-11 'huge' LUT next to 8-warp
    groups, whole traces per group (>= 2 traces per group). Aggregates of a sample
    of traces against the oracle; the global histogram against a per-step run of every trace."""
    T, S, step = 1184, 5056 * 64, 1  # 3.8e8 timesteps
    caps = cs.generate_traces(T, S, step_seconds=step, kind=kind, seed=2306)
    torch.cuda.synchronize()
    tables = cs.Tables.stage(ten, "f32")
    res = tables.evaluate(caps, S, step_seconds=step, check_violations=True)
    torch.cuda.synchronize()
    plan = tables.last_plan()
    assert plan["lut_shift"] == tables.info.lut_huge_shift and plan["warps_per_group"] == 8, plan
    assert plan["trace_segments"] == 1, plan
    from oracle import oracle

    pick = [0, 1, 2, 591, 592, 1000, T - 2, T - 1]
    avg, idle, en, _ = oracle.simulate_batch(_oracle_grids(ten), caps[pick, :S].cpu().numpy(), step, 0.0,
                                             n_threads=16)
    assert np.array_equal(res.idle_steps[pick].cpu().numpy(), idle)
    assert np.allclose(res.avg_throughput_ips[pick].cpu().numpy(), avg, rtol=REL_TOL, atol=0)
    assert np.allclose(res.energy_proxy_wh[pick].cpu().numpy(), en, rtol=REL_TOL, atol=0)
    assert int(res.violations.sum()) == 0
    ps = tables.evaluate(caps, S, step_seconds=step, per_step=True)
    hist = np.zeros(tables.n_union_bins, np.int64)
    for a in range(0, T, 128):  # bincount in slices (4e8 bins)
        ub = ps.step_bins[a:a + 128, :S].cpu().numpy().view(np.uint16).astype(np.int64)
        hist += np.bincount(ub.ravel(), minlength=tables.n_union_bins)
    assert np.array_equal(res.hist.cpu().numpy(), hist)


def test_long_traces_penalty_direct_histogram(cs, torch, ten):
    """Several grids with a switching penalty over long traces: the segment epilogue with switch
    counters, warp-owned (grid, policy) pairs and each trace's histogram folded straight into
    global memory (>= 64 steps per union bin). Sampled traces against the oracle (aggregates and
    switch counts); the global histogram against a per-step run."""
    from oracle import oracle

    grids = ten[:3]
    tables = cs.Tables.stage(grids, "f32")
    U = tables.n_union_bins
    T, S, step, pen = 1184, ((U * 64 + 127) // 128) * 128, 1, 10.0
    caps = cs.generate_traces(T, S, step_seconds=step, kind="mixed", seed=7)
    torch.cuda.synchronize()
    res = tables.evaluate(caps, S, step_seconds=step, switch_penalty_s=pen, check_violations=True)
    torch.cuda.synchronize()
    plan = tables.last_plan()
    assert plan["trace_segments"] == 1 and plan["epilogue"] in (0, 1), plan
    pick = [0, 1, 500, T - 1]
    caps_np = caps[pick, :S].cpu().numpy()
    og = _oracle_grids(grids)
    avg, idle, en, _ = oracle.simulate_batch(og, caps_np, step, pen, n_threads=16)
    assert np.array_equal(res.idle_steps[pick].cpu().numpy(), idle)
    assert np.allclose(res.avg_throughput_ips[pick].cpu().numpy(), avg, rtol=REL_TOL, atol=0)
    assert np.allclose(res.energy_proxy_wh[pick].cpu().numpy(), en, rtol=REL_TOL, atol=0)
    for i, t in enumerate(pick[:2]):
        for m in range(len(grids)):
            for p, regime in enumerate(REGIMES):
                r = oracle.simulate(og[m], caps_np[i].astype(np.float64), regime, step, pen)
                assert int(res.switches[t, m, p]) == int(np.sum(r.sel[1:] != r.sel[:-1])), (t, m, regime)
    ps = tables.evaluate(caps, S, step_seconds=step, per_step=True)
    hist = np.zeros(U, np.int64)
    for a in range(0, T, 256):
        ub = ps.step_bins[a:a + 256, :S].cpu().numpy().view(np.uint16).astype(np.int64)
        hist += np.bincount(ub.ravel(), minlength=U)
    assert np.array_equal(res.hist.cpu().numpy(), hist)


@pytest.mark.parametrize("pen", [0.0, 10.0])
@pytest.mark.parametrize("T", [1, 2])
def test_c2_plan_split_trace_finalize(cs, torch, ten, pen, T):
    S, step = 300_007, 60  # one or two long traces: split across worker groups + per-grid finalize
    caps = cs.generate_traces(T, S, step_seconds=step, kind="mixed", seed=2306)
    torch.cuda.synchronize()
    caps_np = caps[:, :S].cpu().numpy()
    tables = cs.Tables.stage(ten, "f32")
    res = tables.evaluate(caps, S, step_seconds=step, switch_penalty_s=pen)
    torch.cuda.synchronize()
    plan = tables.last_plan()
    assert plan["trace_segments"] > 1, plan
    assert tables.launch_count() == 3  # prep, eval, finalize (of the last grid chunk, if chunked)
    _check_aggs(res, caps_np, ten, step, pen)
    _check_hist_and_switches(res, tables, caps, S, step, pen)
    _check_switches(res, caps_np, ten, step, pen, traces=range(T))
    # the captured graph (what the bench replays) reproduces it
    g = tables.capture(caps, S, step_seconds=step, switch_penalty_s=pen)
    r = g.replay()
    torch.cuda.synchronize()
    assert torch.equal(r.agg, res.agg)
    assert r.config_histograms() == res.config_histograms()


def test_c4_plan_bin_epilogue_on_bench_traces(cs, torch):
    """C4's plan (one grid, per-bin epilogue, staged finer LUT) on the bench generator's traces."""
    import bench

    grids = bench.make_grids("mobilenet")
    T, S = 10_000, 10080  # > 2 x (148 SMs x 32 one-warp groups): whole traces per group, as at C4
    caps = cs.generate_traces(T, S, step_seconds=60, kind="mixed", seed=2306)
    torch.cuda.synchronize()
    tables = cs.Tables.stage(grids, "f32")
    res = tables.evaluate(caps, S, step_seconds=60)
    torch.cuda.synchronize()
    plan = tables.last_plan()
    assert plan["epilogue"] == 2 and plan["trace_segments"] == 1, plan
    _check_aggs(res, caps[:, :S].cpu().numpy(), grids, 60, 0.0)
    _check_hist_and_switches(res, tables, caps, S, 60, 0.0)


@pytest.mark.parametrize("kind", ["mixed", "iid"])
@pytest.mark.parametrize("pen", [10.0, 60.0, 7.5])
def test_c5_plan_packed_penalty(cs, torch, kind, pen):
    """C5's plan: the fine 8x512 grid with a switching penalty -> the packed-penalty kernel (PK:
    16|16-bit step / switched-step counters, policy 1's delta in registers, per-touched-bin
    epilogue). Against the oracle and against the segment-counter path (segment_epilogue=True)."""
    import bench

    grids = bench.make_grids("fine")
    T, S, step = 2400, 10080, 60  # 24.2M timesteps: whole traces per worker group (>= 2 per group)
    caps = cs.generate_traces(T, S, step_seconds=step, kind=kind, seed=2306)
    torch.cuda.synchronize()
    caps_np = caps[:, :S].cpu().numpy()
    tables = cs.Tables.stage(grids, "f32")
    res = tables.evaluate(caps, S, step_seconds=step, switch_penalty_s=pen, check_violations=True)
    torch.cuda.synchronize()
    plan = tables.last_plan()
    assert plan["epilogue"] in (3, 4) and plan["trace_segments"] == 1, plan
    _check_aggs(res, caps_np, grids, step, pen)
    _check_hist_and_switches(res, tables, caps, S, step, pen)
    _check_switches(res, caps_np, grids, step, pen, traces=(0, 1, 7, T - 1))
    old = tables.evaluate(caps, S, step_seconds=step, switch_penalty_s=pen, check_violations=True,
                          segment_epilogue=True)
    torch.cuda.synchronize()
    assert tables.last_plan()["epilogue"] in (0, 1)
    for f in ("idle_steps", "switches", "violations"):
        assert torch.equal(getattr(res, f), getattr(old, f)), f
    assert torch.equal(res.hist, old.hist)
    assert torch.allclose(res.avg_throughput_ips, old.avg_throughput_ips, rtol=1e-12, atol=0)
    assert torch.allclose(res.energy_proxy_wh, old.energy_proxy_wh, rtol=1e-12, atol=0)


@pytest.mark.parametrize("kind", ["iid", "mixed"])
def test_pk_short_traces_and_tails(cs, torch, kind):
    """PK with ragged lengths (tails of < 4 caps, last blocks partly filled with the last cap,
    whole blocks only: 1280 steps), a trace of one step, and the plan falling back when a trace
    would be split (few traces)."""
    import bench
    from oracle import oracle

    grids = bench.make_grids("fine")
    og = bench.oracle_grids(grids)
    tables = cs.Tables.stage(grids, "f32")
    for T, S in ((4800, 1023), (4800, 5), (4800, 1), (4800, 1280), (4800, 2305), (3, 9000)):
        caps = cs.generate_traces(T, S, step_seconds=60, kind=kind, seed=11)
        torch.cuda.synchronize()
        res = tables.evaluate(caps, S, step_seconds=60, switch_penalty_s=10.0)
        torch.cuda.synchronize()
        caps_np = caps[:, :S].cpu().numpy()
        avg, idle, en, _ = oracle.simulate_batch(og, caps_np, 60, 10.0, n_threads=16)
        assert np.array_equal(res.idle_steps.cpu().numpy(), idle), (T, S)
        assert np.allclose(res.avg_throughput_ips.cpu().numpy(), avg, rtol=REL_TOL, atol=0), (T, S)
        assert np.allclose(res.energy_proxy_wh.cpu().numpy(), en, rtol=REL_TOL, atol=0), (T, S)
        for t in (0, T - 1):
            for p, regime in enumerate(REGIMES):
                r = oracle.simulate(og[0], caps_np[t].astype(np.float64), regime, 60, 10.0)
                assert int(res.switches[t, 0, p]) == int(np.sum(r.sel[1:] != r.sel[:-1])), (T, S, t, regime)
