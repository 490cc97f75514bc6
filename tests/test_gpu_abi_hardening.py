"""C-ABI hardening: padded / strided host matrices, engines reused
with more grids, zero-trace launches and bad arguments. Results must equal the device path
(which the parity tests pin to the oracle); bad calls must fail with an error, never write out
of bounds (tools/sanitize_small.py runs this file under compute-sanitizer memcheck)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch(cuda_ok):
    import torch as T

    return T


@pytest.fixture(scope="module")
def cs(cuda_ok):
    import paper_2306_12247_b200 as m

    return m


def _grids(cs, n):
    return [cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=32, t_max_ips=2000.0 + 500 * i, seed=i,
                                              noise_pct=1.0, model_name=f"g{i}")) for i in range(n)]


def _caps(T, S, seed=3):
    rng = np.random.default_rng(seed)
    return np.clip(np.cumsum(rng.normal(0, 9, (T, S)), axis=1) + 170, 0, 350).astype(np.float32)


def test_engine_accepts_padded_host_rows(cs, torch):
    """ld (host pitch) wider than the engine's device pitch: rows are copied 2-D into the pitch."""
    T, S = 37, 1000
    caps = _caps(T, S)
    wide = torch.zeros((T, S + 77), dtype=torch.float32).pin_memory()  # ld = 1077: not even a multiple of 4
    wide[:, :S] = torch.from_numpy(caps)
    t = cs.Tables.stage(_grids(cs, 1), "f32")
    ref = t.evaluate(torch.from_numpy(caps).cuda(), S, step_seconds=60)
    eng = cs.HostEngine(t, chunk_traces=8, n_steps_max=S)
    agg, hist, h2d, _ = eng.evaluate(wide[:, :S], S, step_seconds=60)
    torch.cuda.synchronize()
    assert torch.equal(agg, ref.agg.cpu()) and torch.equal(hist, ref.hist.cpu())
    assert h2d == T * S * 4  # only the samples travel
    agg2, _, _, _ = eng.evaluate(wide, S, step_seconds=60)  # n_steps < row length, pitch = 1077
    assert torch.equal(agg2, ref.agg.cpu())


def test_engine_grows_for_more_grids(cs, torch):
    """One engine, a one-grid call then a ten-grid call: the aggregate buffers grow."""
    T, S = 20, 800
    caps = torch.from_numpy(_caps(T, S, 4)).pin_memory()
    t1, t10 = cs.Tables.stage(_grids(cs, 1), "f32"), cs.Tables.stage(_grids(cs, 10), "f32")
    eng = cs.HostEngine(t1, chunk_traces=6, n_steps_max=S)
    a1, _, _, _ = eng.evaluate(caps, S, step_seconds=60)
    eng.tables = t10
    a10, h10, _, _ = eng.evaluate(caps, S, step_seconds=60, switch_penalty_s=5.0)
    ref = t10.evaluate(caps.cuda(), S, step_seconds=60, switch_penalty_s=5.0)
    torch.cuda.synchronize()
    assert torch.equal(a10, ref.agg.cpu()) and torch.equal(h10, ref.hist.cpu())
    assert torch.equal(a1, t1.evaluate(caps.cuda(), S, step_seconds=60).agg.cpu())


def test_engine_rejects_bad_arguments(cs, torch):
    from paper_2306_12247_b200 import _native as N

    t = cs.Tables.stage(_grids(cs, 1), "f32")
    eng = cs.HostEngine(t, chunk_traces=4, n_steps_max=100)
    with pytest.raises(ValueError):
        eng.evaluate(torch.zeros((3, 100), dtype=torch.float64), 100, step_seconds=60)  # dtype of the tables
    with pytest.raises(ValueError):
        eng.evaluate(torch.zeros((3, 100), dtype=torch.float32).t().contiguous().t(), 100, step_seconds=60)
    with pytest.raises(ValueError):
        eng.evaluate(torch.zeros((3, 100), dtype=torch.float32), 101, step_seconds=60)
    host = np.zeros((3, 200), np.float32)
    agg = np.zeros((3, 1, 3, 6))
    h2d, d2h = C.c_int64(), C.c_int64()
    # n_steps beyond the engine's allocation, and ld < n_steps, straight through the C ABI
    for n_steps, ld in ((200, 200), (100, 50)):
        rc = N.lib().cs_engine_eval_host(eng._h, t.handle, host.ctypes.data, 3, n_steps, ld, 60, 0.0, 0,
                                         agg.ctypes.data, None, C.byref(h2d), C.byref(d2h))
        assert rc == N.CS_E_INVALID, (n_steps, ld)


def test_zero_trace_launch_zeroes_histogram(cs, torch):
    """A rank that owns no traces must contribute an all-zero histogram to the reduction."""
    t = cs.Tables.stage(_grids(cs, 2), "f32")
    hist = torch.full((t.n_union_bins,), 12345, dtype=torch.int64, device="cuda")
    empty = torch.zeros((0, 128), dtype=torch.float32, device="cuda")
    r = t.evaluate(empty, 100, step_seconds=60)
    torch.cuda.synchronize()
    assert r.agg.shape[0] == 0 and int(r.hist.abs().sum()) == 0
    t.evaluate(empty, 100, step_seconds=60, accumulate_hist=hist)  # accumulate: untouched
    torch.cuda.synchronize()
    assert int(hist.min()) == 12345


def test_tiny_plan_with_many_grids(cs, torch):
    """A short single trace over > 170 grids needs 1024-thread CTAs (3M + 1 per-group counters):
    the small-CTA preference must not make the plan fail."""
    from oracle import oracle

    import bench

    grids = [cs.synthesize_grid(cs.SynthParams(mtl_cap=1, bs_cap=2, t_max_ips=1000.0 + 37 * i, p_idle_w=40.0 + i % 50,
                                               model_name=f"m{i}")) for i in range(200)]
    caps = _caps(1, 1440, 9)
    t = cs.Tables.stage(grids, "f32")
    res = t.evaluate(torch.from_numpy(caps).cuda(), 1440, step_seconds=60, per_step=True)
    torch.cuda.synchronize()
    assert t.last_plan()["threads"] == 1024
    avg, idle, en, _ = oracle.simulate_batch(bench.oracle_grids(grids), caps, 60, 0.0)
    assert np.array_equal(res.idle_steps.cpu().numpy(), idle)
    assert np.allclose(res.avg_throughput_ips.cpu().numpy(), avg, rtol=1e-6, atol=0)
