"""GPU edge cases of the batched engine against the oracle: ragged and tiny trace lengths (the
vector loop's tails), padded rows, all-idle and above-every-threshold traces, a penalty at and
beyond the step length (sim.py:111: full loss), large step lengths, and a 24-grid union (many
thousand union bins: the plan's shared-memory limits and multi-level LUT)."""

from __future__ import annotations

import numpy as np
import pytest

from test_gpu_parity import _engine_vs_oracle, _random_caps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(cuda_ok):
    import torch

    import paper_2306_12247_b200 as cs

    return cs, torch


@pytest.mark.parametrize("S", [1, 2, 3, 4, 5, 7, 127, 129, 513, 4099])
def test_ragged_lengths(env, S):
    cs, torch = env
    rng = np.random.default_rng(S)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
    _engine_vs_oracle(cs, torch, [g], _random_caps(rng, 5, S, "smooth"), 60, 0.0)
    _engine_vs_oracle(cs, torch, [g], _random_caps(rng, 3, S, "iid"), 60, 20.0, ld=(S + 3) // 4 * 4 + 8)


def test_idle_and_saturated_traces(env):
    cs, torch = env
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=32, p_idle_w=80.0))
    S = 1000
    caps = np.zeros((4, S), np.float32)
    caps[1] = 1e6                      # above every threshold: the global best every step
    caps[2] = np.float32(79.999)       # just below the lowest power: idle
    caps[3, ::2] = 350.0               # alternating idle / best: a switch every step
    for pen in (0.0, 30.0, 60.0, 600.0):   # pf = 0, 1/2, 1 (full loss), clamped to 1
        _engine_vs_oracle(cs, torch, [g], caps, 60, pen)


@pytest.mark.parametrize("step", [1, 3600, 86400])
def test_step_lengths(env, step):
    cs, torch = env
    rng = np.random.default_rng(step)
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=3, bs_cap=64))
    _engine_vs_oracle(cs, torch, [g], _random_caps(rng, 4, 777, "smooth"), step, step / 3.0)


def test_large_union(env):
    """24 noisy grids: the merged tables exceed shared memory, so evaluate() runs grid chunks;
    aggregates and per-grid config histograms still match the oracle exactly."""
    from oracle import oracle
    from test_gpu_parity import oracle_grid

    cs, torch = env
    rng = np.random.default_rng(24)
    grids = [cs.synthesize_grid(cs.SynthParams(t_max_ips=float(rng.uniform(1000, 20000)), tau=float(rng.uniform(8, 128)),
                                               contention=float(rng.uniform(0.7, 1.0)),
                                               gamma=float(rng.uniform(0.5, 1.5)), p_idle_w=float(rng.uniform(30, 100)),
                                               mtl_cap=4, bs_cap=128, seed=i, noise_pct=2.0, model_name=f"g{i}"))
             for i in range(24)]
    tables = cs.Tables.stage(grids, "f32")
    assert tables.n_union_bins > 8000
    for pen, kind, T, S in ((0.0, "smooth", 5, 2000), (15.0, "iid", 3, 1500)):
        caps = _random_caps(rng, T, S, kind)
        host = np.zeros((T, (S + 3) // 4 * 4), np.float32)
        host[:, :S] = caps
        res = tables.evaluate(torch.from_numpy(host).cuda(), S, step_seconds=60, switch_penalty_s=pen)
        torch.cuda.synchronize()
        assert res.parts is not None and len(res.parts) >= 2  # chunked
        avg, idle, en, _ = oracle.simulate_batch([oracle_grid(g) for g in grids], caps, 60, pen, n_threads=8)
        assert np.array_equal(res.idle_steps.cpu().numpy(), idle)
        assert np.allclose(res.avg_throughput_ips.cpu().numpy(), avg, rtol=1e-6, atol=0)
        assert np.allclose(res.energy_proxy_wh.cpu().numpy(), en, rtol=1e-6, atol=0)
        assert int(res.violations.sum()) == 0
        hists = res.config_histograms()
        for m in (0, 7, 23):
            cfgs = grids[m].columns()[0]
            for p, regime in enumerate(("batching", "multi-tenant", "combination")):
                want: dict = {}
                for t in range(T):
                    for sidx in oracle.simulate(oracle_grid(grids[m]), caps[t].astype(np.float64), regime, 60,
                                                pen).sel:
                        key = None if sidx < 0 else cfgs[sidx]
                        want[key] = want.get(key, 0) + 1
                assert hists[m][p] == want, (m, regime)
