"""Pins the CPU oracle (oracle/capsim_oracle.c) to the reference's own outputs.

The golden vectors were produced by the unmodified reference (tests/golden/make_golden.py);
every case here must match bit-for-bit before the oracle is trusted as the GPU checker.
"""

from __future__ import annotations

import hashlib
import math
import struct

import numpy as np
import pytest

from conftest import REGIMES, golden, grid_arrays, sel_tuple
from oracle import oracle


def test_policy_select_matches_reference():
    doc = golden("policy_golden.json")
    n_checked = 0
    for case in doc["cases"]:
        g = grid_arrays(case["grid"])
        for regime in REGIMES:
            idx = oracle.Index(g, regime, case["batching_mtl"], case["multi_tenant_bs"])
            for cap, want in zip(case["caps"], case["select"][regime]):
                sel, cnt = idx.select(cap)
                assert sel_tuple(case["grid"], sel, cnt) == want, (case["name"], regime, cap)
                bf = oracle.bruteforce(g, regime, cap, case["batching_mtl"], case["multi_tenant_bs"])
                assert bf == sel, (case["name"], regime, cap)
                n_checked += 1
    assert n_checked > 10_000


def test_policy_quirks_inf_nan():
    doc = golden("policy_golden.json")
    g1 = doc["cases"][0]
    assert g1["name"] == "g1"
    g = grid_arrays(g1["grid"])
    for regime in REGIMES:
        idx = oracle.Index(g, regime)
        for key, cap in (("inf", math.inf), ("nan", math.nan)):
            sel, cnt = idx.select(cap)
            assert sel_tuple(g1["grid"], sel, cnt) == doc["g1_quirks"][regime][key]


def test_negative_cap_rejected():
    g = grid_arrays(golden("policy_golden.json")["cases"][0]["grid"])
    with pytest.raises(ValueError):
        oracle.Index(g, "combination").select(-1.0)


def _digest(grid_doc, sel, cnt):
    order = [-1 if s < 0 else grid_doc["entries"][s][0] * 100000 + grid_doc["entries"][s][1] for s in sel]
    raw = struct.pack(f"<{len(order)}q", *order) + struct.pack(f"<{len(cnt)}q", *[int(c) for c in cnt])
    return hashlib.sha256(raw).hexdigest()


def test_simulate_matches_reference_exactly():
    doc = golden("sim_golden.json")
    for run in doc["runs"]:
        gdoc = doc["grids"][run["grid"]]
        g = grid_arrays(gdoc)
        caps = doc["traces"][run["trace"]]
        r = oracle.simulate(g, caps, run["policy"], run["step_seconds"], run["switch_penalty_s"])
        key = (run["name"], run["policy"], run["switch_penalty_s"])
        assert r.avg_throughput_ips == run["avg_throughput_ips"], key
        assert r.energy_proxy_wh == run["energy_proxy_wh"], key
        assert r.idle_steps == run["idle_steps"], key
        assert _digest(gdoc, r.sel, r.count) == run["digest"]["sha256"], key
        if "steps" in run:
            got = [sel_tuple(gdoc, int(s), int(c)) for s, c in zip(r.sel, r.count)]
            assert got == run["steps"], key


def test_fsum_is_exactly_rounded():
    rng = np.random.default_rng(5)
    for _ in range(50):
        x = rng.standard_normal(rng.integers(1, 2000)) * 10.0 ** rng.integers(-5, 8, 1)
        assert oracle.fsum(x) == math.fsum(x.tolist())
    assert oracle.fsum([1e100, 1.0, -1e100, 1e-100]) == math.fsum([1e100, 1.0, -1e100, 1e-100])


def test_batch_driver_matches_single_runs():
    doc = golden("sim_golden.json")
    grids = [grid_arrays(doc["grids"][k]) for k in ("synth-a", "synth-b")]
    rng = np.random.default_rng(3)
    caps = (rng.random((5, 300)) * 350).astype(np.float32)
    avg, idle, en, used = oracle.simulate_batch(grids, caps, 60, 15.0, n_threads=3)
    assert used == 3
    for t in range(caps.shape[0]):
        for m, g in enumerate(grids):
            for p, regime in enumerate(REGIMES):
                r = oracle.simulate(g, caps[t].astype(np.float64), regime, 60, 15.0)
                assert avg[t, m, p] == r.avg_throughput_ips
                assert idle[t, m, p] == r.idle_steps
                assert en[t, m, p] == r.energy_proxy_wh
