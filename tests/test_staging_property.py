"""Property test of N1 staging (CPU): for random and tie-heavy grids, merged into unions of up to
four grids, every LUT the kernel can stage (default and finer, fp32 and fp64 caps) maps every
cap to the union bin whose decoded (selection, feasible_count) per regime equals the oracle's
PolicyIndex restatement (itself pinned to the reference's golden vectors)."""

from __future__ import annotations

import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import oracle
from paper_2306_12247_b200 import Config, ProfileEntry, ProfileGrid
from paper_2306_12247_b200.engine import Tables

REG = ("batching", "multi-tenant", "combination")


@st.composite
def grids(draw):
    n = draw(st.integers(1, 60))
    tie = draw(st.booleans())
    keys = draw(st.lists(st.tuples(st.integers(1, 4), st.integers(1, 32)), min_size=n, max_size=n, unique=True))
    entries = {}
    for mtl, bs in keys:
        if tie:  # quantised values: equal powers and throughputs exercise the tie-break chain
            thr = float(draw(st.integers(1, 8)) * 50)
            pw = float(draw(st.integers(1, 7)) * 50)
        else:
            thr = draw(st.floats(1.0, 20000.0, allow_nan=False))
            pw = draw(st.floats(1.0, 350.0, allow_nan=False))
        entries[Config(mtl, bs)] = ProfileEntry(Config(mtl, bs), thr, pw)
    return ProfileGrid("m", "gpu", 350.0, 1e6, entries)


def oracle_grid(g: ProfileGrid):
    cfgs = list(g.entries)
    return cfgs, oracle.GridArrays(np.array([c.mtl for c in cfgs], np.int32), np.array([c.bs for c in cfgs], np.int32),
                                   np.array([g.entries[c].throughput_ips for c in cfgs]),
                                   np.array([g.entries[c].power_w for c in cfgs]), 0.0)


def caps_for(gs, rng):
    pw = np.concatenate([np.array([e.power_w for e in g.entries.values()]) for g in gs])
    c = np.concatenate([pw, np.nextafter(pw, 0), np.nextafter(pw, 1e9), rng.uniform(0, 400, 64),
                        [0.0, -0.0, 1e-300, 350.0, 1e30, np.inf]])
    return c


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.lists(grids(), min_size=1, max_size=4), st.integers(0, 2**31 - 1))
def test_union_lut_matches_oracle(gs, seed):
    rng = np.random.default_rng(seed)
    caps64 = caps_for(gs, rng)
    for dtype in ("f64", "f32"):
        caps = caps64.astype(np.float32) if dtype == "f32" else caps64
        exact = caps.astype(np.float64)
        t = Tables.stage(gs, dtype)
        luts = ["main"] + (["big"] if t.info.lut_big_entries else [])
        for lut in luts:
            ub = t.lookup_host(caps, lut)
            for m, g in enumerate(gs):
                cfgs, og = oracle_grid(g)
                gb = t.grid_bins(m)
                gcfgs = g.columns()[0]
                for p, regime in enumerate(REG):
                    idx = oracle.Index(og, regime)
                    for cap, u in zip(exact, ub):
                        s_want, c_want = idx.select(max(float(cap), 0.0) if cap == cap else float(cap))
                        b = int(gb.umap[u])
                        s_got, c_got = int(gb.sel[p, b]), int(gb.count[p, b])
                        want = None if s_want < 0 else cfgs[s_want]
                        got = None if s_got < 0 else gcfgs[s_got]
                        assert (got, c_got) == (want, c_want), (dtype, lut, m, regime, float(cap))
