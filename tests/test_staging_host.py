"""N1 staging (host C++) checked against the reference's golden selections, on CPU.

cs_tables_lookup_host restates the device LUT search on the host, so the staged LUT,
the union-bin maps and the per-bin decode tables can be verified here without a GPU.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import REGIMES, golden, sel_tuple
from paper_2306_12247_b200 import Config, ProfileEntry, ProfileGrid, SynthParams, synthesize_grid
from paper_2306_12247_b200.engine import Tables


def grid_from_doc(doc) -> ProfileGrid:
    entries = {}
    for m, b, t, p in doc["entries"]:
        c = Config(m, b)
        entries[c] = ProfileEntry(c, t, p)
    return ProfileGrid(model_name=doc["model_name"], gpu_name="gpu-x", gpu_max_power_w=doc["gpu_max_power_w"],
                       gpu_memory_mb=doc["gpu_memory_mb"], entries=entries, gpu_idle_power_w=doc["gpu_idle_power_w"])


def decode(grid: ProfileGrid, tables: Tables, m: int, ubins, p: int):
    gb = tables.grid_bins(m)
    cfgs = grid.columns()[0]
    out = []
    for u in ubins:
        b = int(gb.umap[u])
        s, c = int(gb.sel[p, b]), int(gb.count[p, b])
        if s < 0:
            out.append(None)
        else:
            e = grid.entries[cfgs[s]]
            out.append([e.config.mtl, e.config.bs, e.throughput_ips, e.power_w, c])
    return out


def is_f32(x: float) -> bool:
    return float(np.float32(x)) == x


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_lut_and_decode_match_reference(dtype):
    doc = golden("policy_golden.json")
    checked = 0
    for case in doc["cases"]:
        grid = grid_from_doc(case["grid"])
        t = Tables.stage([grid], dtype, batching_mtl=case["batching_mtl"], multi_tenant_bs=case["multi_tenant_bs"])
        idx = [i for i, c in enumerate(case["caps"]) if dtype == "f64" or is_f32(c)]
        caps = np.array([case["caps"][i] for i in idx])
        luts = ["main"] + (["big"] if t.info.lut_big_entries else []) + (["huge"] if t.info.lut_huge_entries else [])
        for lut in luts:
            ub = t.lookup_host(caps, lut)
            for p, regime in enumerate(REGIMES):
                got = decode(grid, t, 0, ub, p)
                want = [case["select"][regime][i] for i in idx]
                assert got == want, (case["name"], dtype, regime, lut)
                checked += len(idx)
    assert checked > 5000


def test_union_of_grids_matches_per_grid_reference():
    """Several grids share one union-threshold LUT; each maps back to its own bins."""
    doc = golden("policy_golden.json")
    cases = [c for c in doc["cases"] if c["batching_mtl"] == 1 and c["multi_tenant_bs"] == 1][:40]
    for k in range(0, len(cases) - 4, 5):
        group = cases[k:k + 5]
        grids = [grid_from_doc(c["grid"]) for c in group]
        t = Tables.stage(grids, "f64")
        for m, c in enumerate(group):
            ub = t.lookup_host(np.array(c["caps"]))
            for p, regime in enumerate(REGIMES):
                assert decode(grids[m], t, m, ub, p) == c["select"][regime]


def test_dense_fine_grid_lut_is_exact():
    """8x512 grid: thousands of thresholds packed near p_max (multi-level sub-tables)."""
    from oracle import oracle

    g = synthesize_grid(SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    cfgs, mtl, bs, thr, pw = g.columns()
    ga = oracle.GridArrays(np.array(mtl, np.int32), np.array(bs, np.int32), np.array(thr), np.array(pw), 60.0)
    rng = np.random.default_rng(0)
    pws = np.array(pw)
    f32 = np.concatenate([
        rng.uniform(0, 360, 20000).astype(np.float32),
        pws.astype(np.float32),
        np.nextafter(pws.astype(np.float32), np.float32(np.inf)),
        np.nextafter(pws.astype(np.float32), np.float32(0)),
        np.array([0.0, -0.0, 350.0, 1e30], np.float32),
    ])
    for dtype, caps in (("f32", f32), ("f64", np.concatenate([f32.astype(np.float64), pws,
                                                              np.nextafter(pws, 0), np.nextafter(pws, 400)]))):
        t = Tables.stage([g], dtype)
        ub = t.lookup_host(caps)
        if dtype == "f32":  # the finer LUT the kernel prefers must give the same bins
            assert t.info.lut_big_entries > 0 and t.info.lut_big_shift < t.info.lut_shift
            assert np.array_equal(t.lookup_host(caps, "big"), ub)
        gb = t.grid_bins(0)
        idx = oracle.Index(ga, "combination")
        for cap, u in zip(caps.astype(np.float64)[::7], ub[::7]):
            s, cnt = idx.select(float(cap) if cap >= 0 else 0.0)
            b = gb.umap[u]
            assert int(gb.sel[2, b]) == s and int(gb.count[2, b]) == cnt


def test_negative_zero_and_bad_grids():
    g = ProfileGrid("m", "g", 350.0, 1000.0, {Config(1, 1): ProfileEntry(Config(1, 1), 10.0, 100.0)})
    for dt in ("f32", "f64"):
        t = Tables.stage([g], dt)
        assert list(t.lookup_host(np.array([-0.0, 0.0, 99.9, 100.0, 1e9]))) == [0, 0, 0, 1, 1]


def test_lut_leaves_proven_violation_free():
    """Every fp32 LUT leaf of every golden grid is proven (at staging) to select only configs
    whose power fits all caps the leaf serves — the basis of the kernel's per-step check."""
    doc = golden("policy_golden.json")
    for case in doc["cases"]:
        grid = grid_from_doc(case["grid"])
        t = Tables.stage([grid], "f32", batching_mtl=case["batching_mtl"], multi_tenant_bs=case["multi_tenant_bs"])
        assert t.info.lut_unsafe_leaves == 0 and t.info.lut_big_unsafe_leaves == 0, case["name"]
        assert t.info.lut_huge_unsafe_leaves == 0, case["name"]
        assert t.info.n_segments >= 3
    g = synthesize_grid(SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0))
    info = Tables.stage([g], "f32").info
    assert info.lut_unsafe_leaves == 0 and info.lut_big_unsafe_leaves == 0


def test_huge_lut_for_many_grids():
    """Ten grids (thousands of union thresholds): the staging also builds the shift-11 'huge' LUT
    that eval_kernel stages next to 8-warp groups; every LUT gives the same bins and is proven."""
    import bench

    t = Tables.stage(bench.make_grids("ten"), "f32")
    info = t.info
    assert info.lut_huge_entries > 0 and info.lut_huge_shift < info.lut_shift
    assert info.lut_huge_unsafe_leaves == 0
    rng = np.random.default_rng(5)
    thr = np.array(sorted({p for g in bench.make_grids("ten") for p in g.columns()[4]}), np.float64)
    caps = np.concatenate([rng.uniform(0, 360, 50000), thr, np.nextafter(thr, 0), np.nextafter(thr, 400),
                           [0.0, -0.0, 1e30, np.inf]]).astype(np.float32)
    ub = t.lookup_host(caps)
    assert np.array_equal(t.lookup_host(caps, "huge"), ub)
