"""Generate the golden vectors that pin the oracle (and the CUDA path) to the reference.

Run ONCE in the build container, where the reference package is importable:

    CAPSIM_REF=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the UNMODIFIED reference (capsim 0.1.0) plus its own test helpers
(pkg/tests/conftest.py: random_grid, synthetic_year_values) and records the reference's
outputs as JSON. Nothing in the repo imports the reference at run time; the GPU box never
sees /root/reference. Floats are stored via json (repr round-trips exactly).

Vector sets (reference file:line they pin):
  policy_golden.json  PolicyIndex.select / select_config / feasible_set   policy.py:110-188
  sim_golden.json     simulate + _aggregate (+ slice_report, compare)      sim.py:104-252
  synth_golden.json   synthesize_grid                                      profile.py:169-215
  controller_golden.json  controller.replay                                controller.py:96-231
  sampling_golden.json    select_sampling + simulate(sampling_policy)      policy.py:191-273, sim.py:159-163
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import random
import struct
import sys
from pathlib import Path

REF = os.environ.get("CAPSIM_REF", "/root/reference/pkg/src")
REF_TESTS = str(Path(REF).parent / "tests")
sys.path.insert(0, REF)
sys.path.insert(0, REF_TESTS)

import capsim  # noqa: E402  (reference, build container only)
from capsim.policy import (  # noqa: E402
    BATCHING,
    COMBINATION,
    MULTI_TENANT,
    PolicyIndex,
    feasible_set,
    select_config,
)
from capsim.profile import Config, ProfileEntry, ProfileGrid, SynthParams, grid_csv_text, synthesize_grid  # noqa: E402
from capsim.sim import compare, simulate, slice_report  # noqa: E402
from capsim.trace import PowerTrace, normalize_trace  # noqa: E402
from conftest import G1_POINTS, random_grid, synthetic_year_values  # noqa: E402

OUT = Path(__file__).resolve().parent
KINDS = {"batching": BATCHING, "multi-tenant": MULTI_TENANT, "combination": COMBINATION}
T0 = __import__("datetime").datetime(2020, 1, 1, tzinfo=__import__("datetime").timezone.utc)


def f32(x: float) -> float:
    return struct.unpack("<f", struct.pack("<f", x))[0]


def grid_doc(grid: ProfileGrid) -> dict:
    return {
        "model_name": grid.model_name,
        "gpu_max_power_w": grid.gpu_max_power_w,
        "gpu_memory_mb": grid.gpu_memory_mb,
        "gpu_idle_power_w": grid.gpu_idle_power_w,
        "entries": [[c.mtl, c.bs, e.throughput_ips, e.power_w] for c, e in sorted(grid.entries.items())],
    }


def build(points: dict, **kw) -> ProfileGrid:
    entries = {}
    for (mtl, bs), (ips, w) in points.items():
        c = Config(mtl, bs)
        entries[c] = ProfileEntry(c, ips, w)
    return ProfileGrid(
        model_name=kw.pop("model_name", "model-a"),
        gpu_name="gpu-x",
        gpu_max_power_w=kw.pop("gpu_max_power_w", 350.0),
        gpu_memory_mb=24576.0,
        entries=entries,
        **kw,
    )


def sel_doc(sel) -> list | None:
    if sel.config is None:
        return None
    return [sel.config.mtl, sel.config.bs, sel.throughput_ips, sel.power_w, sel.feasible_count]


def boundary_caps(grid: ProfileGrid, rng: random.Random, n_random: int) -> list[float]:
    caps = [0.0, -0.0]
    pws = [e.power_w for e in grid.entries.values()]
    for p in rng.sample(pws, min(len(pws), 12)):
        caps += [p, math.nextafter(p, math.inf), math.nextafter(p, -math.inf)]
        # fp32 neighbours: the fp32 kernel must agree with fp64 semantics on every fp32 cap
        q = f32(p)
        caps += [q, f32(math.nextafter(q, math.inf)) if q < 3e38 else q]
        dn = struct.unpack("<f", struct.pack("<I", struct.unpack("<I", struct.pack("<f", q))[0] - 1))[0] if q > 0 else 0.0
        caps.append(dn)
    caps += [rng.uniform(0.0, 360.0) for _ in range(n_random)]
    caps += [f32(rng.uniform(0.0, 360.0)) for _ in range(n_random)]
    return [c for c in caps if c >= 0 or c == 0.0]


def policy_golden() -> dict:
    rng = random.Random(20240612)
    cases = []
    g1 = build(G1_POINTS)
    g1_caps = [0.0, -0.0, 50.0, 99.999999, 100.0, 120.0, 149.99999999999997, 150.0, 159.999999, 160.0,
               180.0, 200.0, 219.99, 220.0, 250.0, 300.0, 350.0, 1e9]
    cases.append(("g1", g1, g1_caps, 1, 1))
    ties = [
        {(1, 4): (500.0, 210.0), (2, 2): (500.0, 200.0), (3, 1): (400.0, 150.0)},
        {(2, 3): (500.0, 200.0), (1, 6): (500.0, 200.0)},
        {(2, 5): (500.0, 200.0), (2, 3): (500.0, 200.0)},
        {(1, 1): (100.0, 150.0), (1, 2): (100.0, 150.0), (2, 1): (100.0, 150.0)},  # equal powers, count 3
    ]
    for i, pts in enumerate(ties):
        cases.append((f"tie{i}", build(pts), [0.0, 149.0, 150.0, 199.9, 200.0, 205.0, 210.0, 300.0], 1, 1))
    for i in range(96):
        grid = random_grid(rng, tie_heavy=(i % 2 == 0))
        cases.append((f"rand{i}", grid, boundary_caps(grid, rng, 16), 1, 1))
    # non-default regime parameters (policy.py:118-125, 151-179)
    for i in range(12):
        grid = random_grid(rng, tie_heavy=(i % 3 == 0))
        mtls = sorted({c.mtl for c in grid.entries})
        bss = sorted({c.bs for c in grid.entries})
        cases.append((f"regime{i}", grid, boundary_caps(grid, rng, 8), rng.choice(mtls), rng.choice(bss)))
    # a synthetic 4x128 grid (dense thresholds near p_max)
    sg = synthesize_grid(SynthParams(mtl_cap=4, bs_cap=128, model_name="mobilenet-v1"))
    cases.append(("synth512", sg, boundary_caps(sg, rng, 64), 1, 1))

    docs = []
    for name, grid, caps, bmtl, mbs in cases:
        res = {}
        for label, kind in KINDS.items():
            idx = PolicyIndex(grid, kind, batching_mtl=bmtl, multi_tenant_bs=mbs)
            res[label] = [sel_doc(idx.select(c)) for c in caps]
            for c, s in zip(caps, res[label]):
                assert s == sel_doc(select_config(grid, kind, c, batching_mtl=bmtl, multi_tenant_bs=mbs))
        fs_caps = caps[:6]
        fsets = {
            label: [sorted([c.mtl, c.bs] for c in feasible_set(grid, kind, cap, batching_mtl=bmtl,
                                                               multi_tenant_bs=mbs)) for cap in fs_caps]
            for label, kind in KINDS.items()
        }
        docs.append({"name": name, "grid": grid_doc(grid), "batching_mtl": bmtl, "multi_tenant_bs": mbs,
                     "caps": caps, "select": res, "feasible_caps": fs_caps, "feasible_set": fsets})
    # bisect quirks (policy.py:136-148): +inf selects the global best; NaN is not < 0 and also
    # bisects to the end. Stored as strings because JSON has no inf/nan.
    quirks = {}
    for label, kind in KINDS.items():
        quirks[label] = {"inf": sel_doc(select_config(g1, kind, math.inf)),
                         "nan": sel_doc(select_config(g1, kind, math.nan))}
    # PolicyIndex of a sampling kind: _regime_entries gives it every entry (policy.py:100-107), so
    # it answers like the combination index (it is select_config that rejects sampling kinds)
    from capsim.policy import sampling_policy

    sampling_index = {}
    for name, grid, caps, _, _ in (cases[0], cases[-1]):
        idx = PolicyIndex(grid, sampling_policy(4, 2))
        sampling_index[name] = [sel_doc(idx.select(c)) for c in caps]
    return {"source": "capsim 0.1.0 reference, policy.py:110-188", "cases": docs, "g1_quirks": quirks,
            "sampling_index": sampling_index}


def steps_digest(report) -> dict:
    order = []
    counts = []
    for s in report.steps:
        order.append(-1 if s.selection.config is None else s.selection.config.mtl * 100000 + s.selection.config.bs)
        counts.append(s.selection.feasible_count)
    raw = struct.pack(f"<{len(order)}q", *order) + struct.pack(f"<{len(counts)}q", *counts)
    return {"sha256": hashlib.sha256(raw).hexdigest()}


def report_doc(report, full_steps: bool) -> dict:
    d = {
        "avg_throughput_ips": report.avg_throughput_ips,
        "idle_steps": report.idle_steps,
        "energy_proxy_wh": report.energy_proxy_wh,
        "num_steps": report.num_steps,
        "idle_power_w": report.idle_power_w,
        "digest": steps_digest(report),
    }
    if full_steps:
        d["steps"] = [sel_doc(s.selection) for s in report.steps]
    return d


MODEL_PARAMS = [
    dict(t_max_ips=12000.0, tau=96.0, contention=0.95, gamma=0.7, p_idle_w=60.0, mem_model_mb=4096.0,
         model_name="synth-a", seed=101),
    dict(t_max_ips=9000.0, tau=128.0, contention=0.90, gamma=1.0, p_idle_w=50.0, mem_model_mb=6144.0,
         model_name="synth-b", seed=102),
    dict(t_max_ips=15000.0, tau=64.0, contention=0.97, gamma=0.8, p_idle_w=70.0, mem_model_mb=2048.0,
         model_name="synth-c", seed=103),
]


def sim_golden() -> dict:
    rng = random.Random(77)
    runs = []

    def add(name, grid, values, step_seconds, penalties, full):
        trace = PowerTrace(source_label=name, step_seconds=step_seconds, start_time=T0, values=tuple(values))
        for label, kind in KINDS.items():
            for pen in penalties:
                import warnings

                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    rep = simulate(grid, trace, kind, switch_penalty_s=pen)
                runs.append({"name": name, "policy": label, "switch_penalty_s": pen, "step_seconds": step_seconds,
                             "trace": name, **report_doc(rep, full)})

    traces = {}
    g1 = build(G1_POINTS)
    caps = [200.0, 100.0, 250.0]
    traces["caps3"] = caps
    add("caps3", g1, caps, 3600, [0.0, 1800.0, 3600.0, 5000.0], True)
    traces["zeros"] = [0.0, 0.0, 0.0]
    add("zeros", g1, traces["zeros"], 3600, [0.0], True)
    idle_grid = build({(1, 1): (100.0, 100.0)}, gpu_idle_power_w=40.0)
    traces["idle2"] = [150.0, 10.0]
    grids = {"g1": grid_doc(g1), "idle_grid": grid_doc(idle_grid)}
    runs_before = len(runs)
    add("idle2", idle_grid, traces["idle2"], 3600, [0.0], True)
    for r in runs[runs_before:]:
        r["grid"] = "idle_grid"
    for r in runs[:runs_before]:
        r["grid"] = "g1"
    # random grids x random traces, fp64 and fp32-representable caps, various step sizes
    for i in range(24):
        grid = random_grid(rng, tie_heavy=(i % 2 == 0))
        gname = f"rgrid{i}"
        grids[gname] = grid_doc(grid)
        n = rng.choice([1, 2, 7, 40, 101, 500])
        vals = [rng.uniform(0.0, 350.0) for _ in range(n)]
        if i % 3 == 0:
            vals = [f32(v) for v in vals]
        if i % 4 == 0 and n > 3:  # exact threshold hits
            pws = [e.power_w for e in grid.entries.values()]
            for j in range(0, n, 3):
                vals[j] = rng.choice(pws)
        step = rng.choice([1, 60, 3600])
        tname = f"rtrace{i}"
        traces[tname] = vals
        before = len(runs)
        add(tname, grid, vals, step, [0.0, step / 4.0, float(step), 2.0 * step], n <= 101)
        for r in runs[before:]:
            r["grid"] = gname
    # synthetic models x the synthetic year (test_acceptance.py:62-81, 166-179, 254-270)
    year = normalize_trace(
        PowerTrace(source_label="synth-year", step_seconds=3600, start_time=T0,
                   values=tuple(float(v) for v in synthetic_year_values(2020))), 350.0)
    traces["synth-year"] = list(year.values)
    for p in MODEL_PARAMS:
        grid = synthesize_grid(SynthParams(**p))
        gname = p["model_name"]
        grids[gname] = grid_doc(grid)
        before = len(runs)
        add("synth-year", grid, year.values, 3600, [0.0, 600.0], False)
        for r in runs[before:]:
            r["grid"] = gname
    # slice/compare on caps3 (sim.py:191-252)
    rep = simulate(g1, PowerTrace("fixture", 3600, T0, tuple(caps)), COMBINATION)
    rb = simulate(g1, PowerTrace("fixture", 3600, T0, tuple(caps)), BATCHING)
    sl = slice_report(rep, 0, 2)
    table = compare([rep, rb])
    extras = {
        "slice_0_2_avg": sl.avg_throughput_ips,
        "compare_rows": [[r.policy_a, r.policy_b, r.improvement_pct] for r in table.rows],
        "best_policy": table.best_policy,
    }
    return {"source": "capsim 0.1.0 reference, sim.py:104-252", "grids": grids, "traces": traces, "runs": runs,
            "extras": extras}


def synth_golden() -> dict:
    params = [
        dict(mtl_cap=2, bs_cap=8, seed=11),
        dict(mtl_cap=3, bs_cap=5, seed=7, noise_pct=1.5),
        dict(mtl_cap=4, bs_cap=128, model_name="mobilenet-v1"),
        dict(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0, model_name="fine-8x512"),
    ] + MODEL_PARAMS
    out = []
    for p in params:
        g = synthesize_grid(SynthParams(**p))
        text = grid_csv_text(g)
        d = {"params": p, "n": len(g), "csv_sha256": hashlib.sha256(text.encode()).hexdigest()}
        ent = sorted(g.entries.items())
        raw = b"".join(struct.pack("<iidd", c.mtl, c.bs, e.throughput_ips, e.power_w) for c, e in ent)
        d["entries_sha256"] = hashlib.sha256(raw).hexdigest()
        if len(g) <= 64:
            d["entries"] = [[c.mtl, c.bs, e.throughput_ips, e.power_w] for c, e in ent]
        out.append(d)
    return {"source": "capsim 0.1.0 reference, profile.py:169-215", "grids": out}


def controller_golden() -> dict:
    """controller.replay (controller.py:161-231): events, selections and aggregates."""
    from capsim.controller import REACTIVE, proactive, replay

    rng = random.Random(9)
    g1 = build(G1_POINTS)
    g2 = build({(1, 1): (100.0, 100.0), (1, 2): (180.0, 150.0), (2, 1): (200.0, 240.0), (2, 2): (320.0, 260.0)})
    cases = [
        ("g1_rising", g1, [100.0, 150.0, 200.0, 250.0, 300.0], None, "reactive", 1, 0.0, 0),
        ("g1_fixture_r", g1, [250.0, 250.0, 150.0], (2, 2), "reactive", 1, 0.0, 0),
        ("g1_fixture_p", g1, [250.0, 250.0, 150.0], (2, 2), "proactive", 2, 0.0, 0),
        ("g1_flat", g1, [200.0] * 20, None, "proactive", 3, 0.0, 0),
        ("g1_noise", g1, [200.0, 180.0, 160.0, 220.0, 140.0], None, "reactive", 1, 2.0, 13),
        ("g1_idle", g1, [250.0, 10.0], (2, 2), "reactive", 1, 0.0, 0),
        ("g2_pre", g2, [230.0, 250.0, 270.0, 200.0, 150.0, 300.0], (2, 2), "proactive", 3, 0.0, 0),
    ]
    for i in range(30):
        grid = random_grid(rng, tie_heavy=(i % 3 == 0))
        n = rng.choice([1, 5, 40, 200])
        caps = [rng.uniform(0.0, 350.0) for _ in range(n)]
        mode = rng.choice(["reactive", "proactive"])
        k = rng.randint(1, 6)
        noise = rng.choice([0.0, 0.5, 2.0, 10.0])
        seed = rng.choice([0, 1, 5, 123456789, 2**40 + 7, -77, 2**70 + 3])
        init = None
        if i % 2 == 0:
            c = rng.choice(sorted(grid.entries))
            init = (c.mtl, c.bs)
        cases.append((f"rand{i}", grid, caps, init, mode, k, noise, seed))
    docs = []
    for name, grid, caps, init, mode, k, noise, seed in cases:
        m = REACTIVE if mode == "reactive" else proactive(k)
        rep = replay(grid, PowerTrace(name, 60, T0, tuple(caps)), m,
                     initial_config=None if init is None else Config(*init), noise_pct=noise, seed=seed)
        docs.append({
            "name": name, "grid": grid_doc(grid), "caps": caps, "initial": init, "mode": mode, "window_k": k,
            "noise_pct": noise, "seed": seed,
            "events": [[e.step_index, e.kind.value, e.cap_w, e.power_w] for e in rep.events],
            "selections": [sel_doc(s) if s.config is not None else None for s in rep.selections],
            "violations": rep.violations, "reconfigs": rep.reconfigs,
            "violation_fraction": rep.violation_fraction, "avg_throughput_ips": rep.avg_throughput_ips,
            "num_steps": rep.num_steps,
        })
    return {"source": "capsim 0.1.0 reference, controller.py:96-231", "cases": docs}


def sampling_golden() -> dict:
    """select_sampling (policy.py:218-273) incl. both random.sample branches (pool: n <= setsize,
    set: n > setsize), the hill climb, and simulate() with a sampling policy (sim.py:159-163)."""
    from capsim.policy import sampling_policy, select_sampling

    rng = random.Random(31337)
    g1 = build(G1_POINTS)
    chain = build({(1, 1): (100.0, 100.0), (1, 2): (200.0, 120.0), (1, 4): (300.0, 140.0), (1, 8): (400.0, 160.0)})
    sg = synthesize_grid(SynthParams(mtl_cap=4, bs_cap=128, model_name="mobilenet-v1"))
    seeds = [0, 1, 7, 12345, -5, 2**31 - 1, 2**32, 2**40 + 1, 2**70 + 3, -(2**33) - 9]
    cases = []

    def add(name, grid, caps, budgets, rounds, seed_list):
        sels = []
        for cap in caps:
            for b in budgets:
                for r in rounds:
                    for sd in seed_list:
                        sels.append([cap, b, r, sd, sel_doc_count(select_sampling(grid, b, r, cap, sd))])
        cases.append({"name": name, "grid": grid_doc(grid), "queries": sels})

    add("g1", g1, [0.0, 50.0, 100.0, 150.0, 200.0, 250.0, 350.0], [1, 2, 4, 10], [0, 1, 3], seeds[:6])
    add("chain", chain, [0.0, 130.0, 200.0], [1, 2], [0, 1, 3], seeds)
    for i in range(30):
        grid = random_grid(rng, tie_heavy=(i % 3 == 0))
        caps = boundary_caps(grid, rng, 2)[:10]
        add(f"rand{i}", grid, caps, [1, 2, 3, 6, rng.randint(7, 40)], [0, 1, 4], [rng.choice(seeds), i])
    caps = [0.0, 61.0, 100.0, 150.0, 200.0, 260.0, 300.0, 349.0, 350.0]
    add("synth512", sg, caps, [1, 5, 6, 8, 50, 200, 511, 600], [0, 2, 8], [3, -(2**33) - 9])

    runs = []
    sim_cases = [
        ("g1_caps", g1, [200.0, 100.0, 250.0, 0.0, 180.0, 300.0], [(2, 1), (1, 0), (4, 3)], [0, 5], [0.0, 1800.0]),
        ("synth_day", sg, [rng.uniform(0.0, 350.0) for _ in range(96)], [(1, 0), (4, 2), (30, 1)], [0, -3, 2**40],
         [0.0, 600.0]),
    ]
    for name, grid, vals, kinds, sds, pens in sim_cases:
        trace = PowerTrace(source_label=name, step_seconds=3600, start_time=T0, values=tuple(vals))
        for b, r in kinds:
            for sd in sds:
                for pen in pens:
                    rep = simulate(grid, trace, sampling_policy(b, r), seed=sd, switch_penalty_s=pen)
                    runs.append({"name": name, "budget_m": b, "rounds_r": r, "seed": sd, "switch_penalty_s": pen,
                                 **report_doc(rep, True)})
    return {"source": "capsim 0.1.0 reference, policy.py:191-273 + sim.py:159-163", "cases": cases,
            "sim": {"grids": {"g1_caps": grid_doc(g1), "synth_day": grid_doc(sg)},
                    "traces": {n: v for n, _, v, *_ in sim_cases}, "runs": runs}}


def sel_doc_count(sel) -> list:
    """Like sel_doc, but idle keeps its feasible_count (always 0) so the record is never null."""
    if sel.config is None:
        return [0, 0, 0.0, 0.0, sel.feasible_count]
    return sel_doc(sel)


def main() -> None:
    print("reference capsim from", capsim.__file__)
    for name, fn in (("policy_golden.json", policy_golden), ("sim_golden.json", sim_golden),
                     ("synth_golden.json", synth_golden), ("controller_golden.json", controller_golden),
                     ("sampling_golden.json", sampling_golden)):
        doc = fn()
        (OUT / name).write_text(json.dumps(doc, separators=(",", ":")) + "\n")
        print("wrote", name, (OUT / name).stat().st_size, "bytes")


if __name__ == "__main__":
    main()
