"""Host-side input API of the drop-in (profile tables, traces, records) vs the reference's
documented behaviour and golden outputs. CPU only."""

from __future__ import annotations

import hashlib
import math
import struct
from datetime import datetime, timezone

import pytest

from conftest import golden
import paper_2306_12247_b200 as cs
from paper_2306_12247_b200.errors import ParseError, ValidationError


def test_synthesize_grid_bit_identical_to_reference():
    for d in golden("synth_golden.json")["grids"]:
        g = cs.synthesize_grid(cs.SynthParams(**d["params"]))
        assert len(g) == d["n"]
        assert hashlib.sha256(cs.grid_csv_text(g).encode()).hexdigest() == d["csv_sha256"]
        raw = b"".join(struct.pack("<iidd", c.mtl, c.bs, e.throughput_ips, e.power_w)
                       for c, e in sorted(g.entries.items()))
        assert hashlib.sha256(raw).hexdigest() == d["entries_sha256"]


def test_grid_csv_round_trip(tmp_path):
    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=8, seed=11))
    p = tmp_path / "g.csv"
    cs.save_grid(g, p)
    assert cs.grid_csv_text(cs.load_grid(p)) == cs.grid_csv_text(g)


def test_trace_csv_round_trip_and_gap_fill(tmp_path):
    text = "timestamp,capacity_w\n2020-01-01T00:00:00Z,100.000000\n2020-01-01T01:00:00Z,157.250000\n" \
           "2020-01-01T02:00:00Z,0.000000\n"
    p = tmp_path / "t.csv"
    p.write_text(text)
    assert cs.trace_csv_text(cs.load_trace(p, 3600)) == text
    gap = "timestamp,capacity_w\n2020-01-01T00:00:00Z,5\n2020-01-01T03:00:00Z,7\n"
    p.write_text(gap)
    with pytest.raises(ValidationError, match="gap"):
        cs.load_trace(p, 3600)
    assert cs.load_trace(p, 3600, gap_fill=True).values == (5.0, 5.0, 5.0, 7.0)
    p.write_text("timestamp,capacity_w\n2020-01-01T00:00:00Z,-5\n")
    with pytest.raises(ValidationError, match="negative"):
        cs.load_trace(p, 3600)
    p.write_text("time,cap\n")
    with pytest.raises(ParseError):
        cs.load_trace(p, 3600)


def test_power_trace_invariants():
    t0 = datetime(2020, 1, 1, tzinfo=timezone.utc)
    with pytest.raises(ValidationError):
        cs.PowerTrace("x", 60, t0, ())
    with pytest.raises(ValidationError):
        cs.PowerTrace("x", 60, t0, (1.0, math.inf))
    with pytest.raises(ValidationError):
        cs.PowerTrace("x", 0, t0, (1.0,))
    tr = cs.PowerTrace("x", 60, t0, (-0.0, 5))  # -0.0 is accepted (trace.py:50 rejects < 0 only)
    assert tr.values == (-0.0, 5.0)
    n = cs.normalize_trace(cs.PowerTrace("x", 60, t0, (0, 50, 100)), 350.0)
    assert n.values == (0.0, 175.0, 350.0)
    st = cs.trace_stats(cs.PowerTrace("x", 60, t0, (239.57 - 76.1, 239.57 + 76.1)))
    assert st.variation_pct == pytest.approx(31.76, abs=0.01)


def test_grid_validation_messages():
    e = cs.ProfileEntry(cs.Config(1, 1), 10.0, 400.0)
    with pytest.raises(ValidationError, match="exceeds GPU max"):
        cs.ProfileGrid("m", "g", 350.0, 1000.0, {cs.Config(1, 1): e})
    with pytest.raises(ValidationError):
        cs.ProfileEntry(cs.Config(1, 1), 0.0, 10.0)
    with pytest.raises(ValidationError):
        cs.Config(0, 1)
    with pytest.raises(ValidationError):
        cs.sampling_policy(0)
    assert cs.sampling_policy(4, 2).label == "sampling(m=4,r=2)"
    assert round(cs.improvement_pct(13431.0, 1241.0)) == 982
    assert cs.profiling_cost(4, 128, 60.0) == 30720.0


def test_report_json_schema_round_trip(tmp_path):
    sel = cs.Selection(cs.Config(2, 1), 190.0, 160.0, 3)
    steps = (cs.StepRecord(0, 200.0, sel, False), cs.StepRecord(1, 50.0, cs.IDLE_SELECTION, True))
    rep = cs.SimReport("m", cs.COMBINATION, "fixture", 3600, 0.0, 2, 95.0, 1, 160.0, steps)
    p = tmp_path / "r.json"
    cs.save_report(rep, p)
    assert cs.load_report(p) == rep
    assert cs.slice_report(rep, 0, 2) == rep
    doc = cs.report_to_dict(rep)
    doc["schema_version"] = 99
    with pytest.raises(ValidationError, match="schema"):
        cs.report_from_dict(doc)
    with pytest.raises(ValidationError, match="elided"):
        cs.slice_report(cs.report_from_dict(cs.report_to_dict(rep, summary_only=True)), 0, 1)
