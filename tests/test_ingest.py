"""Trace ingestion fast path (csrc/ingest.cpp) against the reference's load_trace outcomes.

tests/golden/ingest_golden.json holds what the UNMODIFIED reference (trace.py:87-169) returned
or raised for 55 CSV texts; every case must come out identical through the drop-in
load_trace, and the native parser must accept exactly the files of its grammar and never
accept a file the reference rejects. CPU only (host parsing, no device)."""

from __future__ import annotations

import hashlib
import math
import random
import struct
from datetime import timedelta

import numpy as np
import pytest

from conftest import golden

import paper_2306_12247_b200 as cs
from paper_2306_12247_b200 import trace as T

CASES = golden("ingest_golden.json")["cases"]
# files the native grammar must take (the rest may legitimately go through the rules loader)
NATIVE = {"canonical_hourly", "minute_day", "second_week_head", "long_100k", "crlf", "cr_only",
          "no_trailing_newline", "blank_and_space_rows", "field_whitespace", "header_padded",
          "vt_ff_fs_separators", "lower_z", "offset_plus", "offset_minus_zero", "naive_utc", "space_separator",
          "fraction_6", "fraction_3", "leap_day", "year_boundary", "old_date", "gap_filled",
          "gap_filled_minutes"}


def rows(values, step, start, dec):
    return [f"{(start + timedelta(seconds=i * step)).strftime('%Y-%m-%dT%H:%M:%SZ')},{v:.{dec}f}"
            for i, v in enumerate(values)]


def case_text(c) -> str:
    if "text" in c:
        return c["text"]
    s = c["gen"]  # same recipe as tests/golden/make_ingest_golden.py:gen_text
    g = random.Random(s["seed"])
    vals = [round(g.uniform(0, 350), s["dec"]) for _ in range(s["n"])]
    start = __import__("datetime").datetime(2020, 1, 1, tzinfo=__import__("datetime").timezone.utc)
    return "\n".join(["timestamp,capacity_w"] + rows(vals, s["step"], start, s["dec"])) + "\n"


def write(tmp_path, c):
    p = tmp_path / f"{c['name']}.csv"
    p.write_bytes(case_text(c).encode("utf-8"))
    return p


def bits(values):
    return struct.pack(f"<{len(values)}d", *values)


def native_status(path, step, gap_fill):
    with T._Parsed([path], step, gap_fill, 1) as p:
        inf = p.info(0)
        return inf.status, (p.values(0, inf.n_values) if inf.status == 0 else None)


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_load_trace_matches_reference(tmp_path, c):
    p = write(tmp_path, c)
    want = c["result"]
    if not want["ok"]:
        exc = getattr(cs, want["exc"], None) or {"ValueError": ValueError}[want["exc"]]
        with pytest.raises(exc) as ei:
            cs.load_trace(p, c["step_seconds"], gap_fill=c["gap_fill"])
        assert type(ei.value).__name__ == want["exc"]
        assert str(ei.value) == want["msg"].replace("{path}", str(p))
        return
    tr = cs.load_trace(p, c["step_seconds"], gap_fill=c["gap_fill"])
    assert tr.source_label == want["label"] and tr.step_seconds == want["step_seconds"]
    assert tr.start_time.isoformat() == want["start"]
    assert len(tr.values) == want["n"]
    assert hashlib.sha256(bits(tr.values)).hexdigest() == want["sha256"]  # bit-exact, -0.0 included
    if "values" in want:
        assert bits(tr.values) == bits(want["values"])
    assert all(type(v) is float for v in tr.values[:10])
    assert np.array_equal(cs.trace_array(tr), np.array(tr.values))


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_native_grammar_is_sound(tmp_path, c):
    """Native OK => the reference loaded the file and the samples are identical; the native
    grammar covers every canonical spelling (so the fast path is what actually runs)."""
    if c["step_seconds"] <= 0:
        return
    p = write(tmp_path, c)
    st, vals = native_status(p, c["step_seconds"], c["gap_fill"])
    if st == 0:
        assert c["result"]["ok"], c["name"]
        assert hashlib.sha256(bits(vals.tolist())).hexdigest() == c["result"]["sha256"]
    if c["name"] in NATIVE:
        assert st == 0, c["name"]


def test_native_parser_is_what_runs(tmp_path, monkeypatch):
    c = next(c for c in CASES if c["name"] == "minute_day")
    p = write(tmp_path, c)
    monkeypatch.setattr(T, "_load_trace_rules", lambda *a, **k: pytest.fail("rules loader used"))
    tr = cs.load_trace(p, 60)
    assert "_cs_values" in tr.__dict__ and len(tr) == 1440


def test_batch_and_matrix_loaders(tmp_path):
    rng = random.Random(5)
    start = __import__("datetime").datetime(2021, 6, 1, tzinfo=__import__("datetime").timezone.utc)
    paths = []
    for i in range(48):
        vals = [round(rng.uniform(0, 350), 6) for _ in range(777)]
        p = tmp_path / f"t{i:03d}.csv"
        p.write_text("\n".join(["timestamp,capacity_w"] + rows(vals, 60, start + timedelta(days=i), 6)) + "\n")
        paths.append(p)
    one = [cs.load_trace(p, 60) for p in paths]
    many = cs.load_traces(paths, 60, n_threads=4)
    assert many == one
    m64 = cs.load_trace_matrix(paths, 60, n_threads=4)
    assert m64.values.shape == (48, 778) and m64.n_steps == 777
    assert m64.start_times == tuple(t.start_time for t in one) and m64.labels == tuple(t.source_label for t in one)
    for i, t in enumerate(one):
        assert bits(m64.values[i, :777].tolist()) == bits(t.values) and m64.values[i, 777] == 0.0
    m32 = cs.load_trace_matrix(paths, 60, dtype="f32")
    assert m32.values.shape == (48, 780)
    assert np.array_equal(m32.values[:, :777], m64.values[:, :777].astype(np.float32))
    # an exotic spelling in the batch goes through the rules loader for that file only
    q = tmp_path / "t999.csv"
    q.write_text(paths[0].read_text().replace("T00:00:00Z", "x00:00:00"))
    mx = cs.load_trace_matrix(paths[:3] + [q], 60)
    assert np.array_equal(mx.values[3], mx.values[0])
    with pytest.raises(ValueError, match="differ in length"):
        r = tmp_path / "short.csv"
        r.write_text("\n".join(paths[0].read_text().splitlines()[:10]) + "\n")
        cs.load_trace_matrix(paths[:2] + [r], 60)


def test_fuzz_native_vs_rules(tmp_path):
    """Random files in and around the native grammar: native results equal the Python
    restatement of the reference rules (itself pinned to the golden outcomes above)."""
    rng = random.Random(11)
    fmts = ["%Y-%m-%dT%H:%M:%SZ", "%Y-%m-%dT%H:%M:%Sz", "%Y-%m-%d %H:%M:%S", "%Y-%m-%dT%H:%M:%S+00:00",
            "%Y-%m-%dT%H:%M:%S.%f", "%Y-%m-%dT%H:%M:%S"]
    nums = [lambda v: f"{v:.6f}", lambda v: repr(v), lambda v: f"{v:.3e}", lambda v: f" {v:g} ", lambda v: f"+{v}",
            lambda v: f"{int(v)}"]
    checked = 0
    for k in range(150):
        step = rng.choice([1, 60, 900, 3600])
        n = rng.randint(1, 60)
        t0 = __import__("datetime").datetime(rng.randint(1970, 2030), rng.randint(1, 12), rng.randint(1, 28),
                                             tzinfo=__import__("datetime").timezone.utc)
        lines, t = ["timestamp,capacity_w"], t0
        for i in range(n):
            t += timedelta(seconds=step * (1 if rng.random() > 0.1 else rng.randint(1, 3)))
            v = rng.uniform(0, 400) if rng.random() > 0.05 else rng.choice([0.0, -0.0, 1e-300])
            lines.append(f"{t.strftime(rng.choice(fmts))},{rng.choice(nums)(v)}")
            if rng.random() < 0.05:
                lines.append(rng.choice(["", "  ", "\t"]))
        nl = rng.choice(["\n", "\r\n", "\r"])
        p = tmp_path / f"f{k}.csv"
        p.write_bytes((nl.join(lines) + nl).encode())
        gap_fill = rng.random() < 0.7
        try:
            want = T._load_trace_rules(p, step, gap_fill, p.stem)
        except Exception as exc:  # noqa: BLE001
            want = exc
        st, vals = native_status(p, step, gap_fill)
        if st == 0:
            assert not isinstance(want, Exception), (k, want)
            assert bits(vals.tolist()) == bits(want.values)
            checked += 1
        got = None
        try:
            got = cs.load_trace(p, step, gap_fill=gap_fill)
        except Exception as exc:  # noqa: BLE001
            got = exc
        if isinstance(want, Exception):
            assert type(got) is type(want) and str(got) == str(want)
        else:
            assert got == want and got.start_time == want.start_time
            assert all(math.copysign(1, a) == math.copysign(1, b) for a, b in zip(got.values, want.values))
    assert checked > 60


def test_os_errors_match_the_reference_loader(tmp_path):
    """Unreadable paths fall through to the rules loader, which raises what open() raises."""
    with pytest.raises(FileNotFoundError):
        cs.load_trace(tmp_path / "missing.csv", 60)
    with pytest.raises(IsADirectoryError):
        cs.load_trace(tmp_path, 60)
    with pytest.raises(ValueError, match="step_seconds must be positive"):
        cs.load_traces([tmp_path / "missing.csv"], 0)


def test_large_gap_fill_and_long_rows(tmp_path):
    p = tmp_path / "gappy.csv"
    p.write_text("timestamp,capacity_w\n2020-01-01T00:00:00Z,5.5\n2021-01-01T00:00:00Z,6.5\n")
    tr = cs.load_trace(p, 60, gap_fill=True)
    assert len(tr) == 366 * 1440 + 1 and tr.values[-2] == 5.5 and tr.values[-1] == 6.5
    assert "_cs_values" in tr.__dict__  # filled natively
