"""Golden outcomes of the reference's load_trace (trace.py:87-169) for the ingestion fast path.

Run ONCE in the build container, where the reference package is importable:

    CAPSIM_REF=/root/reference/pkg/src python tests/golden/make_ingest_golden.py

Each case is a CSV text (canonical save_trace output, line-ending and whitespace variants,
timestamp spellings, gaps with and without gap_fill, and every error the loader raises). The
UNMODIFIED reference loads it from a file named <case>.csv; the JSON records either the samples
(exact floats; long traces as a sha256 of the packed fp64 plus head/tail) and start time, or the
exception type and message with the file path replaced by {path}. Nothing imports the reference
at test time.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import struct
import sys
import tempfile
from datetime import datetime, timedelta, timezone
from pathlib import Path

REF = os.environ.get("CAPSIM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from capsim.trace import PowerTrace, load_trace, trace_csv_text  # noqa: E402  (reference, build container only)

OUT = Path(__file__).resolve().parent / "ingest_golden.json"
T0 = datetime(2020, 1, 1, tzinfo=timezone.utc)


def rows(values, step, start=T0, fmt="%Y-%m-%dT%H:%M:%SZ", dec=6):
    return [f"{(start + timedelta(seconds=i * step)).strftime(fmt)},{v:.{dec}f}" for i, v in enumerate(values)]


def text(rows_, nl="\n", header="timestamp,capacity_w", trailing=True):
    return nl.join([header] + rows_) + (nl if trailing else "")


def gen_text(spec: dict) -> str:
    """Long cases are stored as a recipe, not text (tests/test_ingest.py rebuilds the same text)."""
    g = random.Random(spec["seed"])
    vals = [round(g.uniform(0, 350), spec["dec"]) for _ in range(spec["n"])]
    return text(rows(vals, spec["step"], dec=spec["dec"]))


def digest(values) -> str:
    return hashlib.sha256(struct.pack(f"<{len(values)}d", *values)).hexdigest()


def cases():
    rng = random.Random(2306)
    solar = [max(0.0, 350 * max(0.0, __import__("math").sin((h % 24 - 6) / 12 * 3.14159)) + rng.uniform(-5, 5))
             for h in range(72)]
    out = []

    def add(name, body, step=3600, gap_fill=False):
        if isinstance(body, dict):
            out.append({"name": name, "gen": body, "step_seconds": step, "gap_fill": gap_fill})
        else:
            out.append({"name": name, "text": body, "step_seconds": step, "gap_fill": gap_fill})

    tr = PowerTrace("canon", 3600, T0, tuple(round(v, 6) for v in solar))
    add("canonical_hourly", trace_csv_text(tr))
    minute = [round(rng.uniform(0, 350), 6) for _ in range(1440)]
    add("minute_day", text(rows(minute, 60)), step=60)
    add("second_week_head", {"seed": 7, "n": 5000, "step": 1, "dec": 3}, step=1)
    add("long_100k", {"seed": 8, "n": 100_000, "step": 60, "dec": 6}, step=60)
    add("crlf", text(rows(solar[:24], 3600), nl="\r\n"))
    add("cr_only", text(rows(solar[:24], 3600), nl="\r"))
    add("no_trailing_newline", text(rows(solar[:5], 3600), trailing=False))
    r = rows(solar[:6], 3600)
    add("blank_and_space_rows", text(r[:2] + ["", "   ", "\t"] + r[2:4] + [" \x1f "] + r[4:] + ["", ""]))
    add("field_whitespace", text([f"  {a} ,\t{b}  " for a, b in (x.split(",") for x in r)]))
    add("header_padded", text(r, header="  timestamp,capacity_w \t"))
    add("vt_ff_fs_separators", "timestamp,capacity_w\x0b" + "\x0c".join(r[:3]) + "\x1c" + "\x1d".join(r[3:]) + "\x1e")
    add("lower_z", text(rows(solar[:4], 3600, fmt="%Y-%m-%dT%H:%M:%Sz")))
    add("offset_plus", text(rows(solar[:4], 3600, fmt="%Y-%m-%dT%H:%M:%S+00:00")))
    add("offset_minus_zero", text(rows(solar[:4], 3600, fmt="%Y-%m-%dT%H:%M:%S-00:00")))
    add("naive_utc", text(rows(solar[:4], 3600, fmt="%Y-%m-%dT%H:%M:%S")))
    add("space_separator", text(rows(solar[:4], 3600, fmt="%Y-%m-%d %H:%M:%S")))
    add("fraction_6", text(rows(solar[:4], 3600, fmt="%Y-%m-%dT%H:%M:%S.000000Z")))
    add("fraction_3", text(rows(solar[:4], 3600, fmt="%Y-%m-%dT%H:%M:%S.000")))
    add("fraction_7_exotic", text(rows(solar[:4], 3600, fmt="%Y-%m-%dT%H:%M:%S.0000000")))
    add("basic_format_exotic", text(rows(solar[:4], 3600, fmt="%Y%m%dT%H%M%S")))
    add("other_separator_exotic", text(rows(solar[:4], 3600, fmt="%Y-%m-%dx%H:%M:%S")))
    add("leap_day", text(rows([1.0, 2.0, 3.0], 86400, start=datetime(2020, 2, 28, tzinfo=timezone.utc))), step=86400)
    add("year_boundary", text(rows([1.0, 2.0, 3.0], 3600, start=datetime(2020, 12, 31, 23, tzinfo=timezone.utc))))
    add("old_date", text(rows([5.0, 6.0], 3600, start=datetime(1900, 3, 1, tzinfo=timezone.utc))))
    add("number_spellings", text([
        "2020-01-01T00:00:00Z,1e2", "2020-01-01T01:00:00Z,.5", "2020-01-01T02:00:00Z,5.",
        "2020-01-01T03:00:00Z,+3", "2020-01-01T04:00:00Z,-0.0", "2020-01-01T05:00:00Z,0",
        "2020-01-01T06:00:00Z,1.5E-3", "2020-01-01T07:00:00Z,349.99999999999999",
        "2020-01-01T08:00:00Z,0.1", "2020-01-01T09:00:00Z,123456789012345678901234567890",
        "2020-01-01T10:00:00Z,2.2250738585072014e-308", "2020-01-01T11:00:00Z,1e-320"]))
    add("underscore_exotic", text(["2020-01-01T00:00:00Z,1_000.5", "2020-01-01T01:00:00Z,2"]))
    gap = rows([1.0, 2.0], 3600) + rows([3.0, 4.0], 3600, start=T0 + timedelta(hours=5))
    add("gap_error", text(gap))
    add("gap_filled", text(gap), gap_fill=True)
    add("gap_filled_minutes", text(rows([1.0], 60) + rows([2.0], 60, start=T0 + timedelta(minutes=100))), step=60,
        gap_fill=True)
    add("off_grid", text(rows([1.0], 3600) + ["2020-01-01T01:30:00Z,2.0"]))
    add("off_grid_fraction", text(rows([1.0], 3600) + ["2020-01-01T01:00:00.5Z,2.0"]))
    add("non_monotonic", text(rows([1.0, 2.0], 3600) + ["2020-01-01T00:30:00Z,3.0"]))
    add("duplicate_ts", text(rows([1.0, 2.0], 3600) + [rows([1.0, 2.0], 3600)[1]]))
    add("negative", text(rows([1.0, -2.0], 3600)))
    add("nan", text(rows([1.0], 3600) + ["2020-01-01T01:00:00Z,nan"]))
    add("inf", text(rows([1.0], 3600) + ["2020-01-01T01:00:00Z,inf"]))
    add("overflow", text(rows([1.0], 3600) + ["2020-01-01T01:00:00Z,1e999"]))
    add("bad_number", text(rows([1.0], 3600) + ["2020-01-01T01:00:00Z,abc"]))
    add("empty_number", text(rows([1.0], 3600) + ["2020-01-01T01:00:00Z,"]))
    add("three_fields", text(rows([1.0], 3600) + ["2020-01-01T01:00:00Z,1,2"]))
    add("one_field", text(rows([1.0], 3600) + ["2020-01-01T01:00:00Z"]))
    add("bad_header", text(rows([1.0], 3600), header="time,cap"))
    add("bom_header", "﻿" + text(rows([1.0], 3600)))
    add("empty_file", "")
    add("header_only", "timestamp,capacity_w\n")
    add("blank_first_line", "\n" + text(rows([1.0], 3600)))
    add("non_utc", text(["2020-01-01T00:00:00+01:00,1.0"]))
    add("bad_date", text(["2021-02-29T00:00:00Z,1.0"]))
    add("bad_hour", text(["2020-01-01T24:00:00Z,1.0"]))
    add("year_zero", text(["0000-01-01T00:00:00Z,1.0"]))
    add("garbage_ts", text(["yesterday,1.0"]))
    add("unicode_line_sep", "timestamp,capacity_w " + " ".join(rows([1.0, 2.0], 3600)))
    add("nel_line_sep", "timestamp,capacity_w\x85" + "\x85".join(rows([1.0, 2.0], 3600)))
    add("unicode_space_field", text(["2020-01-01T00:00:00Z, 1.0", "2020-01-01T01:00:00Z,2.0"]))
    add("step_zero", text(rows([1.0], 3600)), step=0)
    return out


def run(case, d: Path) -> dict:
    path = d / f"{case['name']}.csv"
    body = case["text"] if "text" in case else gen_text(case["gen"])
    path.write_bytes(body.encode("utf-8"))
    try:
        tr = load_trace(path, case["step_seconds"], gap_fill=case["gap_fill"])
    except Exception as exc:  # noqa: BLE001 - recorded verbatim
        return {"ok": False, "exc": type(exc).__name__, "msg": str(exc).replace(str(path), "{path}")}
    vals = list(tr.values)
    res = {"ok": True, "label": tr.source_label, "step_seconds": tr.step_seconds,
           "start": tr.start_time.isoformat(), "n": len(vals), "sha256": digest(vals)}
    if len(vals) <= 2000:
        res["values"] = vals
    else:
        res["head"], res["tail"] = vals[:50], vals[-50:]
    return res


def main() -> None:
    doc = {"reference": "capsim 0.1.0 trace.load_trace (pkg/src/capsim/trace.py:87-169)", "cases": []}
    with tempfile.TemporaryDirectory() as tmp:
        for c in cases():
            c = dict(c)
            c["result"] = run(c, Path(tmp))
            doc["cases"].append(c)
    OUT.write_text(json.dumps(doc, indent=None, separators=(",", ":")))
    ok = sum(c["result"]["ok"] for c in doc["cases"])
    print(f"{OUT.name}: {len(doc['cases'])} cases ({ok} load, {len(doc['cases']) - ok} raise), "
          f"{OUT.stat().st_size // 1024} KiB")


if __name__ == "__main__":
    main()
