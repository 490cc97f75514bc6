"""Ingestion fast path throughput: CSV rows/s of the native parser
(csrc/ingest.cpp via load_traces / load_trace_matrix) next to the reference-rules loader in
Python (trace.py's restatement of trace.py:87-169, i.e. the reference's own algorithm).

    python tools/bench_ingest.py [n_files] [rows_per_file] [--out profiles/r01/ingest.json]
"""

from __future__ import annotations

import json
import os
import random
import sys
import tempfile
import time
from datetime import datetime, timedelta, timezone
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2306_12247_b200 as cs  # noqa: E402
from paper_2306_12247_b200 import trace as T  # noqa: E402


def main() -> None:
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n_files = int(args[0]) if args else 256
    n_rows = int(args[1]) if len(args) > 1 else 10_080
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    rng = random.Random(1)
    t0 = datetime(2020, 1, 1, tzinfo=timezone.utc)
    with tempfile.TemporaryDirectory() as d:
        paths = []
        for i in range(n_files):
            p = Path(d) / f"trace{i:05d}.csv"
            lines = ["timestamp,capacity_w"]
            for k in range(n_rows):
                lines.append(f"{(t0 + timedelta(minutes=k)).strftime('%Y-%m-%dT%H:%M:%SZ')},{rng.uniform(0, 350):.6f}")
            p.write_text("\n".join(lines) + "\n")
            paths.append(p)
        nbytes = sum(p.stat().st_size for p in paths)
        cores = len(os.sched_getaffinity(0))
        res = {"files": n_files, "rows_per_file": n_rows, "bytes": nbytes, "host_threads": cores}
        # native, all threads: PowerTrace objects (tuple values, the drop-in API)
        t = time.perf_counter()
        trs = cs.load_traces(paths, 60)
        res["native_load_traces_rows_per_s"] = n_files * n_rows / (time.perf_counter() - t)
        # native, all threads, straight into the engine's [T, ld] matrix (no Python objects)
        t = time.perf_counter()
        m = cs.load_trace_matrix(paths, 60, dtype="f64")
        dt = time.perf_counter() - t
        res["native_matrix_rows_per_s"] = n_files * n_rows / dt
        res["native_matrix_MB_per_s"] = nbytes / dt / 1e6
        # native, one thread
        t = time.perf_counter()
        cs.load_trace_matrix(paths[:16], 60, dtype="f64", n_threads=1)
        res["native_matrix_1thread_rows_per_s"] = 16 * n_rows / (time.perf_counter() - t)
        # reference rules in Python (one thread), a bounded sample
        k = min(8, n_files)
        t = time.perf_counter()
        ref = [T._load_trace_rules(p, 60, False, p.stem) for p in paths[:k]]
        res["python_rules_1thread_rows_per_s"] = k * n_rows / (time.perf_counter() - t)
        assert all(a == b for a, b in zip(ref, trs[:k]))
        assert float(m.values[0, 5]) == trs[0].values[5]
    res["speedup_matrix_vs_python_1thread"] = res["native_matrix_rows_per_s"] / res["python_rules_1thread_rows_per_s"]
    line = json.dumps(res)
    print(line)
    if out:
        Path(out).write_text(line + "\n")


if __name__ == "__main__":
    main()
