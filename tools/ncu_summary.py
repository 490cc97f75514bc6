"""Summarise an ncu report of eval_kernel into the numbers DESIGN.md / bench.py cite.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --traces 100000 --steps 10080 \
        --out profiles/r01/ncu_eval_kernel.json [--traffic-key C4:mixed:f32]

Writes a JSON summary (duration, DRAM bytes, throughput %, occupancy, issue, L1TEX/smem
pipe utilisation, instructions per timestep, stall mix) and, with --traffic-key, records the
measured DRAM bytes per timestep in profiles/ncu_traffic.json so bench.py can report
roofline.traffic scaled to its launch.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "l1tex_lsu_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
    "warp_instructions": ("smsp__inst_executed.sum", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "block_size": ("launch__block_size", 1.0),
    "grid_size": ("launch__grid_size", 1.0),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "msecond": 1.0, "usecond": 1e-3,
              "nsecond": 1e-6, "ms": 1.0, "us": 1e-3, "ns": 1e-6}


def raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, zip(r, units))) for r in rows[2:]]


def summarise(rec: dict, timesteps: int) -> dict:
    s = {}
    for name, (metric, _) in KEYS.items():
        if metric not in rec:
            continue
        val, unit = rec[metric]
        try:
            v = float(val.replace(",", ""))
        except ValueError:
            continue
        if name.startswith("dram_") and name.endswith("_bytes"):
            v *= UNIT_SCALE.get(unit, 1)
        if name == "duration_ms":
            v *= UNIT_SCALE.get(unit, 1)
        s[name] = v
    s["kernel"] = rec.get("Kernel Name", ("?",))[0]
    if timesteps:
        s["timesteps"] = timesteps
        if "warp_instructions" in s:
            s["thread_instructions_per_timestep"] = s["warp_instructions"] * 32 / timesteps
        if "dram_read_bytes" in s:
            s["dram_bytes_per_timestep"] = (s["dram_read_bytes"] + s.get("dram_write_bytes", 0.0)) / timesteps
        if "duration_ms" in s and "dram_read_bytes" in s:
            s["achieved_dram_gbs_cold"] = (s["dram_read_bytes"] + s.get("dram_write_bytes", 0.0)) / (
                s["duration_ms"] * 1e-3) / 1e9
    return s


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--traces", type=int, default=0)
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-key", default=None)
    a = ap.parse_args()
    recs = [r for r in raw(a.report) if "eval_kernel" in r.get("Kernel Name", ("",))[0]]
    if not recs:
        raise SystemExit("no eval_kernel in report")
    summ = summarise(recs[0], a.traces * a.steps)
    Path(a.out).write_text(json.dumps(summ, indent=2) + "\n")
    print(json.dumps(summ, indent=2))
    if a.traffic_key and "dram_bytes_per_timestep" in summ:
        p = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
        doc = json.loads(p.read_text()) if p.exists() else {}
        doc[a.traffic_key] = {"dram_bytes_per_timestep": summ["dram_bytes_per_timestep"], "source": a.out,
                              "kernel": summ.get("kernel", "eval_kernel")}
        p.write_text(json.dumps(doc, indent=2) + "\n")


if __name__ == "__main__":
    main()
