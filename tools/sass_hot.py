"""Summarise an ncu report's SASS source page: instruction mix (thread instructions by opcode),
warp-stall samples by opcode, and the hottest instructions. Usage:
    python tools/sass_hot.py report.ncu-rep [timesteps] [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
ti = Counter()
st = Counter()
tot_ti = tot_st = 0
hot = []
for r in data:
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    t = float(r[ix["Thread Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ti[op] += t
    st[op] += s
    tot_ti += t
    tot_st += s
    hot.append((s, t, r[ix["Address"]][-5:], src))
print(f"total thread instr {tot_ti:.3e}" + (f" = {tot_ti / steps:.2f} / timestep" if steps else ""), f"samples {tot_st:.0f}")
print("opcode              thr-instr/step  %instr  %stall")
for op, t in ti.most_common(30):
    print(f"{op:18s} {t / steps if steps else t:10.3f} {100 * t / tot_ti:7.1f} {100 * st[op] / max(tot_st, 1):7.1f}")
print("--- hottest by stall samples")
for s, t, a, src in sorted(hot, reverse=True)[:top]:
    print(f"{a} {100 * s / max(tot_st, 1):5.1f}% {t / steps if steps else t:8.3f}  {src}")
# instruction mass grouped by per-timestep execution rate (instructions of one loop share a rate)
print("--- mass by execution rate (thread instr / timestep of one instruction)")
buck = Counter()
bs = Counter()
nins = Counter()
for s, t, a, src in hot:
    if steps and t:
        k = round(t / steps, 3)
        buck[k] += t / steps
        bs[k] += s
        nins[k] += 1
for k, m in sorted(buck.items(), key=lambda kv: -kv[1])[:25]:
    print(f"rate {k:8.3f}: {nins[k]:5d} instrs, {m:7.2f} thr-instr/step, {100 * bs[k] / max(tot_st, 1):5.1f}% stalls")
