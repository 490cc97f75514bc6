"""Top instructions for one stall reason from an ncu report's SASS source page:
    python tools/sass_stall.py report.ncu-rep stall_long_sb [timesteps] [top]"""
import csv
import io
import subprocess
import sys

rep, col = sys.argv[1], sys.argv[2]
steps = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
ix = {h: i for i, h in enumerate(rows[0])}
data = rows[1:]
tot = sum(float(r[ix[col]] or 0) for r in data)
print(f"{col}: {tot:.0f} samples")
for r in sorted(data, key=lambda r: -float(r[ix[col]] or 0))[:top]:
    t = float(r[ix["Thread Instructions Executed"]] or 0) / steps
    print(f"{r[ix['Address']][-5:]} {100 * float(r[ix[col]] or 0) / max(tot, 1):5.1f}% rate {t:6.3f}  {r[ix['Source']].strip()}")
