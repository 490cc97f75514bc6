"""Kernel-only timing of one BASELINE config's eval launch (the bench's workload, fewer traces):
    python tools/diag_config.py C5 [traces] [kind]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_12247_b200 as cs  # noqa: E402
from paper_2306_12247_b200 import _native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = bench.CONFIGS[name]
T = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["traces"]
kind = sys.argv[3] if len(sys.argv) > 3 else cfg["kind"]
S = cfg["steps"]
tab = cs.Tables.stage(bench.make_grids(cfg["grids"]), "f32")
caps = cs.generate_traces(T, S, step_seconds=cfg["step_seconds"], kind=kind, seed=2306)
torch.cuda.synchronize()
ms = []
for i in range(8):
    tab.evaluate(caps, S, step_seconds=cfg["step_seconds"], switch_penalty_s=cfg["penalty"])
    torch.cuda.synchronize()
    x = C.c_float()
    N.check(N.lib().cs_eval_last_kernel_ms(C.byref(x)))
    if i >= 2:
        ms.append(x.value)
m = statistics.median(ms)
print(f"{name} {kind} T={T}: kernel {m:.3f} ms  {T * S / m / 1e9:.3f} Tsteps/s  {T * S * 4 / m / 1e6:.0f} GB/s "
      f"plan {tab.last_plan()}")
