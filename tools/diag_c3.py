"""Kernel-only timing of the C3 shape (ten grids, 1-s steps) on a reduced trace count, for A/B and
ncu captures of eval_kernel variants. Usage: [CAPSIM_B200_LIB=...] python tools/diag_c3.py [traces] [kind] [reps]"""

import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import ctypes as C  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_12247_b200 as cs  # noqa: E402
from paper_2306_12247_b200 import _native as N  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
kind = sys.argv[2] if len(sys.argv) > 2 else "mixed"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
S = 604_800
tab = cs.Tables.stage(bench.make_grids("ten"), "f32")
caps = cs.generate_traces(T, S, step_seconds=1, kind=kind, seed=2306)
torch.cuda.synchronize()
ms = []
for i in range(reps + 2):
    tab.evaluate(caps, S, step_seconds=1, check_violations=True)
    torch.cuda.synchronize()
    x = C.c_float()
    N.check(N.lib().cs_eval_last_kernel_ms(C.byref(x)))
    if i >= 2:
        ms.append(x.value)
m = statistics.median(ms)
print(f"{N.LIB_PATH.name} C3 {kind} T={T}: kernel {m:.3f} ms  {T * S / m / 1e6:.3f} Tsteps/s  {T * S * 4 / m / 1e6:.0f} GB/s")
print("plan", tab.last_plan())
