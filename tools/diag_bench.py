"""Kernel-only timing of eval_kernel variants (diagnostic builds produce WRONG results; never
used for a reported number). Usage: CAPSIM_B200_LIB=... python tools/diag_bench.py [traces]"""

import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402
from paper_2306_12247_b200 import _native as N  # noqa: E402
import ctypes as C  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
kind = sys.argv[2] if len(sys.argv) > 2 else "mixed"
S = 10080
g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
tab = cs.Tables.stage([g], "f32")
caps = cs.generate_traces(T, S, step_seconds=60, kind=kind, seed=2306)
torch.cuda.synchronize()
ms = []
for i in range(13):
    tab.evaluate(caps, S, step_seconds=60)
    torch.cuda.synchronize()
    x = C.c_float()
    N.check(N.lib().cs_eval_last_kernel_ms(C.byref(x)))
    if i >= 3:
        ms.append(x.value)
m = statistics.median(ms)
print(f"{N.LIB_PATH.name} {kind}: kernel {m:.3f} ms  {T*S/m/1e9:.1f} Gsteps/s  {T*S*4/m/1e6:.0f} GB/s")
