"""fp64 (drop-in PowerTrace values) evaluation throughput: the f32 bench workload widened to fp64.
Usage: python tools/diag_f64.py [traces] [switch_penalty_s]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402
from paper_2306_12247_b200 import _native as N  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
PEN = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0  # switching penalty (s)
S = 10080
g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
caps32 = cs.generate_traces(T, S, step_seconds=60, kind="mixed", seed=2306)
caps = caps32.double()
del caps32
tab = cs.Tables.stage([g], "f64")
ms = []
for i in range(6):
    tab.evaluate(caps, S, step_seconds=60, switch_penalty_s=PEN)
    torch.cuda.synchronize()
    x = C.c_float()
    N.check(N.lib().cs_eval_last_kernel_ms(C.byref(x)))
    if i >= 2:
        ms.append(x.value)
m = statistics.median(ms)
print(f"f64 T={T} pen={PEN}: kernel {m:.3f} ms  {T * S / m / 1e9:.3f} Tsteps/s  {T * S * 8 / m / 1e6:.0f} GB/s plan {tab.last_plan()}")
