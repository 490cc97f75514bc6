"""Kernel-only timing of the C5 penalty path (fine 8x512 grid, 10 s switching penalty) for A/B
of eval_kernel variants. Usage: [CAPSIM_B200_LIB=...] python tools/diag_c5.py [traces] [kind] [reps]"""

import hashlib
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import ctypes as C  # noqa: E402

import torch  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402
from paper_2306_12247_b200 import _native as N  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
kind = sys.argv[2] if len(sys.argv) > 2 else "mixed"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
S = 10080
g = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0, model_name="fine-8x512"))
tab = cs.Tables.stage([g], "f32")
caps = cs.generate_traces(T, S, step_seconds=60, kind=kind, seed=2306)
torch.cuda.synchronize()
ms = []
res = None
for i in range(reps + 3):
    res = tab.evaluate(caps, S, step_seconds=60, switch_penalty_s=10.0, check_violations=True)
    torch.cuda.synchronize()
    x = C.c_float()
    N.check(N.lib().cs_eval_last_kernel_ms(C.byref(x)))
    if i >= 3:
        ms.append(x.value)
m = statistics.median(ms)
print(f"{N.LIB_PATH.name} {kind} T={T}: kernel {m:.3f} ms  {T*S/m/1e9:.1f} Gsteps/s  {T*S*4/m/1e6:.0f} GB/s")
print("plan", tab.last_plan())
print("agg sha", hashlib.sha256(res.agg.cpu().numpy().tobytes()).hexdigest()[:16])
