"""Diagnostic: kernel per-step union bins vs the host LUT restatement (cs_tables_lookup_host) on
>= 4M timesteps (the launch size that stages the finer LUT and the bin epilogue)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402

g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
t = cs.Tables.stage([g], "f32")
T, S = 420, 10080
for kind in ("mixed", "iid"):
    caps = cs.generate_traces(T, S, step_seconds=60, kind=kind, seed=5)
    r = t.evaluate(caps, S, step_seconds=60, per_step=True)
    torch.cuda.synchronize()
    got = r.step_bins[:, :S].cpu().numpy().view(np.uint16).astype(np.int64).ravel()
    c = caps[:, :S].cpu().numpy().ravel()
    want = t.lookup_host(c).astype(np.int64)
    bad = np.nonzero(got != want)[0]
    print(kind, "mismatches", bad.size, "of", got.size)
    for i in bad[:12]:
        print(f"  cap {c[i]!r} bits {c[i:i+1].view(np.uint32)[0]:#x} kernel {got[i]} host {want[i]}")
