"""Throughput of the §8(f) widenings next to the reference algorithm on the host (the C oracle
port, all host threads): controller replay (replay_many, reactive / proactive with 2 % sensor
noise) and the sampling selector (simulate_many with sampling_policy(m, r)).

    python tools/bench_aux.py [traces] [steps]
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = int(sys.argv[2]) if len(sys.argv) > 2 else 8784
g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
rng = np.random.default_rng(7)
caps = np.clip(np.cumsum(rng.normal(0, 6.0, (T, S)), axis=1) + rng.uniform(50, 300, (T, 1)), 0, 350)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


for name, mode in (("reactive", cs.REACTIVE), ("proactive(k=3)", cs.proactive(3))):
    dt = timed(lambda: cs.replay_many(g, caps, mode, noise_pct=2.0, seed=1))
    print(f"controller {name}: {T}x{S} in {dt * 1e3:.1f} ms -> {T * S / dt / 1e9:.2f} G steps/s (host->device incl.)")

traces = [cs.PowerTrace(f"t{i}", 3600, __import__("datetime").datetime(2020, 1, 1), tuple(caps[i].tolist()))
          for i in range(min(T, 256))]
for m, r in ((8, 2), (64, 2)):
    kind = cs.sampling_policy(m, r)
    dt = timed(lambda: cs.simulate_many([g], traces, kinds=[kind]), reps=1)
    n = len(traces) * S
    print(f"sampling(m={m},r={r}): {len(traces)}x{S} in {dt * 1e3:.1f} ms -> {n / dt / 1e6:.1f} M steps/s")

# the sampling kernel alone (per-step entries on the device, no host aggregation)
tables = cs.Tables.stage([g], "f64")
cd = torch.from_numpy(np.ascontiguousarray(caps[:256])).cuda()
for m in (8, 64):
    dt = timed(lambda: tables.select_sampling(0, cd, S, m, 2, 0))
    print(f"sampling kernel (m={m},r=2): 256x{S} in {dt * 1e3:.1f} ms -> {256 * S / dt / 1e6:.1f} M steps/s")
