"""Drop-in simulate() on one year of 1-min caps (527,040 steps): wall time per call and where it
goes (device evaluation vs building the tuple of StepRecords)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import datetime  # noqa: E402

import numpy as np  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402

g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
rng = np.random.default_rng(0)
caps = np.clip(np.cumsum(rng.normal(0, 4, 527040)) + 200, 0, 350)
tr = cs.PowerTrace("year", 60, datetime.datetime(2020, 1, 1), tuple(caps.tolist()))
for kind in (cs.COMBINATION, cs.BATCHING):
    cs.simulate(g, tr, kind)
    t = time.perf_counter()
    r = cs.simulate(g, tr, kind)
    dt = time.perf_counter() - t
    print(f"{kind.label}: {dt * 1e3:.0f} ms per simulate ({len(r.steps) / dt / 1e6:.2f} M steps/s), "
          f"avg {r.avg_throughput_ips:.3f}")
t = time.perf_counter()
reps = cs.simulate_many([g], [tr])
print(f"simulate_many (3 policies, summary only): {(time.perf_counter() - t) * 1e3:.0f} ms")
