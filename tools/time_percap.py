"""Per-call latency of the per-cap drop-in API (select_config, PolicyIndex.select, feasible_set)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402

g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
caps = np.random.default_rng(0).uniform(0, 360, 2000).tolist()
idx = cs.PolicyIndex(g, cs.COMBINATION)
for name, fn in (("PolicyIndex.select", lambda c: idx.select(c)),
                 ("select_config", lambda c: cs.select_config(g, cs.BATCHING, c)),
                 ("feasible_set", lambda c: cs.feasible_set(g, cs.MULTI_TENANT, c))):
    for c in caps[:20]:
        fn(c)
    t = time.perf_counter()
    for c in caps:
        fn(c)
    dt = (time.perf_counter() - t) / len(caps)
    print(f"{name}: {dt * 1e6:.1f} us per call")
t = time.perf_counter()
idx.select_many(caps)
print(f"PolicyIndex.select_many (2000 caps, one launch): {(time.perf_counter() - t) * 1e6:.0f} us")
