"""PK parity probe: per-field mismatch counts vs the oracle on C5-shaped traces.
    python tools/diag_pk_parity.py [T] [S] [kind] [pen]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_12247_b200 as cs  # noqa: E402
from oracle import oracle  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
S = int(sys.argv[2]) if len(sys.argv) > 2 else 10080
kind = sys.argv[3] if len(sys.argv) > 3 else "mixed"
pen = float(sys.argv[4]) if len(sys.argv) > 4 else 10.0
grids = bench.make_grids("fine")
og = bench.oracle_grids(grids)
tab = cs.Tables.stage(grids, "f32")
caps = cs.generate_traces(T, S, step_seconds=60, kind=kind, seed=2306)
res = tab.evaluate(caps, S, step_seconds=60, switch_penalty_s=pen, check_violations=True)
torch.cuda.synchronize()
print("plan", tab.last_plan())
cn = caps[:, :S].cpu().numpy()
avg, idle, en, _ = oracle.simulate_batch(og, cn, 60, pen, n_threads=16)
ga, gi, ge = res.avg_throughput_ips.cpu().numpy(), res.idle_steps.cpu().numpy(), res.energy_proxy_wh.cpu().numpy()
print("idle mismatches", int(np.sum(gi != idle)), "avg rel>1e-6", int(np.sum(~np.isclose(ga, avg, rtol=1e-6, atol=0))),
      "energy rel>1e-6", int(np.sum(~np.isclose(ge, en, rtol=1e-6, atol=0))), "viol", int(res.violations.sum()))
bad = np.argwhere(~np.isclose(ga, avg, rtol=1e-6, atol=0) | (gi != idle) | ~np.isclose(ge, en, rtol=1e-6, atol=0))
for t, m, p in bad[:8]:
    r = oracle.simulate(og[0], cn[t].astype(np.float64), ["batching", "multi-tenant", "combination"][p], 60, pen)
    sw = int(np.sum(r.sel[1:] != r.sel[:-1]))
    print(f"t={t} p={p}: avg {ga[t, m, p]!r} vs {avg[t, m, p]!r}; idle {gi[t, m, p]} vs {idle[t, m, p]}; "
          f"energy {ge[t, m, p]!r} vs {en[t, m, p]!r}; switches {int(res.switches[t, m, p])} vs {sw}")
