"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
batched eval (segment and per-bin epilogues, penalty, per-step output, split traces + finalize,
fp64), per-cap queries, controller replay, sampling, entry aggregation, the generator."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import datetime  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_12247_b200 as cs  # noqa: E402

g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=32))
g2 = cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=16, t_max_ips=3000.0, model_name="b"))
caps = cs.generate_traces(64, 2000, step_seconds=60, kind="mixed", seed=3)
t32 = cs.Tables.stage([g, g2], "f32")
t32.evaluate(caps, 2000, step_seconds=60)
t32.evaluate(caps, 2000, step_seconds=60, switch_penalty_s=20.0, per_step=True)
t32.evaluate(caps[:1], 2000, step_seconds=60)  # tiny plan
big = cs.generate_traces(2, 300000, step_seconds=60, kind="iid", seed=4)
t32.evaluate(big, 300000, step_seconds=60, switch_penalty_s=10.0)  # split traces + finalize
t1 = cs.Tables.stage([g], "f32")
many = cs.generate_traces(420, 10080, step_seconds=60, kind="mixed", seed=5)
t1.evaluate(many, 10080, step_seconds=60)  # big LUT + per-bin epilogue
# fine grid (2,038 bins): multi-warp worker groups, several traces each (warp 0 finishes a trace's
# records while the group's other warps start the next)
fine = cs.synthesize_grid(cs.SynthParams(mtl_cap=8, bs_cap=512, mem_model_mb=3072.0, model_name="fine"))
tf = cs.Tables.stage([fine], "f32")
fc = cs.generate_traces(4000, 256, step_seconds=60, kind="mixed", seed=6)
tf.evaluate(fc, 256, step_seconds=60, switch_penalty_s=10.0)
tf.evaluate(fc, 256, step_seconds=60)
# packed-penalty kernel (PK): several 512-step blocks per trace, ragged tail, idle fast path
fc2 = cs.generate_traces(2400, 1203, step_seconds=60, kind="mixed", seed=7)
tf.evaluate(fc2, 1203, step_seconds=60, switch_penalty_s=10.0, check_violations=True)
assert tf.last_plan()["epilogue"] in (3, 4), tf.last_plan()
cs.Tables.stage([fine], "f64").evaluate(fc[:600].double(), 256, step_seconds=60, switch_penalty_s=10.0)
# ten grids (5,055 union thresholds): redirect-heavy LUT (per-lane predicated sub-table loads)
import bench  # noqa: E402

# ten grids, long traces (>= 4M timesteps, >= 64 steps per union bin): the huge LUT staged next to
# 8-warp groups, each trace's histogram folded straight into global memory
tten = cs.Tables.stage(bench.make_grids("ten"), "f32")
lt = cs.generate_traces(7, 604800, step_seconds=1, kind="mixed", seed=8)
tten.evaluate(lt, 604800, step_seconds=1)
assert tten.last_plan()["lut_shift"] == tten.info.lut_huge_shift, tten.last_plan()

cs.Tables.stage(bench.make_grids("ten"), "f32").evaluate(caps, 2000, step_seconds=60)
t64 = cs.Tables.stage([g], "f64")
t64.evaluate(caps.double(), 2000, step_seconds=60, switch_penalty_s=5.0)
idx = cs.PolicyIndex(g, cs.COMBINATION)
idx.select(150.0)
cs.select_config(g, cs.BATCHING, 200.0)
cs.feasible_set(g, cs.MULTI_TENANT, 200.0)
vals = np.clip(np.cumsum(np.random.default_rng(0).normal(0, 20, (8, 500)), axis=1) + 150, 0, 350)
cs.replay_many(g, vals, cs.proactive(3), noise_pct=2.0, seed=1)
trs = [cs.PowerTrace(f"t{i}", 60, datetime.datetime(2020, 1, 1), tuple(v.tolist())) for i, v in enumerate(vals)]
cs.simulate_many([g], trs, kinds=[cs.sampling_policy(4, 1), cs.COMBINATION], switch_penalty_s=30.0)
# C-ABI hardening cases (tests/test_gpu_abi_hardening.py): padded host rows copied 2-D into the
# engine's pitch, an engine reused with more grids, a zero-trace launch
host = torch.zeros((37, 1077), dtype=torch.float32).pin_memory()
host[:, :1000] = caps[:37, :1000].cpu()
eng = cs.HostEngine(cs.Tables.stage([g], "f32"), chunk_traces=8, n_steps_max=1000)
eng.evaluate(host[:, :1000], 1000, step_seconds=60)
eng.evaluate(host, 1000, step_seconds=60)
eng.tables = t32
eng.evaluate(host, 1000, step_seconds=60, switch_penalty_s=5.0)
t32.evaluate(torch.zeros((0, 128), dtype=torch.float32, device="cuda"), 100, step_seconds=60)
torch.cuda.synchronize()
print("sanitize workload done")
