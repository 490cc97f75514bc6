import sys, time, torch
sys.path.insert(0, ".")
import bench, paper_2306_12247_b200 as cs
cfg = bench.CONFIGS["C3"]
tab = cs.Tables.stage(bench.make_grids("ten"), "f32")
caps = cs.generate_traces(10000, cfg["steps"], step_seconds=1, kind="mixed", seed=2306)
kw = dict(step_seconds=1, switch_penalty_s=0.0, check_violations=True, want_hist=True)
g = tab.capture(caps, cfg["steps"], sweep_totals=True, **kw)
g2 = tab.capture(caps, cfg["steps"], sweep_totals=False, **kw)
def timeit(f, n=10):
    for _ in range(2): f()
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n
print("evaluate()       ", timeit(lambda: tab.evaluate(caps, cfg["steps"], **kw)))
print("graph+sweep      ", timeit(g.replay))
print("graph no sweep   ", timeit(g2.replay))
print("evaluate()       ", timeit(lambda: tab.evaluate(caps, cfg["steps"], **kw)))
