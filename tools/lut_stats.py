"""Diagnostic: how often do synthetic caps hit multi-threshold LUT buckets (the redirect path)
for each level-1 shift? Usage: python tools/lut_stats.py [traces] [kind]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_12247_b200 as cs  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
kind = sys.argv[2] if len(sys.argv) > 2 else "mixed"
S = 10080
g = bench.make_grids("mobilenet")
caps = cs.generate_traces(T, S, step_seconds=60, kind=kind, seed=2306)[:, :S].cpu().numpy()
bits = caps.view(np.uint32).astype(np.int64)
pw = np.array(g[0].columns()[4])
thr = np.unique(np.array([np.nextafter(np.float32(p), np.float32(np.inf)) if np.float32(p) < p else np.float32(p)
                          for p in pw], np.float32).view(np.uint32).astype(np.int64))
print("caps: frac == max", float((caps == caps.max()).mean()), "max", caps.max(), "frac >= 349", float((caps >= 349).mean()),
      "frac 0", float((caps <= 0).mean()))
for s in range(8, 14):
    kb = thr >> s
    uk, cnt = np.unique(kb, return_counts=True)
    multi = set(uk[cnt >= 2].tolist())
    ck = bits >> s
    hit = np.isin(ck, list(multi))
    w = hit.reshape(T, -1)[:, : (S // 128) * 128].reshape(T, -1, 128).any(-1)
    print(f"s={s} level1~{(thr[-1] >> s) - (thr[0] >> s) + 3} multi-buckets={len(multi)} cap-frac={hit.mean():.4f} "
          f"warp-chunk-frac={w.mean():.4f}")
