"""The controller-replay restatement (oracle ora_replay, incl. CPython's MT19937 noise stream)
pinned to the reference's own replays (tests/golden/controller_golden.json)."""

from __future__ import annotations

import random

import numpy as np

from conftest import golden, grid_arrays
from oracle import oracle


def _sel_doc(grid_doc, sel):
    idx, cnt = sel
    if idx < 0:
        return None
    m, b, t, p = grid_doc["entries"][idx]
    return [m, b, t, p, cnt]


def test_mt19937_matches_cpython():
    for seed in (0, 1, 5, 123456789, 2**40 + 7, -77, 2**70 + 3):
        import ctypes as C

        st = (C.c_uint32 * 625)()
        key = oracle.seed_key(seed)
        L = oracle.lib()
        L.ora_mt_seed.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(dtype=np.uint32), C.c_int]
        L.ora_mt_random.argtypes = [C.c_void_p]
        L.ora_mt_random.restype = C.c_double
        L.ora_mt_seed(C.addressof(st), key, key.shape[0])
        ref = random.Random(seed)
        for _ in range(2000):
            assert L.ora_mt_random(C.addressof(st)) == ref.random()


def test_replay_matches_reference():
    for case in golden("controller_golden.json")["cases"]:
        gdoc = case["grid"]
        g = grid_arrays(gdoc)
        init = -1
        if case["initial"] is not None:
            init = [i for i, e in enumerate(gdoc["entries"]) if [e[0], e[1]] == list(case["initial"])][0]
        res = oracle.replay(g, case["caps"], case["mode"], case["window_k"], init, case["noise_pct"], case["seed"])
        assert res.violations == case["violations"], case["name"]
        assert res.reconfigs == case["reconfigs"], case["name"]
        assert res.avg_throughput_ips == case["avg_throughput_ips"], case["name"]
        events, sels = oracle.replay_events(res, case["caps"], g.pw)
        assert events == case["events"], case["name"]
        assert [_sel_doc(gdoc, s) for s in sels] == case["selections"], case["name"]
