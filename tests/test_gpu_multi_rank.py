"""The sharded sweep with the real kernels: two ranks on cuda:0 (gloo for the collective; the
driver's box has one GPU) against the single-process run. Per-trace aggregates, the reduced
union-bin histogram and the sweep totals must equal N=1 (integer words bit-identical), and the
totals must equal the exact sums of the per-trace values (cs_sweep_totals restated in Python)."""

from __future__ import annotations

import hashlib
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T_TOTAL, S, STEP, PEN = 3001, 2048, 60, 10.0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank: int, world: int):
    import torch

    import bench
    import paper_2306_12247_b200 as cs

    torch.cuda.set_device(0)
    tables = cs.Tables.stage(bench.make_grids("ten")[:3], "f32")
    lo, hi = cs.shard_range(T_TOTAL, rank, world)
    caps = cs.generate_traces(hi - lo, S, step_seconds=STEP, kind="mixed", seed=2306, first_trace_id=lo)
    sw = cs.evaluate_sharded(tables, caps, S, step_seconds=STEP, switch_penalty_s=PEN)
    torch.cuda.synchronize()
    hist = sw.hist.cpu().numpy()
    return (hashlib.sha256(hist.astype("<i8").tobytes()).hexdigest(), sw.totals.words.tolist(),
            sw.local.agg.cpu().numpy(), lo, sw.totals.n_traces)


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = _run(rank, world)
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one(cuda_ok):
    import torch.multiprocessing as mp

    single = _run(0, 1)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in (0, 1):
        assert out[r][0] == single[0]          # reduced histogram
        assert out[r][1] == single[1]          # sweep totals (integer words)
        assert out[r][4] == T_TOTAL
    agg2 = np.concatenate([out[0][2], out[1][2]])
    assert agg2.shape == single[2].shape
    same = np.mean(agg2.view(np.int64) == single[2].view(np.int64))
    assert same > 0.999, same  # per-trace aggregates (sums are fsum-exact in >= 99.9 % of cases)
    assert np.allclose(agg2, single[2], rtol=1e-12, atol=0)


def test_sweep_totals_are_exact_sums(cuda_ok):
    """cs_sweep_totals words == the integer sums restated on the host (tests/test_multi_rank.py)."""
    import torch

    import paper_2306_12247_b200 as cs
    from test_multi_rank import fixed_limbs

    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=4, bs_cap=128))
    caps = cs.generate_traces(5000, 1440, step_seconds=60, kind="mixed", seed=1)
    t = cs.Tables.stage([g], "f32")
    res = t.evaluate(caps, 1440, step_seconds=60, switch_penalty_s=30.0)
    words = cs.sweep_words(t, res.agg).cpu().numpy()
    agg = res.agg.cpu().numpy()
    ints = agg.view(np.int64)
    for p in range(3):
        w = np.zeros(12, np.int64)
        w[0] = ints[:, 0, p, 5].sum()
        w[1] = ints[:, 0, p, 2].sum()
        w[2] = ints[:, 0, p, 3].sum()
        w[3] = ints[:, 0, p, 4].sum()
        for x in agg[:, 0, p, 0]:
            w[4:8] += fixed_limbs(float(x))
        for x in agg[:, 0, p, 1]:
            w[8:12] += fixed_limbs(float(x))
        assert np.array_equal(words[p], w), p
    # accumulate mode adds on top (peer / multi-launch accumulation)
    again = cs.sweep_words(t, res.agg, out=torch.from_numpy(words).cuda(), accumulate=True).cpu().numpy()
    assert np.array_equal(again, 2 * words)
