"""World-size-2 gloo tests of the multi-GPU host logic (shard ranges + the sweep's single
reduction of [union-bin histogram | sweep totals]). The per-shard compute is the CPU oracle
standing in for the device kernels (tests/test_gpu_multi_rank.py runs the kernels themselves)."""

from __future__ import annotations

import os
import socket
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORDS = 12


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _workload():
    import paper_2306_12247_b200 as cs

    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=2, bs_cap=16))
    rng = np.random.default_rng(21)
    caps = np.clip(np.cumsum(rng.normal(0, 9, (13, 200)), axis=1) + 150, 0, 350).astype(np.float32)
    return g, caps


def _hist_of(g, caps) -> np.ndarray:
    """Union-bin histogram of a cap block via fp32 round-up thresholds (combination rank + 1 bins)."""
    cfgs, mtl, bs, thr, pw = g.columns()
    powers = np.unique(np.array([np.float32(p) if np.float32(p) >= p else np.nextafter(np.float32(p), np.float32(np.inf))
                                 for p in pw], dtype=np.float32))
    h = np.zeros(len(powers) + 1, np.int64)
    for row in caps:
        for c in row:
            h[np.searchsorted(powers, c, side="right")] += 1
    return h


def fixed_limbs(x: float) -> list[int]:
    """csrc/sweep.cu add_fixed restated: x >= 0 as floor(x * 2^50) in four 32-bit limbs."""
    if not x > 0:
        return [0, 0, 0, 0]
    m, e = Fraction(x).numerator, Fraction(x).denominator
    n = (m << 50) // e
    return [(n >> (32 * k)) & 0xFFFFFFFF for k in range(4)]


def _words_of(g, caps, step=60, pen=10.0) -> np.ndarray:
    """cs_sweep_totals restated over the oracle's per-trace aggregates of one grid."""
    from oracle import oracle

    cfgs, mtl, bs, thr, pw = g.columns()
    og = oracle.GridArrays(np.array(mtl, np.int32), np.array(bs, np.int32), np.array(thr), np.array(pw), 60.0)
    w = np.zeros((3, WORDS), np.int64)
    for p, regime in enumerate(("batching", "multi-tenant", "combination")):
        for row in caps:
            r = oracle.simulate(og, row.astype(np.float64), regime, step, pen)
            w[p, 0] += len(row)
            w[p, 1] += r.idle_steps
            w[p, 2] += int(np.sum(r.sel[1:] != r.sel[:-1]))
            w[p, 4:8] += fixed_limbs(r.avg_throughput_ips)
            w[p, 8:12] += fixed_limbs(r.energy_proxy_wh)
    return w


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_12247_b200.shard import max_over_ranks, reduce_sweep, shard_range

    g, caps = _workload()
    lo, hi = shard_range(caps.shape[0], rank, world)
    h = _hist_of(g, caps[lo:hi])
    w = _words_of(g, caps[lo:hi])
    buf = torch.from_numpy(np.concatenate([h, w.ravel()]))
    reduce_sweep(buf)  # the single collective
    t = max_over_ranks(1.0 + rank)
    out[rank] = (buf.numpy().tolist(), t, hi - lo)
    dist.destroy_process_group()


def test_two_rank_reduction_matches_single_process():
    from paper_2306_12247_b200.shard import SweepTotals

    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    g, caps = _workload()
    h = _hist_of(g, caps)
    want = np.concatenate([h, _words_of(g, caps).ravel()]).tolist()
    assert out[0][0] == want and out[1][0] == want
    assert out[0][1] == 2.0 and out[1][1] == 2.0
    assert out[0][2] + out[1][2] == caps.shape[0]
    # the totals recombine to the exact (truncated-to-2^-50) sums of the per-trace values
    from oracle import oracle

    cfgs, mtl, bs, thr, pw = g.columns()
    og = oracle.GridArrays(np.array(mtl, np.int32), np.array(bs, np.int32), np.array(thr), np.array(pw), 60.0)
    tot = SweepTotals(np.array(out[0][0][len(h):], np.int64).reshape(3, WORDS), caps.shape[0], (g.model_name,))
    for p, regime in enumerate(("batching", "multi-tenant", "combination")):
        avgs = [oracle.simulate(og, r.astype(np.float64), regime, 60, 10.0).avg_throughput_ips for r in caps]
        exact = sum(Fraction(int(Fraction(a) * 2**50), 2**50) for a in avgs)
        assert tot.sum_avg_throughput(0, p) == exact
        assert tot.mean_throughput_ips(0, p) == float(exact / len(avgs))
        assert tot.steps(0, p) == caps.size


def test_fixed_limbs_exact():
    from paper_2306_12247_b200.shard import fixed_to_fraction

    for x in (0.0, 1e-20, 0.75, 3.0, 123.456, 2.0**70 + 2.0**20, 1234567.891):
        assert fixed_to_fraction(fixed_limbs(x)) == Fraction(int(Fraction(x) * 2**50), 2**50)


@pytest.mark.parametrize("n,world", [(10, 3), (1_000_000, 8), (7, 8)])
def test_shard_ranges_cover_exactly(n, world):
    from paper_2306_12247_b200.shard import shard_range

    spans = [shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
