"""World-size-2 gloo test of the multi-GPU host logic (shard ranges + the single histogram
reduction). The per-shard compute is the CPU oracle standing in for the device kernel."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


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
    """Union-bin histogram of a cap block via the oracle (combination rank + 1 bins)."""
    from oracle import oracle

    cfgs, mtl, bs, thr, pw = g.columns()
    ga = oracle.GridArrays(np.array(mtl, np.int32), np.array(bs, np.int32), np.array(thr), np.array(pw))
    idx = oracle.Index(ga, "combination")
    powers = np.unique(np.array([np.float32(p) if np.float32(p) >= p else np.nextafter(np.float32(p), np.float32(np.inf))
                                 for p in pw], dtype=np.float32))
    h = np.zeros(len(powers) + 1, np.int64)
    for row in caps:
        for c in row:
            h[np.searchsorted(powers, c, side="right")] += 1
    del idx
    return h


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_12247_b200.shard import max_over_ranks, reduce_histogram, shard_range

    g, caps = _workload()
    lo, hi = shard_range(caps.shape[0], rank, world)
    h = torch.from_numpy(_hist_of(g, caps[lo:hi]))
    reduce_histogram(h)
    t = max_over_ranks(1.0 + rank)
    out[rank] = (h.numpy().tolist(), t, hi - lo)
    dist.destroy_process_group()


def test_two_rank_reduction_matches_single_process():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    g, caps = _workload()
    want = _hist_of(g, caps).tolist()
    assert out[0][0] == want and out[1][0] == want
    assert out[0][1] == 2.0 and out[1][1] == 2.0
    assert out[0][2] + out[1][2] == caps.shape[0]


@pytest.mark.parametrize("n,world", [(10, 3), (1_000_000, 8), (7, 8)])
def test_shard_ranges_cover_exactly(n, world):
    from paper_2306_12247_b200.shard import shard_range

    spans = [shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
