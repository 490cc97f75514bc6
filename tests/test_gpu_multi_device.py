"""Single-process multi-GPU sweep through the C ABI's NCCL communicator (cs_comm_*:
ncclCommInitAll + one grouped int64 all-reduce). The box has one B200, so the communicator spans
cuda:0 alone: the reduction must be the identity and evaluate_devices must equal the plain
evaluate + sweep totals word for word; the argument checks run too."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_evaluate_devices_single_gpu_equals_plain_path():
    import torch

    import bench
    import paper_2306_12247_b200 as cs

    torch.cuda.set_device(0)
    tables = cs.Tables.stage(bench.make_grids("ten")[:3], "f32")
    caps = cs.generate_traces(777, 4096, step_seconds=60, kind="mixed", seed=2306)
    for pen in (0.0, 10.0):
        md = cs.evaluate_devices(tables, [caps], 4096, step_seconds=60, switch_penalty_s=pen)
        ref = tables.evaluate(caps, 4096, step_seconds=60, switch_penalty_s=pen)
        words = cs.sweep_words(tables, ref.agg)
        torch.cuda.synchronize()
        assert torch.equal(md.local[0].agg, ref.agg)
        assert torch.equal(md.hist.cpu(), ref.hist.cpu())
        assert np.array_equal(md.totals.words, words.cpu().numpy())
        assert md.totals.n_traces == 777
        for m in range(3):
            for p in range(3):
                assert md.totals.steps(m, p) == 777 * 4096


def test_device_comm_identity_and_checks():
    import torch

    import paper_2306_12247_b200 as cs
    from paper_2306_12247_b200 import _native as N

    comm = cs.DeviceComm([0])
    x = torch.arange(1000, dtype=torch.int64, device="cuda:0") * 3 - 7
    y = x.clone()
    comm.allreduce([y])
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    with pytest.raises(ValueError):
        comm.allreduce([y.float()])
    comm.close()
    with pytest.raises(Exception):
        cs.DeviceComm([0, 0])  # a device may appear once per communicator
    with pytest.raises(Exception):
        cs.DeviceComm([torch.cuda.device_count()])
    assert N.lib().cs_comm_destroy(None) == 0
