"""Multi-GPU sharding of independent traces (N4) — one process per GPU.

Units are independent (every (trace, grid, policy) is its own simulate() run, SPEC.md:322;
sim.py:130-188), so ranks own contiguous trace ranges and exchange nothing while computing. The
single collective is one int64 SUM all-reduce (NCCL over NVLink on B200, gloo in the CPU tests)
of ONE buffer holding

* the union-bin histogram (the global config histogram of every grid and policy), and
* the sweep totals per (grid, policy) (cs_sweep_totals): steps, idle steps, switched steps,
  violations, and the sums over traces of the average throughput (switch penalty included) and
  of the energy proxy as exact 128-bit fixed-point limbs.

Every word is an integer sum, so the reduced result is independent of the rank count and of the
reduction order: 1, 2, 4 and 8 GPUs give bit-identical sweep statistics.

    lo, hi = shard_range(T_total, rank, world)
    caps = generate_traces(hi - lo, S, step_seconds=60, first_trace_id=lo)   # keyed by global id
    sweep = evaluate_sharded(tables, caps, S, step_seconds=60)               # local agg + global stats
    sweep.totals.mean_throughput_ips(grid=0, policy="combination")
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native as N

POLICY_ORDER = ("batching", "multi-tenant", "combination")
FIXED_SHIFT = 50  # LSB of the fixed-point sums (csrc/sweep.cu)


def shard_range(n_traces: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the global trace ids owned by ``rank`` (contiguous, sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return n_traces * rank // world, n_traces * (rank + 1) // world


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def reduce_histogram(hist, group=None):
    """Sum the per-rank union-bin histograms in place (int64; exact, order-independent)."""
    dist = _dist()
    if dist is not None and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def reduce_sweep(buf, group=None):
    """The sweep's single collective: SUM all-reduce of the packed int64 [hist | totals] buffer
    (NCCL reduces it in device memory; gloo through a host copy)."""
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return buf
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        h = buf.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        buf.copy_(h)
        return buf
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Device-timed durations are reported as the max over ranks."""
    import torch

    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])


def fixed_to_fraction(limbs) -> Fraction:
    """Exact value of a four-limb fixed-point sum (csrc/sweep.cu): sum_k limb_k 2^(32k) / 2^50."""
    n = 0
    for k, v in enumerate(limbs):
        n += int(np.uint64(v)) << (32 * k)
    return Fraction(n, 1 << FIXED_SHIFT)


@dataclass(frozen=True)
class SweepTotals:
    """Per (grid, policy) statistics of a sweep over ``n_traces`` traces (all ranks).

    ``words`` is the reduced int64 [n_grids * 3, CS_SWEEP_WORDS] array of cs_sweep_totals."""

    words: np.ndarray
    n_traces: int
    model_names: tuple

    def _row(self, grid: int, policy) -> np.ndarray:
        p = POLICY_ORDER.index(policy) if isinstance(policy, str) else int(policy)
        return self.words[3 * grid + p]

    def steps(self, grid: int, policy) -> int:
        return int(self._row(grid, policy)[0])

    def idle_steps(self, grid: int, policy) -> int:
        return int(self._row(grid, policy)[1])

    def switches(self, grid: int, policy) -> int:
        return int(self._row(grid, policy)[2])

    def violations(self, grid: int, policy) -> int:
        return int(self._row(grid, policy)[3])

    def sum_avg_throughput(self, grid: int, policy) -> Fraction:
        """Exact sum over traces of each trace's avg_throughput_ips (penalty included)."""
        return fixed_to_fraction(self._row(grid, policy)[4:8])

    def sum_energy_wh(self, grid: int, policy) -> Fraction:
        return fixed_to_fraction(self._row(grid, policy)[8:12])

    def mean_throughput_ips(self, grid: int, policy) -> float:
        """Sweep mean of the per-trace average throughput (one rounding)."""
        return float(self.sum_avg_throughput(grid, policy) / self.n_traces) if self.n_traces else 0.0

    def total_energy_wh(self, grid: int, policy) -> float:
        return float(self.sum_energy_wh(grid, policy))

    def summary(self, max_grids: int | None = None) -> list[dict]:
        out = []
        for m, name in enumerate(self.model_names[:max_grids]):
            row = {"model": name}
            for p in POLICY_ORDER:
                st = self.steps(m, p)
                row[p] = {"mean_throughput_ips": self.mean_throughput_ips(m, p),
                          "idle_fraction": self.idle_steps(m, p) / st if st else 0.0,
                          "switches": self.switches(m, p), "energy_wh": self.total_energy_wh(m, p),
                          "violations": self.violations(m, p)}
            out.append(row)
        return out


def sweep_words(tables, agg, *, out=None, accumulate: bool = False, stream=None):
    """cs_sweep_totals on the device: int64 [n_grids * 3, CS_SWEEP_WORDS] from per-trace aggregates
    ``agg`` (float64 [T, M, 3, 6], EvalResult.agg)."""
    import ctypes as C

    import torch

    from .engine import _stream_ptr

    rows = tables.n_grids * 3
    if out is None:
        # (zeroed by the call unless accumulating; a fill kernel here cost C1/C2 steps 2.5 us)
        out = (torch.zeros if accumulate else torch.empty)((rows, N.CS_SWEEP_WORDS), dtype=torch.int64,
                                                           device=agg.device)
    if agg.shape[0] and (not agg.is_contiguous() or tuple(agg.shape[1:]) != (tables.n_grids, 3, 6)):
        raise ValueError("agg must be a contiguous [T, M, 3, 6] EvalResult.agg tensor")
    with torch.cuda.device(agg.device):
        N.check(N.lib().cs_sweep_totals(agg.data_ptr() if agg.shape[0] else None, agg.shape[0], rows, out.data_ptr(),
                                        N.CS_FLAG_ACCUMULATE_HIST if accumulate else 0,
                                        C.c_void_p(_stream_ptr(stream))))
    return out


@dataclass
class ShardedResult:
    local: object          # this rank's EvalResult (per-trace aggregates of its own traces)
    hist: object           # int64 [U] global union-bin histogram (all ranks), or None (grid chunks)
    totals: SweepTotals    # global per-(grid, policy) sweep statistics

    def config_histograms(self):
        return self.local.tables.config_histograms(self.hist)


def evaluate_sharded(tables, caps, n_steps: int | None = None, *, step_seconds: int, switch_penalty_s: float = 0.0,
                     n_traces_total: int | None = None, group=None, **kw) -> ShardedResult:
    """This rank's shard through the engine, then the sweep's single collective: one SUM
    all-reduce of [union-bin histogram | sweep totals] (torch.distributed; a no-op when not
    initialised or world size 1)."""
    import torch

    res = tables.evaluate(caps, n_steps, step_seconds=step_seconds, switch_penalty_s=switch_penalty_s, **kw)
    words = sweep_words(tables, res.agg)
    hist = res.hist
    U = hist.numel() if hist is not None else 0
    buf = torch.cat([hist.view(-1) if hist is not None else words.new_zeros(0), words.view(-1)])
    reduce_sweep(buf, group)
    dist = _dist()
    if n_traces_total is None:
        n = torch.tensor([caps.shape[0]], dtype=torch.int64, device=caps.device)
        n_traces_total = int(reduce_sweep(n, group)[0])
    w = buf[U:].view(-1, N.CS_SWEEP_WORDS).cpu().numpy()
    names = tuple(getattr(g, "model_name", f"grid{i}") for i, g in enumerate(tables.grids))
    return ShardedResult(res, buf[:U] if hist is not None else None, SweepTotals(w, n_traces_total, names))


# ---- one process, several GPUs: the sweep's reduction through the C ABI's NCCL communicator ----
class DeviceComm:
    """NCCL communicator over this process's devices (cs_comm_init_all: ncclCommInitAll), for
    single-process multi-GPU sweeps. ``allreduce`` sums one int64 buffer per device in place, in
    one grouped NCCL call."""

    def __init__(self, devices):
        import ctypes as C

        self.devices = [int(d) for d in devices]
        arr = (C.c_int32 * len(self.devices))(*self.devices)
        h = C.c_void_p()
        N.check(N.lib().cs_comm_init_all(len(self.devices), arr, C.byref(h)))
        self._h = h

    def allreduce(self, bufs, streams=None):
        import ctypes as C

        import torch

        if len(bufs) != len(self.devices):
            raise ValueError("one buffer per device")
        n = bufs[0].numel()
        for b, d in zip(bufs, self.devices):
            if b.dtype != torch.int64 or not b.is_contiguous() or b.device != torch.device("cuda", d) or b.numel() != n:
                raise ValueError("buffers must be contiguous int64 tensors of equal size, one on each device")
        ptrs = (C.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
        if streams is None:
            streams = [torch.cuda.current_stream(d) for d in self.devices]
        sp = (C.c_void_p * len(bufs))(*[s.cuda_stream for s in streams])
        N.check(N.lib().cs_comm_allreduce_i64(self._h, ptrs, n, sp))
        return bufs

    def close(self):
        if getattr(self, "_h", None):
            N.lib().cs_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


@dataclass
class MultiDeviceResult:
    local: list            # per-device EvalResult (each device's own traces)
    hist: object           # int64 [U] global union-bin histogram (on the first device), or None
    totals: SweepTotals    # global per-(grid, policy) sweep statistics


def evaluate_devices(tables, caps_per_device, n_steps: int | None = None, *, step_seconds: int,
                     switch_penalty_s: float = 0.0, comm: DeviceComm | None = None, **kw) -> MultiDeviceResult:
    """A sweep sharded over the GPUs of ONE process: ``caps_per_device[i]`` is device i's shard (a
    [T_i, ld] tensor on that device, e.g. ``generate_traces(..., first_trace_id=lo_i)``). Each
    device evaluates its shard on its current stream (kernels of all devices run concurrently),
    then one grouped NCCL int64 SUM all-reduce of every device's [histogram | sweep totals]."""
    import torch

    devices = [c.device.index for c in caps_per_device]
    own = comm is None
    comm = comm or DeviceComm(devices)
    try:
        results, bufs = [], []
        for caps in caps_per_device:
            with torch.cuda.device(caps.device):
                res = tables.evaluate(caps, n_steps, step_seconds=step_seconds, switch_penalty_s=switch_penalty_s,
                                      **kw)
                words = sweep_words(tables, res.agg)
                hist = res.hist
                bufs.append(torch.cat([hist.view(-1) if hist is not None else words.new_zeros(0), words.view(-1)]))
                results.append(res)
        comm.allreduce(bufs)
        U = results[0].hist.numel() if results[0].hist is not None else 0
        with torch.cuda.device(caps_per_device[0].device):
            w = bufs[0][U:].view(-1, N.CS_SWEEP_WORDS).cpu().numpy()
        names = tuple(getattr(g, "model_name", f"grid{i}") for i, g in enumerate(tables.grids))
        n_total = sum(int(c.shape[0]) for c in caps_per_device)
        return MultiDeviceResult(results, bufs[0][:U] if U else None, SweepTotals(w, n_total, names))
    finally:
        if own:
            comm.close()
