"""Device engine: staged policy tables (N1) and batched evaluation (N2+N3) over torch buffers.

This is the layer the drop-in functions (policy.py, sim.py) and the benchmark call. PyTorch is
used for device memory and streams only; all compute runs in libcapsim_b200.so kernels.

    tables = Tables.stage([grid_a, grid_b], cap_dtype="f32")
    res = tables.evaluate(caps_dev, n_steps=S, step_seconds=60)      # caps_dev: [T, ld] cuda
    res.avg_throughput_ips   # torch.float64 [T, M, 3]  (policy order: batching, multi-tenant, combination)
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import ValidationError

POLICY_ORDER = ("batching", "multi-tenant", "combination")
_DTYPES = {"f32": N.CS_CAP_F32, "f64": N.CS_CAP_F64}


def _torch():
    import torch

    return torch


def require_device():
    """The engine has no CPU path: fail loudly when no CUDA device is visible."""
    torch = _torch()
    if not torch.cuda.is_available():
        raise N.NativeLibraryError("no CUDA device visible: libcapsim_b200 runs on B200 (sm_100a) only")
    N.lib()
    return torch.device("cuda", torch.cuda.current_device())


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def grid_arrays(grid):
    """(configs, mtl int32, bs int32, thr f64, pw f64) of a ProfileGrid in its entry order."""
    cfgs, mtl, bs, thr, pw = grid.columns()
    return (cfgs, np.ascontiguousarray(mtl, dtype=np.int32), np.ascontiguousarray(bs, dtype=np.int32),
            np.ascontiguousarray(thr, dtype=np.float64), np.ascontiguousarray(pw, dtype=np.float64))


@dataclass
class GridBins:
    """Host decode table of one grid: per policy, the selected entry (-1 = idle) and the
    feasible_count for every grid bin (policy.py:139-148)."""

    sel: np.ndarray    # int32 [3, B]
    count: np.ndarray  # int64 [3, B]
    umap: np.ndarray   # uint16 [U] union bin -> grid bin


class Tables:
    """Owns one cs_tables handle: the merged rank tables of M grids for one cap dtype."""

    def __init__(self, handle: int, grids: Sequence, cap_dtype: str, batching_mtl: int, multi_tenant_bs: int,
                 keep: list):
        self._h = C.c_void_p(handle)
        self.grids = list(grids)
        self.cap_dtype = cap_dtype
        self.batching_mtl = batching_mtl
        self.multi_tenant_bs = multi_tenant_bs
        self._keep = keep
        info = N.TablesInfo()
        N.check(N.lib().cs_tables_get_info(self._h, C.byref(info)))
        self.info = info
        self.n_grids = info.n_grids
        self.n_union_bins = info.n_union_bins
        self._bins: list[GridBins | None] = [None] * self.n_grids
        self._fin = weakref.finalize(self, N.lib().cs_tables_destroy, self._h)

    # ---- construction ----
    @staticmethod
    def stage(grids: Sequence, cap_dtype: str = "f32", *, batching_mtl: int = 1, multi_tenant_bs: int = 1) -> "Tables":
        """N1: build the rank tables for ``grids`` (PolicyIndex.__init__, policy.py:118-134)."""
        if cap_dtype not in _DTYPES:
            raise ValueError(f"cap_dtype must be one of {tuple(_DTYPES)}")
        grids = list(grids)
        if not grids:
            raise ValidationError("need at least one grid")
        descs = (N.GridDesc * len(grids))()
        keep = []
        for i, g in enumerate(grids):
            _, mtl, bs, thr, pw = grid_arrays(g)
            keep += [mtl, bs, thr, pw]
            idle = g.gpu_idle_power_w
            descs[i] = N.GridDesc(
                len(mtl), mtl.ctypes.data_as(C.POINTER(C.c_int32)), bs.ctypes.data_as(C.POINTER(C.c_int32)),
                thr.ctypes.data_as(C.POINTER(C.c_double)), pw.ctypes.data_as(C.POINTER(C.c_double)),
                float("nan") if idle is None else float(idle))
        h = C.c_void_p()
        N.check(N.lib().cs_tables_create(descs, len(grids), _DTYPES[cap_dtype], int(batching_mtl),
                                         int(multi_tenant_bs), C.byref(h)), invalid=ValidationError)
        return Tables(h.value, grids, cap_dtype, batching_mtl, multi_tenant_bs, [])

    @staticmethod
    def for_grid(grid, cap_dtype: str = "f64", *, batching_mtl: int = 1, multi_tenant_bs: int = 1) -> "Tables":
        """Single-grid tables cached on the (immutable) grid object."""
        cache = grid.__dict__.setdefault("_cs_tables", {})
        key = (cap_dtype, int(batching_mtl), int(multi_tenant_bs))
        t = cache.get(key)
        if t is None:
            t = Tables.stage([grid], cap_dtype, batching_mtl=batching_mtl, multi_tenant_bs=multi_tenant_bs)
            cache[key] = t
        return t

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def grid_bins(self, m: int) -> GridBins:
        gb = self._bins[m]
        if gb is None:
            B = self.info.max_grid_bins
            sel = np.zeros((3, B), dtype=np.int32)
            cnt = np.zeros((3, B), dtype=np.int64)
            nb = C.c_int32()
            for p in range(3):
                N.check(N.lib().cs_tables_grid_bins(self._h, m, p, sel[p].ctypes.data, cnt[p].ctypes.data,
                                                    C.byref(nb)))
            umap = np.zeros(self.n_union_bins, dtype=np.uint16)
            N.check(N.lib().cs_tables_union_map(self._h, m, umap.ctypes.data))
            gb = GridBins(sel[:, :nb.value].copy(), cnt[:, :nb.value].copy(), umap)
            self._bins[m] = gb
        return gb

    def lookup_host(self, caps: np.ndarray, lut: str = "main") -> np.ndarray:
        """Host restatement of the device LUT search (test hook, not used by the product path).
        ``lut="big"`` / ``"huge"`` search the finer fp32 LUTs the evaluation kernel stages when they
        fit."""
        dt = np.float32 if self.cap_dtype == "f32" else np.float64
        caps = np.ascontiguousarray(caps, dtype=dt)
        out = np.zeros(caps.shape[0], dtype=np.int32)
        N.check(N.lib().cs_tables_lookup_host_lut(self._h, caps.ctypes.data, caps.shape[0],
                                                  {"main": 0, "big": 1, "huge": 2}[lut], out.ctypes.data))
        return out

    # ---- evaluation ----
    def evaluate(self, caps, n_steps: int | None = None, *, step_seconds: int, switch_penalty_s: float = 0.0,
                 per_step: bool = False, check_violations: bool = True, want_hist: bool = True,
                 accumulate_hist=None, stream=None, segment_epilogue: bool = False,
                 _prepared_ws=None) -> "EvalResult":
        """N2+N3 over a device cap matrix ``caps`` [T, ld] (torch, cuda, dtype of the tables).

        Every (trace, grid, policy) aggregate of simulate() is produced in one pass; per-step
        union bins are written when ``per_step``."""
        torch = _torch()
        dt = torch.float32 if self.cap_dtype == "f32" else torch.float64
        if not caps.is_cuda or caps.dtype != dt or caps.dim() != 2:
            raise ValueError(f"caps must be a 2-D {dt} CUDA tensor")
        T, ld = caps.shape
        if caps.stride(1) != 1:
            raise ValueError("caps rows must be contiguous")
        ld = caps.stride(0) if T > 1 else ld
        S = int(n_steps if n_steps is not None else caps.shape[1])
        dev = caps.device
        with torch.cuda.device(dev):
            agg = torch.empty((T, self.n_grids, 3, 6), dtype=torch.float64, device=dev)
            hist = accumulate_hist
            if hist is None and want_hist:
                hist = torch.empty(self.n_union_bins, dtype=torch.int64, device=dev)
            bins = None
            ld_bins = 0
            if per_step:
                ld_bins = (S + 3) // 4 * 4
                bins = torch.empty((T, ld_bins), dtype=torch.int16, device=dev)
            a = N.EvalArgs()
            a.caps = caps.data_ptr()
            a.n_traces = T
            a.n_steps = S
            a.ld = ld
            a.step_seconds = int(step_seconds)
            a.switch_penalty_s = float(switch_penalty_s)
            a.flags = (N.CS_FLAG_CHECK_VIOLATIONS if check_violations else 0) | (
                N.CS_FLAG_ACCUMULATE_HIST if accumulate_hist is not None else 0) | (
                N.CS_FLAG_SEGMENT_EPILOGUE if segment_epilogue else 0) | (
                N.CS_FLAG_PREPARED if _prepared_ws is not None else 0)
            a.step_bins = bins.data_ptr() if bins is not None else None
            a.ld_bins = ld_bins
            a.agg = agg.data_ptr()
            a.hist = hist.data_ptr() if hist is not None else None
            ws_bytes = C.c_size_t()
            rc = N.lib().cs_eval_workspace_size(self._h, C.byref(a), C.byref(ws_bytes))
            if rc != N.CS_OK and self.n_grids > 1 and "too large for shared memory" in N.last_error():
                if per_step or accumulate_hist is not None:
                    raise ValueError("per-step output and histogram accumulation need every grid's tables in "
                                     "shared memory at once; split the grids across calls")
                return self._evaluate_chunked(caps, S, step_seconds=step_seconds, switch_penalty_s=switch_penalty_s,
                                              check_violations=check_violations, want_hist=want_hist, stream=stream,
                                              segment_epilogue=segment_epilogue)
            N.check(rc)
            ws = None
            if _prepared_ws is not None:  # EvalGraph: the value tables of an identical earlier launch
                if _prepared_ws.numel() != ws_bytes.value:
                    raise ValueError("prepared workspace does not match this launch")
                ws = _prepared_ws
                a.workspace = ws.data_ptr()
                a.workspace_bytes = ws_bytes.value
            elif ws_bytes.value:
                ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device=dev)
                a.workspace = ws.data_ptr()
                a.workspace_bytes = ws_bytes.value
            N.check(N.lib().cs_eval(self._h, C.byref(a), C.c_void_p(_stream_ptr(stream))))
        return EvalResult(self, agg, hist, bins, S, ws)

    def _evaluate_chunked(self, caps, S: int, **kw) -> "EvalResult":
        """Grids whose merged tables exceed shared memory run as consecutive grid chunks (each a
        Tables of its own, split in halves until each one's launch plan fits). Every grid's
        aggregates are independent of the others, so the chunked result is the same; the union-bin
        histogram is kept per chunk (EvalResult.parts), config histograms per grid are exact."""
        torch = _torch()
        key = (float(kw.get("switch_penalty_s", 0.0)) > 0.0, bool(kw.get("want_hist", True)))  # what sizes the plan
        cache = self.__dict__.setdefault("_chunks", {})
        if key not in cache:
            chunks = []
            todo = [(0, self.n_grids // 2), (self.n_grids // 2, self.n_grids)]  # the whole set does not fit
            while todo:
                lo, hi = todo.pop(0)
                t = Tables.stage(self.grids[lo:hi], self.cap_dtype, batching_mtl=self.batching_mtl,
                                 multi_tenant_bs=self.multi_tenant_bs)
                if hi - lo > 1 and not t._plan_fits(caps, S, kw):
                    mid = (lo + hi) // 2
                    todo[:0] = [(lo, mid), (mid, hi)]
                    continue
                chunks.append((lo, hi, t))
            cache[key] = chunks
        agg = torch.empty((caps.shape[0], self.n_grids, 3, 6), dtype=torch.float64, device=caps.device)
        parts, keep = [], []
        for lo, hi, t in cache[key]:
            r = t.evaluate(caps, S, **kw)
            agg[:, lo:hi] = r.agg
            parts += [(lo + l2, t2, h2) for l2, t2, h2 in r.parts] if r.parts is not None else [(lo, t, r.hist)]
            keep.append(r)
        return EvalResult(self, agg, None, None, S, keep, parts)

    def _plan_fits(self, caps, S: int, kw: dict) -> bool:
        a = N.EvalArgs()
        a.caps = caps.data_ptr()
        a.n_traces = caps.shape[0]
        a.n_steps = S
        a.ld = caps.stride(0) if caps.shape[0] > 1 else caps.shape[1]
        a.step_seconds = int(kw.get("step_seconds", 1))
        a.switch_penalty_s = float(kw.get("switch_penalty_s", 0.0))
        a.flags = N.CS_FLAG_CHECK_VIOLATIONS if kw.get("check_violations", True) else 0
        a.agg = 1
        a.hist = 1 if kw.get("want_hist", True) else None
        ws = C.c_size_t()
        return N.lib().cs_eval_workspace_size(self._h, C.byref(a), C.byref(ws)) == N.CS_OK

    def capture(self, caps, n_steps: int | None = None, **kw) -> EvalGraph:
        """evaluate() as a replayable CUDA graph (same arguments; see EvalGraph)."""
        return EvalGraph(self, caps, n_steps, **kw)

    def last_plan(self) -> dict:
        """Launch plan of the last evaluate() on this thread (CTAs, block size, group size, ...)."""
        p = N.EvalPlan()
        N.check(N.lib().cs_eval_last_plan(C.byref(p)))
        return {f: getattr(p, f) for f, _ in p._fields_}

    def launch_count(self) -> int:
        n = C.c_int32()
        N.check(N.lib().cs_eval_last_launches(C.byref(n)))
        return n.value

    def select_caps(self, grid_index: int, policy: int, caps_dev) -> tuple:
        """select_config for many caps: warp-per-cap argmax kernel (policy.py:172-188)."""
        torch = _torch()
        n = caps_dev.shape[0]
        sel = torch.empty(n, dtype=torch.int32, device=caps_dev.device)
        cnt = torch.empty(n, dtype=torch.int64, device=caps_dev.device)
        with torch.cuda.device(caps_dev.device):
            N.check(N.lib().cs_select_caps(self._h, grid_index, policy, caps_dev.data_ptr(), n, sel.data_ptr(),
                                           cnt.data_ptr(), C.c_void_p(_stream_ptr(None))))
        return sel, cnt

    def select_sampling(self, grid_index: int, caps_dev, n_steps: int, budget_m: int, rounds_r: int,
                        seed_base: int) -> tuple:
        """select_sampling at every (trace, step) of an fp64 [T, ld] cap matrix; step i draws with
        random.Random(seed_base + i) (policy.py:218-273, sim.py:159-163). One thread per step.
        Returns (entry int32 [T, n_steps] caller index or -1, feasible_count int32 [T, n_steps])."""
        torch = _torch()
        if self.cap_dtype != "f64":
            raise ValueError("select_sampling needs tables staged for fp64 caps")
        t = caps_dev.shape[0] if caps_dev.dim() == 2 else 1
        ld = caps_dev.shape[-1]
        lo_v, hi_v = int(seed_base), int(seed_base) + max(int(n_steps) - 1, 0)
        if lo_v < -(1 << 127) or hi_v >= (1 << 127):
            raise NotImplementedError("sampling seeds beyond 127 bits are not supported")
        two = int(seed_base) & ((1 << 128) - 1)
        seed_lo = two & ((1 << 64) - 1)
        seed_hi = two >> 64
        if seed_hi >= 1 << 63:
            seed_hi -= 1 << 64
        ent = torch.empty((t, n_steps), dtype=torch.int32, device=caps_dev.device)
        cnt = torch.empty((t, n_steps), dtype=torch.int32, device=caps_dev.device)
        with torch.cuda.device(caps_dev.device):
            N.check(N.lib().cs_select_sampling(self._h, grid_index, caps_dev.data_ptr(), t, n_steps, ld,
                                               int(budget_m), int(rounds_r), seed_lo, seed_hi, ent.data_ptr(),
                                               cnt.data_ptr(), C.c_void_p(_stream_ptr(None))))
        return ent, cnt

    def aggregate_entries(self, grid_index: int, entries_dev, n_steps: int, *, step_seconds: int,
                          switch_penalty_s: float = 0.0):
        """_aggregate (sim.py:104-127) of per-step entry selections ``entries_dev`` int32 [T, ld]
        (caller entry index, -1 idle) on the device: (avg_throughput_ips f64 [T], energy_proxy_wh
        f64 [T], idle_steps int64 [T]). Values are split {hi, lo} so the sums of hi are exact."""
        torch = _torch()
        g = self.grids[grid_index]
        _, _, _, thr, pw = grid_arrays(g)
        idle_pw = g.gpu_idle_power_w if g.gpu_idle_power_w is not None else 0.0
        step = float(step_seconds)
        pf = min(float(switch_penalty_s), step) / step
        thr1 = np.append(thr, 0.0)
        vals = [thr1, thr1 * (1.0 - pf), np.append(pw, idle_pw) * step / 3600.0]  # sim.py:111,120,122
        L = 52
        while L > 1 and float(n_steps) >= 2.0 ** (53 - L):
            L -= 1
        table = np.zeros((3, thr1.shape[0], 2))
        for j, v in enumerate(vals):
            ref = v if j != 1 else vals[0]  # thr and penalised thr share the quantum
            e = np.frexp(max(float(ref.max()), 0.0) or 1.0)[1] - L
            hi = np.ldexp(np.floor(np.ldexp(v, -e)), e)
            table[j, :, 0], table[j, :, 1] = hi, v - hi
        T = entries_dev.shape[0]
        dev = entries_dev.device
        tv = torch.from_numpy(table).to(dev)
        avg = torch.empty(T, dtype=torch.float64, device=dev)
        en = torch.empty(T, dtype=torch.float64, device=dev)
        idle = torch.empty(T, dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            N.check(N.lib().cs_entries_aggregate(entries_dev.data_ptr(), T, int(n_steps), entries_dev.stride(0),
                                                 tv.data_ptr(), int(thr.shape[0]), pf, avg.data_ptr(), en.data_ptr(),
                                                 idle.data_ptr(), C.c_void_p(_stream_ptr(None))))
        return avg, en, idle

    def query(self, kind: int, caps, grid_index: int = 0, policy: int = 0):
        """Low-latency per-cap query from host memory (cs_query_host): one H2D, one kernel, one
        D2H and a sync. kind: N.CS_QUERY_BINS -> union bins int32 [n]; CS_QUERY_SELECT ->
        (entry int32 [n], feasible_count int64 [n]); CS_QUERY_FEASIBLE -> uint32 [n, words]."""
        require_device()
        c = np.ascontiguousarray(caps, dtype=np.float64)
        n = c.shape[0]
        out2 = None
        if kind == N.CS_QUERY_BINS:
            out = np.empty(n, np.int32)
        elif kind == N.CS_QUERY_SELECT:
            out, out2 = np.empty(n, np.int32), np.empty(n, np.int64)
        else:
            out = np.empty((n, (len(self.grids[grid_index].entries) + 31) // 32), np.uint32)
        N.check(N.lib().cs_query_host(self._h, int(kind), int(grid_index), int(policy), c.ctypes.data, n,
                                      out.ctypes.data, None if out2 is None else out2.ctypes.data))
        return out if out2 is None else (out, out2)

    def feasible_caps(self, grid_index: int, policy: int, caps_dev):
        """feasible_set for many caps: warp-per-cap ballot bitmask (policy.py:151-169)."""
        torch = _torch()
        n = caps_dev.shape[0]
        ne = len(self.grids[grid_index].entries)
        words = (ne + 31) // 32
        mask = torch.empty((n, words), dtype=torch.int32, device=caps_dev.device)
        with torch.cuda.device(caps_dev.device):
            N.check(N.lib().cs_feasible_caps(self._h, grid_index, policy, caps_dev.data_ptr(), n, mask.data_ptr(),
                                             C.c_void_p(_stream_ptr(None))))
        return mask

    def config_histograms(self, hist) -> list[list[dict]]:
        """Global config histograms per (grid, policy) from the union-bin histogram:
        {Config or None (idle): steps}. Integer-exact (no sums of floats involved)."""
        h = np.asarray(hist.cpu() if hasattr(hist, "cpu") else hist, dtype=np.int64)
        out = []
        for m, g in enumerate(self.grids):
            cfgs = g.columns()[0]
            gb = self.grid_bins(m)
            gh = np.zeros(gb.sel.shape[1], dtype=np.int64)
            np.add.at(gh, gb.umap.astype(np.int64), h)
            row = []
            for p in range(3):
                d: dict = {}
                for b in np.nonzero(gh)[0]:
                    s = int(gb.sel[p, b])
                    key = None if s < 0 else cfgs[s]
                    d[key] = d.get(key, 0) + int(gh[b])
                row.append(d)
            out.append(row)
        return out


class EvalGraph:
    """One ``Tables.evaluate`` captured as a CUDA graph. ``replay()`` re-runs the launch sequence
    (eval, finalize kernels and the histogram memset) on the same device buffers in a single
    graph launch: for latency-bound sweeps (a few traces) the host path — Python, ctypes, plan —
    costs more than the kernels. The per-launch value tables (prep kernel) depend only on the
    tables and the arguments, so the warm-up launch writes them once into a workspace the graph
    keeps (CS_FLAG_PREPARED). Inputs are read from ``caps`` at replay time, so refill it in place
    to evaluate new data; ``result`` holds the outputs of the latest replay."""

    def __init__(self, tables: "Tables", caps, n_steps: int | None = None, *, sweep_totals: bool = False, **kw):
        torch = _torch()
        from .shard import sweep_words

        self.tables = tables
        warm = tables.evaluate(caps, n_steps, **kw)  # outside capture: upload, plan memo, value tables
        torch.cuda.synchronize()
        self._ws = warm._ws
        self.graph = torch.cuda.CUDAGraph()
        self.words = None  # sweep_totals: cs_sweep_totals of the replay's aggregates (same graph)
        with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
            self.result = tables.evaluate(caps, n_steps, _prepared_ws=self._ws, **kw)
            if sweep_totals:
                self.words = sweep_words(tables, self.result.agg)
        torch.cuda.synchronize()

    def replay(self) -> "EvalResult":
        self.graph.replay()
        return self.result


@dataclass
class EvalResult:
    tables: Tables
    agg: "object"        # torch.float64 [T, M, 3, 6] (cs_agg rows)
    hist: "object"       # torch.int64 [U] or None
    step_bins: "object"  # torch.int16 [T, ld_bins] or None (union bin per step, as uint16)
    n_steps: int
    _ws: "object" = None
    parts: "object" = None  # chunked runs: [(first grid, chunk Tables, chunk union-bin hist)]

    def config_histograms(self) -> list[list[dict]]:
        """Per (grid, policy) config histograms {Config or None: steps} (chunked runs included)."""
        if self.parts is None:
            return self.tables.config_histograms(self.hist)
        out = []
        for _, t, h in self.parts:
            out += t.config_histograms(h)
        return out

    @property
    def avg_throughput_ips(self):
        return self.agg[..., 0]

    @property
    def energy_proxy_wh(self):
        return self.agg[..., 1]

    def _int(self, k: int):
        return self.agg.view(_torch().int64)[..., k]

    @property
    def idle_steps(self):
        return self._int(2)

    @property
    def switches(self):
        return self._int(3)

    @property
    def violations(self):
        return self._int(4)

    def bins_numpy(self, t: int = 0) -> np.ndarray:
        """Union bin per step of trace t (host copy)."""
        b = self.step_bins[t, : self.n_steps].cpu().numpy().view(np.uint16)
        return b.astype(np.int64)


def generate_traces(n_traces: int, n_steps: int, *, step_seconds: int, kind: str = "mixed", peak_w: float = 350.0,
                    seed: int = 1, first_trace_id: int = 0, ld: int | None = None, out=None, stream=None):
    """Synthetic fp32 cap traces on the device (counter-based RNG keyed by (seed, global trace id),
    so a trace is identical whichever GPU/shard generates it)."""
    torch = _torch()
    dev = require_device()
    ld = ld if ld is not None else (n_steps + 3) // 4 * 4
    if out is None:
        out = torch.zeros((n_traces, ld), dtype=torch.float32, device=dev)
    N.check(N.lib().cs_generate_traces(out.data_ptr(), n_traces, n_steps, ld, first_trace_id, int(step_seconds),
                                       N.TRACE_KINDS[kind], float(peak_w), int(seed) & (2**64 - 1),
                                       C.c_void_p(_stream_ptr(stream))))
    return out


class HostEngine:
    """Host-buffer path (the e2e measurement): chunked H2D -> eval -> D2H on three streams."""

    def __init__(self, tables: Tables, chunk_traces: int, n_steps_max: int, device: int | None = None):
        torch = _torch()
        require_device()
        self.tables = tables
        dev = torch.cuda.current_device() if device is None else device
        h = C.c_void_p()
        N.check(N.lib().cs_engine_create(dev, int(chunk_traces), int(n_steps_max), _DTYPES[tables.cap_dtype],
                                         C.byref(h)))
        self._h = h
        self._fin = weakref.finalize(self, N.lib().cs_engine_destroy, h)

    def evaluate(self, caps_host, n_steps: int, *, step_seconds: int, switch_penalty_s: float = 0.0,
                 check_violations: bool = True, agg_out=None, hist_out=None):
        """caps_host: pinned (or pageable) host tensor [T, ld]. Returns (agg, hist, h2d, d2h)."""
        torch = _torch()
        dt = torch.float32 if self.tables.cap_dtype == "f32" else torch.float64
        if caps_host.dtype != dt or caps_host.dim() != 2 or caps_host.is_cuda:
            raise ValueError(f"caps_host must be a 2-D {dt} host tensor")
        if caps_host.stride(1) != 1:
            raise ValueError("caps_host rows must be contiguous")
        T = caps_host.shape[0]
        if not 1 <= int(n_steps) <= caps_host.shape[1]:
            raise ValueError("n_steps must be in [1, caps_host.shape[1]]")
        M = self.tables.n_grids
        if agg_out is None:
            agg_out = torch.empty((T, M, 3, 6), dtype=torch.float64, pin_memory=True)
        if hist_out is None:
            hist_out = torch.empty(self.tables.n_union_bins, dtype=torch.int64, pin_memory=True)
        h2d, d2h = C.c_int64(), C.c_int64()
        N.check(N.lib().cs_engine_eval_host(
            self._h, self.tables.handle, caps_host.data_ptr(), T, int(n_steps),
            caps_host.stride(0) if T > 1 else caps_host.shape[1],
            int(step_seconds), float(switch_penalty_s), N.CS_FLAG_CHECK_VIOLATIONS if check_violations else 0,
            agg_out.data_ptr(), hist_out.data_ptr(), C.byref(h2d), C.byref(d2h)))
        return agg_out, hist_out, h2d.value, d2h.value
