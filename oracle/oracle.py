"""ctypes front-end of the CPU oracle (oracle/capsim_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs as the checker. The product package never imports it.

A grid is passed as a ``GridArrays`` (plain numpy arrays, no dependency on the product's
classes): mtl int32[n], bs int32[n], thr f64[n], pw f64[n], idle_power_w (0.0 when the grid
has no idle metadata, sim.py:175).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

REGIMES = {"batching": 0, "multi-tenant": 1, "combination": 2}


@dataclass(frozen=True)
class GridArrays:
    mtl: np.ndarray
    bs: np.ndarray
    thr: np.ndarray
    pw: np.ndarray
    idle_power_w: float = 0.0

    @staticmethod
    def from_rows(rows, idle_power_w: float | None = None) -> "GridArrays":
        """rows: iterable of (mtl, bs, throughput_ips, power_w)."""
        rows = list(rows)
        return GridArrays(
            mtl=np.ascontiguousarray([r[0] for r in rows], dtype=np.int32),
            bs=np.ascontiguousarray([r[1] for r in rows], dtype=np.int32),
            thr=np.ascontiguousarray([r[2] for r in rows], dtype=np.float64),
            pw=np.ascontiguousarray([r[3] for r in rows], dtype=np.float64),
            idle_power_w=0.0 if idle_power_w is None else float(idle_power_w),
        )

    def __len__(self) -> int:
        return int(self.mtl.shape[0])


def build() -> Path:
    """Compile the oracle with gcc (oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists() or LIB.stat().st_mtime < (HERE / "capsim_oracle.c").stat().st_mtime:
            build()
        L = C.CDLL(str(LIB))
        i32p, f64p, i64p = (np.ctypeslib.ndpointer(dtype=t, flags="C_CONTIGUOUS") for t in (np.int32, np.float64, np.int64))
        f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
        L.ora_index_build.argtypes = [i32p, i32p, f64p, f64p, C.c_int, C.c_int, C.c_int, C.c_int, f64p, i32p]
        L.ora_index_build.restype = C.c_int
        L.ora_index_select.argtypes = [f64p, i32p, C.c_int, C.c_double, C.POINTER(C.c_int32)]
        L.ora_index_select.restype = C.c_int64
        L.ora_bruteforce.argtypes = [i32p, i32p, f64p, f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
        L.ora_bruteforce.restype = C.c_int32
        L.ora_fsum.argtypes = [f64p, C.c_int64]
        L.ora_fsum.restype = C.c_double
        L.ora_aggregate.argtypes = [f64p, f64p, i32p, C.c_int64, C.c_int32, C.c_double, C.c_double,
                                    C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ora_aggregate.restype = None
        L.ora_simulate.argtypes = [i32p, i32p, f64p, f64p, C.c_int, C.c_int, f64p, C.c_int64, C.c_int32,
                                   C.c_double, C.c_double, i32p, i64p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ora_simulate.restype = C.c_int
        L.ora_simulate_batch.argtypes = [i32p, i32p, f64p, f64p, i64p, f64p, C.c_int, f32p, C.c_int64, C.c_int64,
                                         C.c_int32, C.c_double, C.c_int, f64p, i64p, f64p]
        L.ora_simulate_batch.restype = C.c_int
        u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
        u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
        L.ora_replay.argtypes = [i32p, i32p, f64p, f64p, C.c_int, f64p, C.c_int64, C.c_int, C.c_int, C.c_int32,
                                 C.c_double, u32p, C.c_int, u8p, f64p, i32p, i64p, i32p, i64p,
                                 C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ora_replay.restype = C.c_int
        L.ora_select_sampling.argtypes = [i32p, i32p, f64p, f64p, C.c_int, C.c_int64, C.c_int64, C.c_double, u32p,
                                          C.c_int, C.POINTER(C.c_int64)]
        L.ora_select_sampling.restype = C.c_int32
        L.ora_generate_traces.argtypes = [f32p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                          C.c_float, C.c_uint64, C.c_int]
        L.ora_generate_traces.restype = C.c_int
        _lib = L
    return _lib


class Index:
    """policy.py:110-148 — PolicyIndex restated over GridArrays."""

    def __init__(self, g: GridArrays, regime: str, batching_mtl: int = 1, multi_tenant_bs: int = 1):
        n = len(g)
        self.powers = np.zeros(max(n, 1), dtype=np.float64)
        self.best = np.zeros(max(n, 1), dtype=np.int32)
        self.n = lib().ora_index_build(g.mtl, g.bs, g.thr, g.pw, n, REGIMES[regime], batching_mtl, multi_tenant_bs,
                                       self.powers, self.best)

    def select(self, cap: float) -> tuple[int, int]:
        """-> (entry index or -1 when idle, feasible_count)"""
        if cap < 0:
            raise ValueError(f"cap_w must be >= 0, got {cap}")
        sel = C.c_int32()
        cnt = lib().ora_index_select(self.powers, self.best, self.n, float(cap), C.byref(sel))
        return int(sel.value), int(cnt)


def bruteforce(g: GridArrays, regime: str, cap: float, batching_mtl: int = 1, multi_tenant_bs: int = 1) -> int:
    """tests/conftest.py:100-129 brute-force argmax -> entry index or -1."""
    return int(lib().ora_bruteforce(g.mtl, g.bs, g.thr, g.pw, len(g), REGIMES[regime], batching_mtl,
                                    multi_tenant_bs, float(cap)))


def fsum(x) -> float:
    a = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().ora_fsum(a, a.shape[0]))


@dataclass
class SimResult:
    sel: np.ndarray  # int32 [S] entry index or -1
    count: np.ndarray  # int64 [S] feasible_count
    avg_throughput_ips: float
    idle_steps: int
    energy_proxy_wh: float


def simulate(g: GridArrays, caps, regime: str, step_seconds: int, switch_penalty_s: float = 0.0) -> SimResult:
    """sim.py:130-188 for one exhaustive policy (caps widened exactly to fp64)."""
    caps = np.ascontiguousarray(caps, dtype=np.float64)
    s = caps.shape[0]
    sel = np.zeros(max(s, 1), dtype=np.int32)
    cnt = np.zeros(max(s, 1), dtype=np.int64)
    avg, idle, en = C.c_double(), C.c_int64(), C.c_double()
    rc = lib().ora_simulate(g.mtl, g.bs, g.thr, g.pw, len(g), REGIMES[regime], caps, s, int(step_seconds),
                            float(g.idle_power_w), float(switch_penalty_s), sel, cnt, C.byref(avg), C.byref(idle),
                            C.byref(en))
    if rc != 0:
        raise ValueError("negative cap in trace")
    return SimResult(sel[:s], cnt[:s], avg.value, int(idle.value), en.value)


def simulate_batch(grids: list[GridArrays], caps2d: np.ndarray, step_seconds: int, switch_penalty_s: float = 0.0,
                   n_threads: int | None = None):
    """All (trace, grid, policy) runs of the reference algorithm on host threads.

    caps2d: float32 [T, S]. Returns (avg f64[T,M,3], idle i64[T,M,3], energy f64[T,M,3], threads)
    with policy order (batching, multi-tenant, combination)."""
    caps2d = np.ascontiguousarray(caps2d, dtype=np.float32)
    t, s = caps2d.shape
    m = len(grids)
    offs = np.zeros(m + 1, dtype=np.int64)
    for i, g in enumerate(grids):
        offs[i + 1] = offs[i] + len(g)
    cat = lambda name, dt: np.ascontiguousarray(np.concatenate([getattr(g, name) for g in grids]), dtype=dt)  # noqa: E731
    idle = np.ascontiguousarray([g.idle_power_w for g in grids], dtype=np.float64)
    out_avg = np.zeros(t * m * 3, dtype=np.float64)
    out_idle = np.zeros(t * m * 3, dtype=np.int64)
    out_en = np.zeros(t * m * 3, dtype=np.float64)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    used = lib().ora_simulate_batch(cat("mtl", np.int32), cat("bs", np.int32), cat("thr", np.float64),
                                    cat("pw", np.float64), offs, idle, m, caps2d, t, s, int(step_seconds),
                                    float(switch_penalty_s), int(n_threads), out_avg, out_idle, out_en)
    shp = (t, m, 3)
    return out_avg.reshape(shp), out_idle.reshape(shp), out_en.reshape(shp), used


TRACE_KINDS = {"solar": 0, "wind": 1, "mixed": 2, "iid": 3}


def generate_traces(n_traces: int, n_steps: int, *, step_seconds: int, kind: str = "mixed", peak_w: float = 350.0,
                    seed: int = 1, first_trace_id: int = 0, ld: int | None = None, n_threads: int | None = None):
    """Host port of the engine's synthetic trace generator (cs_generate_traces): bit-identical
    float32 [n_traces, ld] caps for the same arguments (bench inputs, not a reference function)."""
    ld = ld if ld is not None else (n_steps + 3) // 4 * 4
    out = np.zeros((n_traces, ld), dtype=np.float32)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    rc = lib().ora_generate_traces(out, n_traces, n_steps, ld, first_trace_id, int(step_seconds), TRACE_KINDS[kind],
                                   float(peak_w), int(seed) & (2**64 - 1), int(n_threads))
    if rc != 0:
        raise ValueError("bad generator arguments")
    return out


def seed_key(seed: int) -> np.ndarray:
    """random.Random(seed) key for init_by_array: 32-bit words of abs(seed), >= 1 word."""
    n = abs(int(seed))
    words = []
    while True:
        words.append(n & 0xFFFFFFFF)
        n >>= 32
        if not n:
            break
    return np.ascontiguousarray(words, dtype=np.uint32)


@dataclass
class ReplayResult:
    kind_bits: np.ndarray
    measured: np.ndarray
    sel_r: np.ndarray
    cnt_r: np.ndarray
    sel_f: np.ndarray
    cnt_f: np.ndarray
    violations: int
    reconfigs: int
    avg_throughput_ips: float
    start_sel: int
    start_cnt: int


def replay(g: GridArrays, caps, mode: str, window_k: int = 1, initial: int = -1, noise_pct: float = 0.0,
           seed: int = 0) -> ReplayResult:
    """controller.py:161-231 restated (ora_replay). initial: entry index or -1 (auto)."""
    caps = np.ascontiguousarray(caps, dtype=np.float64)
    n = caps.shape[0]
    key = seed_key(seed)
    kb = np.zeros(n, np.uint8)
    meas = np.zeros(n, np.float64)
    sr = np.zeros(n, np.int32)
    cr = np.zeros(n, np.int64)
    sf = np.zeros(n, np.int32)
    cf = np.zeros(n, np.int64)
    v, r, a = C.c_int64(), C.c_int64(), C.c_double()
    rc = lib().ora_replay(g.mtl, g.bs, g.thr, g.pw, len(g), caps, n, 1 if mode == "proactive" else 0,
                          int(window_k), int(initial), float(noise_pct), key, key.shape[0], kb, meas, sr, cr, sf, cf,
                          C.byref(v), C.byref(r), C.byref(a))
    if rc != 0:
        raise ValueError("bad replay arguments")
    if initial >= 0:
        s0, c0 = initial, 0
    else:
        s0, c0 = Index(g, "combination").select(float(caps[0]))
    return ReplayResult(kb, meas, sr, cr, sf, cf, int(v.value), int(r.value), a.value, s0, c0)


def replay_events(res: ReplayResult, caps, pw) -> tuple[list, list]:
    """Rebuild the reference's event log and parallel selection list (controller.py:200-218)
    as ([step, kind, cap, power], [(entry, count) | (-1, 0)])."""
    events, sels = [], []
    prior = (res.start_sel, res.start_cnt)
    for i in range(len(caps)):
        kb = int(res.kind_bits[i])
        cap = float(caps[i])
        rsel = (int(res.sel_r[i]), int(res.cnt_r[i]))
        fsel = (int(res.sel_f[i]), int(res.cnt_f[i]))
        if kb & 1:
            events.append([i, "violation_detected", cap, float(res.measured[i])])
            sels.append(prior)
            events.append([i, "reconfigured", cap, 0.0 if rsel[0] < 0 else float(pw[rsel[0]])])
            sels.append(rsel)
        else:
            events.append([i, "no_action", cap, float(res.measured[i])])
            sels.append(prior)
        if kb & 2:
            events.append([i, "preemptive_reconfigured", cap, 0.0 if fsel[0] < 0 else float(pw[fsel[0]])])
            sels.append(fsel)
        prior = fsel
    return events, sels


def select_sampling(g: GridArrays, budget_m: int, rounds_r: int, cap: float, seed: int) -> tuple[int, int]:
    """policy.py:218-273 restated (ora_select_sampling) -> (entry index or -1, feasible_count)."""
    if budget_m < 1 or rounds_r < 0 or cap < 0:
        raise ValueError("bad sampling arguments")
    key = seed_key(seed)
    cnt = C.c_int64()
    e = lib().ora_select_sampling(g.mtl, g.bs, g.thr, g.pw, len(g), int(budget_m), int(rounds_r), float(cap), key,
                                  key.shape[0], C.byref(cnt))
    return int(e), int(cnt.value)


SEED_STRIDE = 1_000_003  # sim.py:33-35


def simulate_sampling(g: GridArrays, caps, budget_m: int, rounds_r: int, seed: int, step_seconds: int,
                      switch_penalty_s: float = 0.0) -> SimResult:
    """sim.py:159-163 + _aggregate: per-step select_sampling with seed*1_000_003 + step."""
    caps = np.ascontiguousarray(caps, dtype=np.float64)
    s = caps.shape[0]
    sel = np.zeros(max(s, 1), dtype=np.int32)
    cnt = np.zeros(max(s, 1), dtype=np.int64)
    for i in range(s):
        sel[i], cnt[i] = select_sampling(g, budget_m, rounds_r, float(caps[i]), seed * SEED_STRIDE + i)
    avg, idle, en = C.c_double(), C.c_int64(), C.c_double()
    lib().ora_aggregate(g.thr, g.pw, sel, s, int(step_seconds), float(g.idle_power_w), float(switch_penalty_s),
                        C.byref(avg), C.byref(idle), C.byref(en))
    return SimResult(sel[:s], cnt[:s], avg.value, int(idle.value), en.value)
