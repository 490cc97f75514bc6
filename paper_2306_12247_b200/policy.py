"""Policies: batching-only, multi-tenant-only and combination (mirrors capsim.policy).

Same names, signatures, result records and error behaviour as the reference
(policy.py:25-188); every decision is computed on the GPU:

* ``PolicyIndex`` stages the grid once (N1, engine.Tables) and answers caps with the
  per-timestep bin-lookup kernel;
* ``select_config`` is a warp-per-cap argmax kernel over the regime's entries (shuffles);
* ``feasible_set`` is a warp-per-cap ballot kernel.

* ``select_sampling`` / ``sampling_steps`` run the sampling kernel, one thread per step, with
  CPython's random.Random replayed bit for bit (policy.py:191-273).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np

from .errors import ValidationError
from .profile import Config, ProfileGrid


class PolicyTag(str, Enum):
    BATCHING = "batching"
    MULTI_TENANT = "multi-tenant"
    COMBINATION = "combination"
    SAMPLING = "sampling"


_POLICY_INDEX = {PolicyTag.BATCHING: 0, PolicyTag.MULTI_TENANT: 1, PolicyTag.COMBINATION: 2}


@dataclass(frozen=True)
class PolicyKind:
    """Which slice of the grid a selector may search (sampling carries its budget)."""

    tag: PolicyTag
    budget_m: int = 0
    rounds_r: int = 0

    def __post_init__(self) -> None:
        if self.tag is PolicyTag.SAMPLING:
            if self.budget_m < 1:
                raise ValidationError(f"sampling budget must be >= 1, got {self.budget_m}")
            if self.rounds_r < 0:
                raise ValidationError(f"refinement rounds must be >= 0, got {self.rounds_r}")
        elif self.budget_m or self.rounds_r:
            raise ValidationError(f"{self.tag.value} policy takes no sampling parameters")

    @property
    def label(self) -> str:
        if self.tag is PolicyTag.SAMPLING:
            return f"sampling(m={self.budget_m},r={self.rounds_r})"
        return self.tag.value

    @property
    def index(self) -> int:
        """Position in the engine's policy axis (batching, multi-tenant, combination)."""
        if self.tag is PolicyTag.SAMPLING:
            raise ValueError("sampling is not an exhaustive policy; it has no slot on the policy axis")
        return _POLICY_INDEX[self.tag]


BATCHING = PolicyKind(PolicyTag.BATCHING)
MULTI_TENANT = PolicyKind(PolicyTag.MULTI_TENANT)
COMBINATION = PolicyKind(PolicyTag.COMBINATION)


def sampling_policy(budget_m: int, rounds_r: int = 1) -> PolicyKind:
    return PolicyKind(PolicyTag.SAMPLING, budget_m=budget_m, rounds_r=rounds_r)


@dataclass(frozen=True)
class Selection:
    """Chosen config (None = idle), its operating point and the feasible-set size."""

    config: Config | None
    throughput_ips: float
    power_w: float
    feasible_count: int = 0

    def __post_init__(self) -> None:
        if self.config is None:
            if self.throughput_ips != 0 or self.power_w != 0:
                raise ValidationError("idle selection must have zero throughput and power")
        elif self.throughput_ips <= 0:
            raise ValidationError(f"selected throughput must be positive, got {self.throughput_ips}")

    @property
    def idle(self) -> bool:
        return self.config is None


IDLE_SELECTION = Selection(config=None, throughput_ips=0.0, power_w=0.0, feasible_count=0)


def _check_cap(cap_w: float) -> None:
    if cap_w < 0:
        raise ValueError(f"cap_w must be >= 0, got {cap_w}")


def _regime_index(kind: PolicyKind) -> int:
    """_regime_entries (policy.py:100-107): batching and multi-tenant slice the grid, every other
    kind (combination, sampling) takes all entries — so a PolicyIndex of a sampling kind is the
    combination index (policy.py:118-134)."""
    return _POLICY_INDEX.get(kind.tag, _POLICY_INDEX[PolicyTag.COMBINATION])


def _exhaustive(kind: PolicyKind) -> int:
    if kind.tag is PolicyTag.SAMPLING:
        raise ValueError("sampling is not an exhaustive policy; use select_sampling")
    return _POLICY_INDEX[kind.tag]


def selections_for_bins(grid: ProfileGrid, sel: np.ndarray, count: np.ndarray) -> list[Selection]:
    """Decode table: one shared Selection object per grid bin."""
    cfgs = grid.columns()[0]
    out = []
    for s, c in zip(sel.tolist(), count.tolist()):
        if s < 0:
            out.append(IDLE_SELECTION)
        else:
            e = grid.entries[cfgs[s]]
            out.append(Selection(config=e.config, throughput_ips=e.throughput_ips, power_w=e.power_w,
                                 feasible_count=c))
    return out


class PolicyIndex:
    """Best-config-under-cap structure for one (grid, regime) (policy.py:110-148).

    Construction stages the grid's merged rank tables to the device (cached on the grid);
    ``select`` / ``select_many`` run the per-timestep lookup kernel."""

    def __init__(self, grid: ProfileGrid, kind: PolicyKind, *, batching_mtl: int = 1, multi_tenant_bs: int = 1):
        from .engine import Tables

        self.grid = grid
        self.kind = kind
        self._p = _regime_index(kind)
        self._tables = Tables.for_grid(grid, "f64", batching_mtl=batching_mtl, multi_tenant_bs=multi_tenant_bs)
        gb = self._tables.grid_bins(0)
        self._decode = selections_for_bins(grid, gb.sel[self._p], gb.count[self._p])

    def select_many(self, caps: Sequence[float]) -> list[Selection]:
        from . import _native as N
        from .engine import _torch, require_device

        caps = [float(c) for c in caps]
        for c in caps:
            _check_cap(c)
        if not caps:
            return []
        if len(caps) <= 4096:  # latency path: host buffers, one lookup launch
            # a NaN cap bisects to the end in the reference (policy.py:139)
            bins = self._tables.query(N.CS_QUERY_BINS, [math.inf if c != c else c for c in caps])
            return [self._decode[b] for b in bins.tolist()]
        torch = _torch()
        dev = require_device()
        n = len(caps)
        ld = n + (n & 1)
        buf = torch.zeros((1, ld), dtype=torch.float64)
        # a NaN cap bisects to the end in the reference (policy.py:139); canonicalise the sign
        buf[0, :n] = torch.tensor([math.inf if c != c else c for c in caps], dtype=torch.float64)
        res = self._tables.evaluate(buf.to(dev), n, step_seconds=1, per_step=True, check_violations=False,
                                    want_hist=False)
        bins = res.bins_numpy(0)
        return [self._decode[b] for b in bins.tolist()]

    def select(self, cap_w: float) -> Selection:
        return self.select_many([cap_w])[0]


def select_config(grid: ProfileGrid, kind: PolicyKind, cap_w: float, *, batching_mtl: int = 1,
                  multi_tenant_bs: int = 1) -> Selection:
    """Exhaustive argmax of throughput over the regime's feasible set (policy.py:172-188);
    ties go to lower power, then lower mtl, then lower bs. Runs the warp-argmax kernel."""
    return select_configs(grid, kind, [cap_w], batching_mtl=batching_mtl, multi_tenant_bs=multi_tenant_bs)[0]


def select_configs(grid: ProfileGrid, kind: PolicyKind, caps: Sequence[float], *, batching_mtl: int = 1,
                   multi_tenant_bs: int = 1) -> list[Selection]:
    """Batched select_config: one warp per cap."""
    from .engine import Tables, _torch, require_device

    p = _exhaustive(kind)
    caps = [float(c) for c in caps]
    for c in caps:
        _check_cap(c)
    if not caps:
        return []
    tables = Tables.for_grid(grid, "f64", batching_mtl=batching_mtl, multi_tenant_bs=multi_tenant_bs)
    if len(caps) <= 4096:  # latency path: host buffers, one select launch
        from . import _native as N

        sel, cnt = tables.query(N.CS_QUERY_SELECT, caps, 0, p)
        sel, cnt = sel.tolist(), cnt.tolist()
    else:
        torch = _torch()
        dev = require_device()
        sel, cnt = tables.select_caps(0, p, torch.tensor(caps, dtype=torch.float64, device=dev))
        sel, cnt = sel.cpu().tolist(), cnt.cpu().tolist()
    cfgs = grid.columns()[0]
    out = []
    for s, c in zip(sel, cnt):
        if s < 0:
            out.append(IDLE_SELECTION)
        else:
            e = grid.entries[cfgs[s]]
            out.append(Selection(config=e.config, throughput_ips=e.throughput_ips, power_w=e.power_w,
                                 feasible_count=c))
    return out


def feasible_set(grid: ProfileGrid, kind: PolicyKind, cap_w: float, *, batching_mtl: int = 1,
                 multi_tenant_bs: int = 1) -> set[Config]:
    """Configs of the regime whose power fits under the cap (policy.py:151-169); the sampling
    regime searches the combination space. Runs the warp-ballot kernel."""
    from .engine import Tables

    _check_cap(cap_w)
    p = _regime_index(kind)
    from . import _native as N

    tables = Tables.for_grid(grid, "f64", batching_mtl=batching_mtl, multi_tenant_bs=multi_tenant_bs)
    words = tables.query(N.CS_QUERY_FEASIBLE, [float(cap_w)], 0, p)[0]
    cfgs = grid.columns()[0]
    out = set()
    for w, bits in enumerate(words.tolist()):
        j = 0
        while bits:
            if bits & 1:
                out.add(cfgs[w * 32 + j])
            bits >>= 1
            j += 1
    return out


def select_sampling(grid: ProfileGrid, budget_m: int, rounds_r: int, cap_w: float, seed: int) -> Selection:
    """Low-overhead selection (policy.py:218-273): probe ``budget_m`` feasible configs drawn by
    random.Random(seed).sample, then hill-climb ``rounds_r`` rounds over present neighbours,
    accepting only feasible strictly-better moves. Runs the sampling kernel (one thread)."""
    return sampling_steps(grid, budget_m, rounds_r, [cap_w], seed)[0]


def sampling_steps(grid: ProfileGrid, budget_m: int, rounds_r: int, caps: Sequence[float],
                   seed_base: int) -> list[Selection]:
    """select_sampling for a sequence of caps, step i seeded with ``seed_base + i`` (the per-step
    seeds simulate() uses with seed_base = seed * 1_000_003, sim.py:33-35,159-163). One GPU
    thread per step."""
    from .engine import Tables, _torch, require_device

    if budget_m < 1:
        raise ValueError(f"budget_m must be >= 1, got {budget_m}")
    if rounds_r < 0:
        raise ValueError(f"rounds_r must be >= 0, got {rounds_r}")
    caps = [float(c) for c in caps]
    for c in caps:
        _check_cap(c)
    if not caps:
        return []
    torch = _torch()
    dev = require_device()
    tables = Tables.for_grid(grid, "f64")
    # a NaN cap admits nothing (power <= nan is False): the idle bin
    host = torch.tensor([0.0 if c != c else c for c in caps], dtype=torch.float64).reshape(1, -1)
    ent, cnt = tables.select_sampling(0, host.to(dev), len(caps), budget_m, rounds_r, seed_base)
    return decode_entries(grid, ent[0].cpu().numpy(), cnt[0].cpu().numpy())


def decode_entries(grid: ProfileGrid, entries: np.ndarray, counts: np.ndarray) -> list[Selection]:
    """Caller entry indices (-1 idle) + feasible counts -> Selections (shared per distinct pair)."""
    cfgs = grid.columns()[0]
    memo: dict = {}
    out = []
    for s, c in zip(entries.tolist(), counts.tolist()):
        sel = memo.get((s, c))
        if sel is None:
            if s < 0:
                sel = IDLE_SELECTION
            else:
                e = grid.entries[cfgs[s]]
                sel = Selection(config=e.config, throughput_ips=e.throughput_ips, power_w=e.power_w,
                                feasible_count=c)
            memo[(s, c)] = sel
        out.append(sel)
    return out


def improvement_pct(a: float, b: float) -> float:
    """Relative improvement of a over baseline b, in percent (policy.py:276-281)."""
    if b <= 0:
        raise ValueError(f"baseline must be positive, got {b}")
    return (a - b) / b * 100.0
