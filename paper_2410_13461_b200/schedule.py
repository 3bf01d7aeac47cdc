"""Precision-switching schedules (drop-in for the runtime part of ``pmpd.schedule``).

Host-side schedule objects with the reference's names, validation messages
and JSON form (pkg/src/pmpd/schedule.py:25-256), plus their device form: a
fixed-capacity int32 switch-point table consumed by ``pmpd_sched_step``, the
on-device precision hook that replaces ``precision_at`` inside the decode loop
(tinylm.py:512,518) without any host synchronisation.

The offline searches (PAPAlloc, grid solver, brute force — schedule.py:263-457)
are out of scope for the B200 hot path.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field
from typing import Sequence

from .errors import ConfigError, InputError
from .quant import PrecisionSet

TABLE_CAPACITY = 8  # (p, switch point) pairs in a device schedule table


@dataclass(frozen=True)
class QualityTarget:
    """Quality floor ``q_ref - tolerance`` a schedule must meet (schedule.py:25-39)."""

    q_ref: float
    tolerance: float
    metric: str = "rouge_l_f1"

    def __post_init__(self):
        if self.tolerance < 0:
            raise ConfigError(f"tolerance must be >= 0, got {self.tolerance}")

    @property
    def floor(self) -> float:
        return self.q_ref - self.tolerance


@dataclass(frozen=True)
class SwitchGrid:
    """``n`` equally spaced candidate switch points spanning ``[0, horizon]`` (schedule.py:42-62)."""

    n: int
    horizon: int
    points: tuple = field(init=False)

    def __post_init__(self):
        if self.n < 2:
            raise ConfigError(f"grid needs at least 2 points, got {self.n}")
        if self.horizon < 1:
            raise ConfigError(f"horizon must be >= 1, got {self.horizon}")
        pts = tuple(int(math.floor(j * self.horizon / (self.n - 1) + 0.5)) for j in range(self.n))
        if any(a >= b for a, b in zip(pts, pts[1:])):
            raise ConfigError(f"grid points must be strictly increasing; horizon {self.horizon} "
                              f"is too short for {self.n} points: {pts}")
        object.__setattr__(self, "points", pts)


class _WidePrecisions:
    """Precision list for schedules using widths above 8 bits (the 16-bit sentinel)."""

    def __init__(self, ps):
        self.precisions = tuple(int(p) for p in ps)

    @property
    def p_max(self):
        return self.precisions[0]

    @property
    def p_min(self):
        return self.precisions[-1]

    def __iter__(self):
        return iter(self.precisions)

    def __len__(self):
        return len(self.precisions)

    def __contains__(self, p):
        return p in self.precisions


class PrecisionSchedule:
    """Decode precisions plus their switch points and the prefill precision (schedule.py:65-153)."""

    def __init__(self, precisions, p_prefill: int, switch_points: dict, horizon: int, feasible: bool = True):
        if not isinstance(precisions, (PrecisionSet, _WidePrecisions)):
            ps = tuple(int(p) for p in precisions)
            precisions = PrecisionSet(ps) if all(1 <= p <= 8 for p in ps) else _WidePrecisions(ps)
        self.precisions = precisions
        self.p_prefill = int(p_prefill)
        self.switch_points = {int(p): int(i) for p, i in switch_points.items()}
        self.horizon = int(horizon)
        self.feasible = bool(feasible)

    @classmethod
    def constant(cls, p: int, horizon: int, p_prefill: int | None = None, feasible: bool = True):
        return cls((p,), p if p_prefill is None else p_prefill, {p: 0}, horizon, feasible)

    @classmethod
    def two_phase(cls, p_high: int, p_low: int, switch: int, horizon: int, p_prefill: int | None = None):
        return cls(PrecisionSet((p_high, p_low)), p_high if p_prefill is None else p_prefill,
                   {p_high: 0, p_low: switch}, horizon)

    def precision_at(self, i: int) -> int:
        """Lowest precision whose switch point is <= i (schedule.py:93-99)."""
        for p in reversed(self.precisions.precisions):
            if self.switch_points[p] <= i:
                return p
        return self.precisions.p_max

    def validate(self) -> list:
        """All violated constraints, empty when the schedule is well formed (schedule.py:101-126)."""
        ps = self.precisions.precisions
        out = []
        for p in ps:
            if p not in self.switch_points:
                out.append(f"precision {p} has no switch point")
        covered = [p for p in ps if p in self.switch_points]
        for p in covered:
            st = self.switch_points[p]
            if not 0 <= st <= self.horizon:
                out.append(f"switch point of precision {p} is {st}, outside [0, {self.horizon}]")
        for hi, lo in itertools.combinations(covered, 2):
            if hi > lo and self.switch_points[hi] > self.switch_points[lo]:
                out.append(f"precedence violated: {hi} > {lo} but switch "
                           f"{self.switch_points[hi]} > {self.switch_points[lo]}")
        if ps and ps[0] in self.switch_points and self.switch_points[ps[0]] != 0:
            out.append(f"highest decode precision {ps[0]} must start at 0, got {self.switch_points[ps[0]]}")
        return out

    def bit_token_sum(self, tokens: int | None = None) -> int:
        n = self.horizon if tokens is None else tokens
        return sum(self.precision_at(i) for i in range(n))

    def device_table(self) -> list:
        """Flat int32 table ``[p0, st0, p1, st1, ...]`` of TABLE_CAPACITY pairs (unused p = 0)."""
        items = sorted(self.switch_points.items(), reverse=True)
        if len(items) > TABLE_CAPACITY:
            raise ConfigError(f"device schedules hold at most {TABLE_CAPACITY} precisions")
        flat = [0] * (2 * TABLE_CAPACITY)
        for i, (p, st) in enumerate(items):
            flat[2 * i], flat[2 * i + 1] = p, st
        return flat

    def to_json(self) -> dict:
        return {"precisions": list(self.precisions.precisions), "prefill": self.p_prefill,
                "st": {str(p): i for p, i in self.switch_points.items()}, "OL": self.horizon,
                "feasible": self.feasible}

    @classmethod
    def from_json(cls, obj: dict):
        try:
            return cls(tuple(obj["precisions"]), obj["prefill"], {int(p): int(i) for p, i in obj["st"].items()},
                       obj["OL"], obj.get("feasible", True))
        except (KeyError, TypeError, ValueError) as exc:
            raise InputError(f"malformed schedule JSON: {exc}") from exc

    def __repr__(self):
        return (f"PrecisionSchedule(precisions={list(self.precisions)}, prefill={self.p_prefill}, "
                f"st={self.switch_points}, OL={self.horizon}, feasible={self.feasible})")


def validate(schedule: PrecisionSchedule) -> list:
    """Report every violated schedule constraint; never raises (schedule.py:181-183)."""
    return schedule.validate()


def count_schedules(horizon: int, k: int) -> int:
    """Number of precedence-respecting switch maps (schedule.py:186-194)."""
    if horizon < 1:
        raise InputError(f"horizon must be >= 1, got {horizon}")
    if k < 1:
        raise InputError(f"precision count must be >= 1, got {k}")
    return sum(math.comb(horizon, r) * math.comb(k - 1, r) for r in range(k))


class StaticScheduler:
    """Fixed schedule chosen offline; the same for every prompt (schedule.py:213-228)."""

    def __init__(self, schedule: PrecisionSchedule):
        self.schedule = schedule

    @property
    def p_prefill(self) -> int:
        return self.schedule.p_prefill

    @property
    def horizon(self) -> int:
        return self.schedule.horizon

    def resolve(self, cache) -> PrecisionSchedule:
        return self.schedule


class FixedScheduler(StaticScheduler):
    """Single-precision schedule (the uniform baselines, schedule.py:231-236)."""

    def __init__(self, precision: int, horizon: int = 1 << 30, p_prefill: int | None = None):
        super().__init__(PrecisionSchedule.constant(precision, horizon, p_prefill))


def avg_bitwidth(subject, tokens_generated: int | None = None) -> float:
    """Token-weighted mean decode bitwidth (schedule.py:243-256)."""
    if tokens_generated is None:
        precisions = list(subject.precisions)
        if not precisions:
            raise InputError("trace has no generated tokens")
        return sum(precisions) / len(precisions)
    if tokens_generated < 1:
        raise InputError(f"tokens_generated must be >= 1, got {tokens_generated}")
    return subject.bit_token_sum(tokens_generated) / tokens_generated


def weighted_gpu_latency(latency_us: dict, schedule: PrecisionSchedule, gen_len: int):
    """Decode-step-weighted mean of per-precision latencies and its speedup over fp16 (perf.py:231-250)."""
    if gen_len < 1:
        raise InputError(f"gen_len must be >= 1, got {gen_len}")
    table = {int(k): float(v) for k, v in latency_us.items()}
    if 16 not in table:
        raise InputError("latency table lacks the fp16 (16) entry")
    counts = {}
    for i in range(gen_len):
        p = schedule.precision_at(i)
        if p not in table:
            raise InputError(f"latency table lacks precision {p}")
        counts[p] = counts.get(p, 0) + 1
    if len(counts) == 1:
        w = table[next(iter(counts))]
    else:
        w = sum(n * table[p] for p, n in counts.items()) / gen_len
    return w, table[16] / w
