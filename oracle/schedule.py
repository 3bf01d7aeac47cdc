"""Oracle restatement of the precision-switching schedules (reference ``pkg/src/pmpd/schedule.py``).

TEST INFRASTRUCTURE ONLY.  Only the runtime part of the module is restated
(SURVEY §8a rows A16-A18, A20); the offline solvers are out of scope.
"""
from __future__ import annotations

import math

from .errors import ConfigError, InputError


def grid_points(n: int, horizon: int) -> tuple:
    """``SwitchGrid.__post_init__`` (schedule.py:50-62): ``floor(j*OL/(n-1)+0.5)``, strictly increasing."""
    if n < 2:
        raise ConfigError(f"grid needs at least 2 points, got {n}")
    if horizon < 1:
        raise ConfigError(f"horizon must be >= 1, got {horizon}")
    pts = tuple(int(math.floor(j * horizon / (n - 1) + 0.5)) for j in range(n))
    if any(b <= a for a, b in zip(pts, pts[1:])):
        raise ConfigError(f"grid points must be strictly increasing; got {pts}")
    return pts


class Schedule:
    """``PrecisionSchedule`` (schedule.py:65-153): precisions (descending), prefill precision,
    switch points ``{p: first token index}`` and horizon OL."""

    def __init__(self, precisions, p_prefill, switch_points, horizon):
        self.precisions = tuple(int(p) for p in precisions)
        self.p_prefill = int(p_prefill)
        self.switch_points = {int(k): int(v) for k, v in switch_points.items()}
        self.horizon = int(horizon)

    @classmethod
    def constant(cls, p, horizon, p_prefill=None):
        """schedule.py:81-84."""
        return cls((p,), p if p_prefill is None else p_prefill, {p: 0}, horizon)

    @classmethod
    def two_phase(cls, p_high, p_low, switch, horizon, p_prefill=None):
        """schedule.py:86-91."""
        return cls((p_high, p_low), p_high if p_prefill is None else p_prefill,
                   {p_high: 0, p_low: switch}, horizon)

    def precision_at(self, i: int) -> int:
        """schedule.py:93-99: the lowest precision whose switch point is <= i."""
        best = None
        for p in self.precisions:
            if self.switch_points[p] <= i and (best is None or p < best):
                best = p
        return self.precisions[0] if best is None else best

    def validate(self) -> list:
        """schedule.py:101-126 (same messages)."""
        out = []
        ps = self.precisions
        for p in ps:
            if p not in self.switch_points:
                out.append(f"precision {p} has no switch point")
        have = [p for p in ps if p in self.switch_points]
        for p in have:
            st = self.switch_points[p]
            if st < 0 or st > self.horizon:
                out.append(f"switch point of precision {p} is {st}, outside [0, {self.horizon}]")
        for a in range(len(have)):
            for b in range(a + 1, len(have)):
                hi, lo = have[a], have[b]
                if hi > lo and self.switch_points[hi] > self.switch_points[lo]:
                    out.append(f"precedence violated: {hi} > {lo} but switch "
                               f"{self.switch_points[hi]} > {self.switch_points[lo]}")
        if ps and ps[0] in self.switch_points and self.switch_points[ps[0]] != 0:
            out.append(f"highest decode precision {ps[0]} must start at 0, got {self.switch_points[ps[0]]}")
        return out

    def bit_token_sum(self, tokens=None) -> int:
        """schedule.py:128-130."""
        n = self.horizon if tokens is None else tokens
        return sum(self.precision_at(i) for i in range(n))


def avg_bitwidth(sched: Schedule, tokens: int) -> float:
    """schedule.py:243-256 (schedule form)."""
    if tokens < 1:
        raise InputError(f"tokens_generated must be >= 1, got {tokens}")
    return sched.bit_token_sum(tokens) / tokens


def weighted_latency(latency_us: dict, sched: Schedule, gen_len: int):
    """``weighted_gpu_latency`` (perf.py:231-250): decode-step-weighted mean of per-precision
    latencies and its speedup over the fp16 (16) entry."""
    if gen_len < 1:
        raise InputError(f"gen_len must be >= 1, got {gen_len}")
    table = {int(k): float(v) for k, v in latency_us.items()}
    if 16 not in table:
        raise InputError("latency table lacks the fp16 (16) entry")
    counts = {}
    for i in range(gen_len):
        p = sched.precision_at(i)
        if p not in table:
            raise InputError(f"latency table lacks precision {p}")
        counts[p] = counts.get(p, 0) + 1
    if len(counts) == 1:
        w = table[next(iter(counts))]
    else:
        w = sum(n * table[p] for p, n in counts.items()) / gen_len
    return w, table[16] / w
