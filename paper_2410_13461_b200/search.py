"""Offline schedule search on the device.

The reference's offline stages call ``generate`` as a black box (#candidates x #prompts) times:
``solve_static`` scores every grid schedule by Rouge-L against full-precision references
(schedule.py:324-345, 367-416, 443-457) and ``generate_labels`` scores one generation per grid
switch point for every truncated seed prompt (learnsched.py:182-254).  Here those generations run
on the B200: the full-precision references through ``tinylm.generate`` at precision 16 (cuBLAS
fp16 baseline), every candidate schedule through ``tinylm.generate_batch`` (up to 8 prompts per
batch, one CUDA-graph step per token, batched decode GEMVs).  Same API, selection rule, tie
breaks and label rule as the reference; the quality signal is the reference's Rouge-L over token
ids (metrics.py:11-42), restated here because it is the search's objective.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Callable, Iterable, Iterator, Sequence

import numpy as np

from .errors import ConfigError, InputError
from .quant import PrecisionSet
from .schedule import FixedScheduler, PrecisionSchedule, QualityTarget, StaticScheduler, SwitchGrid
from .util import named_rng

MATCH_GUARD = 1e-9  # learnsched.py:29: float guard on the "matches or exceeds" label rule
BATCH = 8           # prompts per generate_batch call (the batched decode GEMV's row limit)


# ------------------------------------------------------------------ Rouge-L (metrics.py:11-42)
def lcs_len(a: Sequence, b: Sequence) -> int:
    """Longest-common-subsequence length (metrics.py:11-26), O(|a||b|) time, O(min) space."""
    if len(b) > len(a):
        a, b = b, a
    if not b:
        return 0
    prev = [0] * (len(b) + 1)
    for x in a:
        cur = [0] * (len(b) + 1)
        for j, y in enumerate(b, start=1):
            cur[j] = prev[j - 1] + 1 if x == y else max(prev[j], cur[j - 1])
        prev = cur
    return prev[len(b)]


@dataclass(frozen=True)
class RougeScore:
    precision: float
    recall: float
    f1: float


def rouge_l(candidate: Sequence, reference: Sequence) -> RougeScore:
    """LCS precision / recall / F1; empty sides score 0 (metrics.py:36-42)."""
    lcs = lcs_len(candidate, reference)
    p = lcs / len(candidate) if candidate else 0.0
    r = lcs / len(reference) if reference else 0.0
    f1 = 2 * p * r / (p + r) if p + r > 0 else 0.0
    return RougeScore(p, r, f1)


# ------------------------------------------------------------------ generations on the device
def enumerate_switch_maps(precisions: Sequence[int], points: Sequence[int]) -> Iterator[dict]:
    """Precedence-respecting switch maps, the lower precisions' points drawn from ``points``
    (schedule.py:197-206; the highest precision is pinned to 0)."""
    ps = sorted(set(int(p) for p in precisions), reverse=True)
    lower = ps[1:]
    for combo in itertools.combinations_with_replacement(sorted(points), len(lower)):
        st = {ps[0]: 0}
        st.update(dict(zip(lower, combo)))
        yield st


def _eos(model, eos_id):
    return model.config.vocab_size - 1 if eos_id is None else eos_id


def reference_outputs(model, prompts, max_new: int, eos_id: int | None = None):
    """Greedy full-precision generations (schedule.py:324-345): prompts whose reference is empty
    or just EOS are dropped and counted.  Returns (kept prompts, references, eos)."""
    from .tinylm import FULL_PRECISION, generate
    eos = _eos(model, eos_id)
    kept, refs = [], []
    for prompt in prompts:
        out = generate(model, list(prompt), FixedScheduler(FULL_PRECISION), eos_id=eos, max_new=max_new).output_tokens
        if not out or out == [eos]:
            continue
        kept.append(list(prompt))
        refs.append(out)
    if not kept:
        raise InputError("every calibration/validation prompt produced an empty reference")
    return kept, refs, eos


def batched_outputs(model, prompts, schedule: PrecisionSchedule, eos: int, max_new: int) -> list:
    """Greedy generations of every prompt under one static schedule, BATCH prompts per
    ``generate_batch`` (each trace equals ``generate``'s for that prompt)."""
    from .tinylm import generate_batch
    out = []
    for i in range(0, len(prompts), BATCH):
        chunk = prompts[i:i + BATCH]
        out += [t.output_tokens for t in generate_batch(model, chunk, StaticScheduler(schedule), eos_id=eos,
                                                       max_new=max_new)]
    return out


def device_quality_fn(model, valset, horizon: int, eos_id: int | None = None) -> Callable:
    """``_generation_quality_fn`` (schedule.py:443-457) on the device: mean Rouge-L F1 of each
    schedule's generations against the full-precision references."""
    kept, refs, eos = reference_outputs(model, valset, horizon, eos_id)

    def quality(schedule: PrecisionSchedule) -> float:
        outs = batched_outputs(model, kept, schedule, eos, horizon)
        return sum(rouge_l(o, r).f1 for o, r in zip(outs, refs)) / len(kept)

    return quality


# ------------------------------------------------------------------ static search (schedule.py:367-416)
def select_best(precisions: PrecisionSet, p_prefill: int, horizon: int, candidates: Iterable[dict],
                quality_fn: Callable, target: QualityTarget, details_out: list | None = None) -> PrecisionSchedule:
    """Among feasible candidates the fewest bit-tokens, ties to earlier switches of the higher
    precisions; none feasible -> the all-high schedule flagged infeasible (schedule.py:367-393)."""
    desc = precisions.precisions
    best_key, best = None, None
    for st in candidates:
        sched = PrecisionSchedule(precisions, p_prefill, st, horizon)
        quality = float(quality_fn(sched))
        feasible = quality >= target.floor
        bits = sched.bit_token_sum()
        if details_out is not None:
            details_out.append({"st": {str(p): st[p] for p in desc}, "quality": quality, "bit_token_sum": bits,
                                "feasible": feasible})
        if not feasible:
            continue
        key = (bits, tuple(st[p] for p in desc))
        if best_key is None or key < best_key:
            best_key, best = key, sched
    if best is None:
        st = {p: (0 if p == desc[0] else horizon) for p in desc}
        return PrecisionSchedule(precisions, p_prefill, st, horizon, feasible=False)
    return best


def solve_static(model, valset, target: QualityTarget, grid: SwitchGrid, *, precisions: PrecisionSet,
                 p_prefill: int, eos_id: int | None = None, quality_fn: Callable | None = None,
                 details_out: list | None = None) -> PrecisionSchedule:
    """Grid-restricted offline schedule search (schedule.py:396-416), generations on the device."""
    if quality_fn is None:
        if not valset:
            raise InputError("validation prompt set is empty")
        quality_fn = device_quality_fn(model, valset, grid.horizon, eos_id)
    candidates = enumerate_switch_maps(precisions.precisions, grid.points)
    return select_best(precisions, p_prefill, grid.horizon, candidates, quality_fn, target, details_out)


# ------------------------------------------------------------------ label generation (learnsched.py:182-254)
@dataclass
class LabeledExample:
    """Pooling inputs from one prefill plus the minimal adequate grid index (learnsched.py:182-189)."""
    k: np.ndarray  # [T, d_k] float32
    v: np.ndarray  # [T, d_v] float32
    label: int
    scores: list = field(default_factory=list)
    prompt_len: int = 0


def label_from_scores(scores: Sequence[float]) -> int:
    """Smallest grid index whose quality matches the all-high run's (learnsched.py:192-199)."""
    threshold = scores[-1] - MATCH_GUARD
    for j, s in enumerate(scores):
        if s >= threshold:
            return j
    return len(scores) - 1


def generate_labels(model, seed_prompts, grid: SwitchGrid, p_high: int, p_low: int, *,
                    p_prefill: int | None = None, eos_id: int | None = None, seed: int = 0,
                    feature_block: int = -1):
    """Training set of the learned scheduler (learnsched.py:203-254): truncate each seed prompt
    at a seeded random point, score one generation per grid switch point against the
    full-precision reference, keep the prefill K/V of the feature block.  The grid-point
    generations of all kept prompts run batched on the device, one batch per grid point."""
    from .tinylm import prefill
    if not seed_prompts:
        raise InputError("seed prompt set is empty")
    rng = named_rng(seed, "truncation")
    eos = _eos(model, eos_id)
    pf = p_high if p_prefill is None else p_prefill
    horizon = grid.horizon
    max_prompt = model.config.max_context - horizon
    if max_prompt < 1:
        raise ConfigError(f"grid horizon {horizon} leaves no room for prompts in a "
                          f"max_context of {model.config.max_context}")
    prompts = []
    for toks in seed_prompts:
        toks = list(toks)
        cut = int(rng.integers(1, len(toks) + 1))  # drawn before any skip
        prompts.append(toks[: max(1, min(cut, max_prompt))])
    kept, refs = [], []
    skipped = 0
    for prompt in prompts:
        try:
            k, r, _ = reference_outputs(model, [prompt], horizon, eos)
        except InputError:
            skipped += 1
            continue
        kept.append(prompt)
        refs.append(r[0])
    scores = [[] for _ in kept]
    for point in grid.points:
        sched = PrecisionSchedule.two_phase(p_high, p_low, point, horizon, pf)
        for i, out in enumerate(batched_outputs(model, kept, sched, eos, horizon)):
            scores[i].append(rouge_l(out, refs[i]).f1)
    examples = []
    for prompt, sc in zip(kept, scores):
        _, cache = prefill(model, pf, prompt)
        K, V = cache.layer_kv(feature_block)
        examples.append(LabeledExample(K.astype(np.float32), V.astype(np.float32), label_from_scores(sc), sc,
                                       len(prompt)))
    return examples, skipped
