"""Oracle restatement of the toy LLaMA-style decoder (reference ``pkg/src/pmpd/tinylm.py``).

TEST INFRASTRUCTURE ONLY.  float64 numpy forward pass, KV cache, greedy
sampling and the generation loop with its per-token precision hook
(SURVEY §8a rows A9-A15).  Used by tests to check the B200 device model.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import quant
from .errors import ConfigError, ContractViolation, InputError
from .rng import named_rng
from .schedule import Schedule

FULL = 16  # tinylm.py:31, the full-precision sentinel


@dataclass(frozen=True)
class Config:
    """``ModelConfig`` (tinylm.py:86-116)."""
    n_layers: int
    n_heads: int
    d_model: int
    d_ff: int
    vocab_size: int = 257
    max_context: int = 512
    rope_theta: float = 10000.0

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads


def weight_shapes(cfg: Config):
    """``_weight_shapes`` (tinylm.py:119-127): matrices stored (d_in, d_out), applied as ``x @ W``."""
    d, f = cfg.d_model, cfg.d_ff
    out = [("embed", (cfg.vocab_size, d))]
    for i in range(cfg.n_layers):
        pre = f"layers.{i}."
        out += [(pre + "wq", (d, d)), (pre + "wk", (d, d)), (pre + "wv", (d, d)), (pre + "wo", (d, d)),
                (pre + "w_up", (d, 2 * f)), (pre + "w_down", (f, d))]
    out.append(("head", (d, cfg.vocab_size)))
    return out


def norm_names(cfg: Config):
    """``_norm_names`` (tinylm.py:130-135)."""
    names = []
    for i in range(cfg.n_layers):
        names += [f"layers.{i}.norm_attn", f"layers.{i}.norm_mlp"]
    return names + ["final_norm"]


def random_weights(cfg: Config, seed: int, std: float | None = None):
    """``random_weights`` (tinylm.py:138-145): one ``named_rng(seed, "weights")`` stream,
    N(0, 1/d_model) per matrix in ``weight_shapes`` order, cast to f32; unit norm gains.
    ``std`` overrides the scale (BASELINE configs use 0.02)."""
    rng = named_rng(seed, "weights")
    s = 1.0 / math.sqrt(cfg.d_model) if std is None else float(std)
    full = {n: rng.normal(0.0, s, shp).astype(np.float32) for n, shp in weight_shapes(cfg)}
    norms = {n: np.ones(cfg.d_model, dtype=np.float32) for n in norm_names(cfg)}
    return full, norms


class Model:
    """``ModelVariants`` (tinylm.py:151-263) without the LRU: ``weights(name, p)``
    dequantizes on demand (memoized per (name, p))."""

    def __init__(self, cfg: Config, precisions, tensors: dict, norms: dict, full: dict | None = None):
        self.config = cfg
        self.precisions = tuple(precisions)
        self.tensors = tensors
        self.norms = {k: np.asarray(v, dtype=np.float64) for k, v in norms.items()}
        self.full = full
        self._memo = {}

    @classmethod
    def from_random(cls, cfg: Config, precisions, seed: int, group_size: int = 64, std=None):
        """``ModelVariants.from_random`` (tinylm.py:184-192)."""
        full, norms = random_weights(cfg, seed, std)
        p_max = max(precisions)
        tensors = {n: quant.quantize(w, p_max, group_size) for n, w in full.items()}
        return cls(cfg, precisions, tensors, norms, full)

    def allowed(self) -> set:
        """tinylm.py:259-263."""
        s = set(self.precisions)
        if self.full is not None:
            s.add(FULL)
        return s

    def weights(self, name: str, p: int) -> np.ndarray:
        """tinylm.py:201-231."""
        if p == FULL:
            if self.full is None:
                raise ConfigError("full-precision weights unavailable")
            return self.full[name].astype(np.float64)
        if p not in self.precisions:
            raise ContractViolation(f"precision {p} not in declared set {list(self.precisions)}")
        key = (name, p)
        if key not in self._memo:
            self._memo[key] = quant.dequantize(self.tensors[name], p)
        return self._memo[key]


class Cache:
    """``KVCache`` (tinylm.py:272-286): post-RoPE K and V rows, flattened heads."""

    def __init__(self, n_layers, width, capacity):
        self.k = np.zeros((n_layers, capacity, width))
        self.v = np.zeros((n_layers, capacity, width))
        self.T = 0

    def layer_kv(self, layer):
        return self.k[layer, :self.T], self.v[layer, :self.T]


def rmsnorm(x, g, eps=1e-6):
    """tinylm.py:293-295."""
    return x / np.sqrt((x * x).mean(axis=-1, keepdims=True) + eps) * g


def rope_tables(positions, d_head, theta):
    """tinylm.py:308-311: ``inv_freq = theta^(-arange(0,d_h,2)/d_h)``; angles in float64."""
    inv = theta ** (-np.arange(0, d_head, 2) / d_head)
    ang = np.outer(positions, inv)
    return np.cos(ang), np.sin(ang)


def rope(x, c, s):
    """Rotate-half RoPE (tinylm.py:314-319); x is [n, heads, d_head]."""
    h = x.shape[-1] // 2
    a, b = x[..., :h], x[..., h:]
    c, s = c[:, None, :], s[:, None, :]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def forward(model: Model, p: int, tokens, cache: Cache) -> np.ndarray:
    """``_forward`` (tinylm.py:322-368): logits for every new position, extending ``cache``."""
    cfg = model.config
    n, t0 = len(tokens), cache.T
    if t0 + n > cfg.max_context:
        raise InputError(f"sequence length {t0 + n} exceeds max_context {cfg.max_context}")
    ids = np.asarray(tokens, dtype=np.int64)
    if ids.size and (ids.min() < 0 or ids.max() >= cfg.vocab_size):
        raise InputError(f"token id outside vocabulary of size {cfg.vocab_size}")
    H, dh = cfg.n_heads, cfg.d_head
    x = model.weights("embed", p)[ids]
    c, s = rope_tables(np.arange(t0, t0 + n, dtype=np.float64), dh, cfg.rope_theta)
    scale = 1.0 / math.sqrt(dh)
    T = t0 + n
    causal = np.arange(T)[None, :] <= (t0 + np.arange(n))[:, None]
    for i in range(cfg.n_layers):
        pre = f"layers.{i}."
        h = rmsnorm(x, model.norms[pre + "norm_attn"])
        q = rope((h @ model.weights(pre + "wq", p)).reshape(n, H, dh), c, s)
        k = rope((h @ model.weights(pre + "wk", p)).reshape(n, H, dh), c, s)
        v = h @ model.weights(pre + "wv", p)
        cache.k[i, t0:T] = k.reshape(n, -1)
        cache.v[i, t0:T] = v
        K = cache.k[i, :T].reshape(T, H, dh)
        V = cache.v[i, :T].reshape(T, H, dh)
        sc = np.einsum("nhd,thd->hnt", q, K) * scale
        if n > 1:
            sc = np.where(causal[None], sc, -np.inf)
        sc = np.exp(sc - sc.max(axis=-1, keepdims=True))
        a = sc / sc.sum(axis=-1, keepdims=True)
        ctx = np.einsum("hnt,thd->nhd", a, V).reshape(n, cfg.d_model)
        x = x + ctx @ model.weights(pre + "wo", p)
        h2 = rmsnorm(x, model.norms[pre + "norm_mlp"])
        u = h2 @ model.weights(pre + "w_up", p)
        g, up = u[:, :cfg.d_ff], u[:, cfg.d_ff:]
        x = x + (g / (1.0 + np.exp(-g)) * up) @ model.weights(pre + "w_down", p)
    cache.T = T
    return rmsnorm(x, model.norms["final_norm"]) @ model.weights("head", p)


def _check_p(model, p):
    if p not in model.allowed():
        raise ContractViolation(f"precision {p} not in the model's set {sorted(model.allowed())}")


def prefill(model: Model, p: int, prompt):
    """tinylm.py:377-388."""
    if len(prompt) == 0:
        raise InputError("prompt is empty")
    if len(prompt) >= model.config.max_context:
        raise InputError(f"prompt length {len(prompt)} must be < max_context {model.config.max_context}")
    _check_p(model, p)
    cfg = model.config
    cache = Cache(cfg.n_layers, cfg.d_model, cfg.max_context)
    return forward(model, p, prompt, cache)[-1], cache


def decode_step(model: Model, p: int, token: int, cache: Cache):
    """tinylm.py:391-400."""
    if cache.T < 1:
        raise InputError("decode_step requires a prefilled cache")
    if cache.T >= model.config.max_context:
        raise InputError(f"context window full at {cache.T} tokens")
    _check_p(model, p)
    return forward(model, p, [token], cache)[-1], cache


def forward_full(model: Model, p: int, tokens):
    """tinylm.py:403-408."""
    _check_p(model, p)
    cfg = model.config
    return forward(model, p, tokens, Cache(cfg.n_layers, cfg.d_model, cfg.max_context))


def greedy(logits) -> int:
    """Greedy branch of ``sample`` (tinylm.py:422-429): argmax, lowest index on ties."""
    logits = np.asarray(logits, dtype=np.float64)
    if not np.isfinite(logits).all():
        raise InputError("logits contain non-finite values")
    return int(np.argmax(logits))


def generate(model: Model, prompt, scheduler, eos_id=None, max_new=64, keep_logits=False):
    """``generate`` (tinylm.py:475-523), greedy sampling.

    ``scheduler`` follows the reference duck type (``p_prefill``, ``horizon``,
    ``resolve(cache) -> Schedule``).  Returns ``(tokens, precisions, schedule,
    termination, logits_list)``; token ``j`` is attributed ``precision_at(j)``
    and decode step ``i`` (consuming token ``i``) runs at ``precision_at(i)``.
    """
    eos = model.config.vocab_size - 1 if eos_id is None else eos_id
    if max_new < 1:
        raise InputError(f"max_new must be >= 1, got {max_new}")
    if max_new > scheduler.horizon:
        raise InputError(f"max_new {max_new} exceeds the schedule horizon {scheduler.horizon}")
    logits, cache = prefill(model, scheduler.p_prefill, prompt)
    sched = scheduler.resolve(cache)
    bad = sched.validate()
    if bad:
        raise ContractViolation("scheduler produced an invalid schedule: " + "; ".join(bad))
    for p in sched.precisions:
        if p not in model.allowed():
            raise ContractViolation(f"schedule uses precision {p} outside the model's set")
    toks, precs, kept = [], [], []
    toks.append(greedy(logits))
    precs.append(sched.precision_at(0))
    if keep_logits:
        kept.append(logits)
    while toks[-1] != eos and len(toks) < max_new:
        i = len(toks) - 1
        logits, cache = decode_step(model, sched.precision_at(i), toks[-1], cache)
        toks.append(greedy(logits))
        precs.append(sched.precision_at(len(toks) - 1))
        if keep_logits:
            kept.append(logits)
    term = "eos" if toks[-1] == eos else "length"
    return toks, precs, sched, term, kept


class StaticSched:
    """``StaticScheduler`` / ``FixedScheduler`` (schedule.py:213-236)."""

    def __init__(self, sched: Schedule):
        self.schedule = sched
        self.p_prefill = sched.p_prefill
        self.horizon = sched.horizon

    def resolve(self, cache):
        return self.schedule

    @classmethod
    def fixed(cls, p, horizon=1 << 30, p_prefill=None):
        return cls(Schedule.constant(p, horizon, p_prefill))
