"""Oracle restatement of the learned (prompt-adaptive) switch predictor
(reference ``pkg/src/pmpd/learnsched.py:32-175``, inference only).

TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np

from .errors import ConfigError
from .rng import named_rng
from .schedule import Schedule, grid_points


class Net:
    """``SchedulerNet`` parameters: query ``q`` (d_k), ``w1`` (H, d_v), ``b1`` (H), ``w2`` (N, H), ``b2`` (N)."""

    def __init__(self, q, w1, b1, w2, b2, grid_n, horizon, p_high, p_low, feature_block=-1):
        self.q, self.w1, self.b1 = (np.asarray(a, dtype=np.float64) for a in (q, w1, b1))
        self.w2, self.b2 = (np.asarray(a, dtype=np.float64) for a in (w2, b2))
        self.points = grid_points(grid_n, horizon)
        self.horizon = int(horizon)
        self.p_high, self.p_low = int(p_high), int(p_low)
        self.feature_block = int(feature_block)

    @classmethod
    def init(cls, d_k, d_v, hidden, grid_n, horizon, p_high, p_low, seed=0, feature_block=-1):
        """``SchedulerNet.init`` (learnsched.py:76-85): ``named_rng(seed, "scheduler-init")`` draws
        q ~ N(0, 1/sqrt(d_k)), w1 ~ N(0, sqrt(2/d_v)), w2 ~ N(0, sqrt(2/H)); zero biases."""
        r = named_rng(seed, "scheduler-init")
        q = r.normal(0.0, 1.0 / np.sqrt(d_k), d_k)
        w1 = r.normal(0.0, np.sqrt(2.0 / d_v), (hidden, d_v))
        w2 = r.normal(0.0, np.sqrt(2.0 / hidden), (grid_n, hidden))
        return cls(q, w1, np.zeros(hidden), w2, np.zeros(grid_n), grid_n, horizon, p_high, p_low,
                   feature_block)


def _check(net: Net, K, V):
    """``_checked`` (learnsched.py:128-137)."""
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    if K.ndim != 2 or V.ndim != 2 or K.shape[0] != V.shape[0] or K.shape[0] < 1:
        raise ConfigError(f"K {K.shape} and V {V.shape} must share a non-empty time axis")
    if K.shape[1] != net.q.shape[0] or V.shape[1] != net.w1.shape[1]:
        raise ConfigError("K/V widths do not match net dims")
    return K, V


def pool(net: Net, K, V) -> np.ndarray:
    """``pool_kv`` (learnsched.py:118-122,140-143): softmax(K q / sqrt(d_k)) V."""
    K, V = _check(net, K, V)
    s = K @ net.q / np.sqrt(net.q.shape[0])
    e = np.exp(s - s.max())
    return (e / e.sum()) @ V


def class_logits(net: Net, K, V) -> np.ndarray:
    """learnsched.py:122-125,146-148: relu(W1 pooled + b1) -> W2 h + b2."""
    h = np.maximum(net.w1 @ pool(net, K, V) + net.b1, 0.0)
    return net.w2 @ h + net.b2


def predict(net: Net, K, V, p_prefill=None) -> Schedule:
    """``predict_schedule`` (learnsched.py:151-160): argmax (lowest index on ties) picks the
    low precision's switch point on the grid; returns a two-phase schedule."""
    cls = int(np.argmax(class_logits(net, K, V)))
    return Schedule.two_phase(net.p_high, net.p_low, net.points[cls], net.horizon, p_prefill)


class LearnedSched:
    """``LearnedScheduler`` (learnsched.py:163-175)."""

    def __init__(self, net: Net, p_prefill=None):
        self.net = net
        self.p_prefill = net.p_high if p_prefill is None else int(p_prefill)
        self.horizon = net.horizon

    def resolve(self, cache):
        K, V = cache.layer_kv(self.net.feature_block)
        return predict(self.net, K, V, self.p_prefill)
