"""Prompt-adaptive learned switch predictor (drop-in for the inference part of ``pmpd.learnsched``).

The network is the reference's (learnsched.py:32-110): a learned query attends
over the prefilled KV cache of one block, the pooled value feeds a
one-hidden-layer ReLU MLP and the argmax class picks the low precision's
switch point on a grid.  Inference runs on the device (``pmpd_learned_predict``)
straight from the f16 KV cache and writes the two-phase schedule into the
device switch-point table, so no host round trip sits between prefill and the
first decode step.  Label generation and training are offline (out of scope).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _capi
from .errors import ConfigError, FormatError
from .schedule import PrecisionSchedule, SwitchGrid
from .util import named_rng

NET_TAG = "pmpd-sched-v1"


class SchedulerNet:
    """Learned query + MLP classifier over candidate switch points (learnsched.py:32-110)."""

    def __init__(self, q, w1, b1, w2, b2, grid: SwitchGrid, p_high: int, p_low: int, feature_block: int = -1):
        self.q = np.asarray(q, dtype=np.float64)
        self.w1 = np.asarray(w1, dtype=np.float64)
        self.b1 = np.asarray(b1, dtype=np.float64)
        self.w2 = np.asarray(w2, dtype=np.float64)
        self.b2 = np.asarray(b2, dtype=np.float64)
        self.grid = grid
        self.p_high, self.p_low = int(p_high), int(p_low)
        self.feature_block = int(feature_block)
        if self.w1.shape != (self.hidden, self.d_v) or self.b1.shape != (self.hidden,):
            raise ConfigError("hidden layer shapes are inconsistent")
        if self.w2.shape != (self.n_classes, self.hidden) or self.b2.shape != (self.n_classes,):
            raise ConfigError("output layer shapes are inconsistent")
        if self.n_classes != grid.n:
            raise ConfigError(f"net has {self.n_classes} classes but grid has {grid.n} points")
        for name, arr in self.params().items():
            if not np.all(np.isfinite(arr)):
                raise ConfigError(f"parameter {name} contains non-finite values")
        self._dev = None

    @property
    def d_k(self) -> int:
        return self.q.shape[0]

    @property
    def d_v(self) -> int:
        return self.w1.shape[1]

    @property
    def hidden(self) -> int:
        return self.w1.shape[0]

    @property
    def n_classes(self) -> int:
        return self.w2.shape[0]

    def params(self) -> dict:
        return {"q": self.q, "w1": self.w1, "b1": self.b1, "w2": self.w2, "b2": self.b2}

    @classmethod
    def init(cls, d_k: int, d_v: int, hidden: int, grid: SwitchGrid, p_high: int, p_low: int, seed: int = 0,
             feature_block: int = -1) -> "SchedulerNet":
        """Same named RNG stream and draw order as the reference (learnsched.py:76-85)."""
        rng = named_rng(seed, "scheduler-init")
        q = rng.normal(0.0, 1.0 / np.sqrt(d_k), d_k)
        w1 = rng.normal(0.0, np.sqrt(2.0 / d_v), (hidden, d_v))
        w2 = rng.normal(0.0, np.sqrt(2.0 / hidden), (grid.n, hidden))
        return cls(q, w1, np.zeros(hidden), w2, np.zeros(grid.n), grid, p_high, p_low, feature_block)

    def to_json(self) -> dict:
        def arr(a):
            return {"shape": list(a.shape), "data": [float(x) for x in a.ravel()]}
        return {"tag": NET_TAG, "grid": {"n": self.grid.n, "OL": self.grid.horizon}, "p_high": self.p_high,
                "p_low": self.p_low, "feature_block": self.feature_block, "q": arr(self.q), "w1": arr(self.w1),
                "b1": arr(self.b1), "w2": arr(self.w2), "b2": arr(self.b2)}

    @classmethod
    def from_json(cls, obj: dict) -> "SchedulerNet":
        if obj.get("tag") != NET_TAG:
            raise FormatError(f"not a scheduler net artifact (tag {obj.get('tag')!r})")

        def arr(entry):
            return np.asarray(entry["data"], dtype=np.float64).reshape(entry["shape"])
        try:
            grid = SwitchGrid(int(obj["grid"]["n"]), int(obj["grid"]["OL"]))
            return cls(arr(obj["q"]), arr(obj["w1"]), arr(obj["b1"]), arr(obj["w2"]), arr(obj["b2"]), grid,
                       obj["p_high"], obj["p_low"], obj.get("feature_block", -1))
        except (KeyError, TypeError, ValueError) as exc:
            raise FormatError(f"malformed scheduler net JSON: {exc}") from exc

    # ------------------------------------------------------------------ device copy
    def device(self):
        if self._dev is None:
            f = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda").contiguous()  # noqa: E731
            self._dev = {"q": f(self.q), "w1": f(self.w1), "b1": f(self.b1), "w2": f(self.w2), "b2": f(self.b2),
                         "grid": torch.tensor(self.grid.points, dtype=torch.int32, device="cuda"),
                         "dbg": torch.zeros(self.n_classes, dtype=torch.float32, device="cuda")}
        return self._dev


def _check_kv(net: SchedulerNet, K: torch.Tensor, V: torch.Tensor):
    if K.dim() != 2 or V.dim() != 2 or K.shape[0] != V.shape[0] or K.shape[0] < 1:
        raise ConfigError(f"K {tuple(K.shape)} and V {tuple(V.shape)} must share a non-empty time axis")
    if K.shape[1] != net.d_k or V.shape[1] != net.d_v:
        raise ConfigError(f"K width {K.shape[1]} / V width {V.shape[1]} do not match "
                          f"net dims ({net.d_k}, {net.d_v})")


def device_predict(net: SchedulerNet, K16: torch.Tensor, V16: torch.Tensor, ldkv: int, T_dev: torch.Tensor,
                   max_T: int, sched_dev: torch.Tensor) -> None:
    """Enqueue the device predictor: writes {p_high: 0, p_low: grid[argmax]} into ``sched_dev``."""
    d = net.device()
    _capi.call("pmpd_learned_predict", K16.data_ptr(), V16.data_ptr(), ldkv, T_dev.data_ptr(), max_T, net.d_k,
               net.d_v, net.hidden, net.n_classes, d["q"].data_ptr(), d["w1"].data_ptr(), d["b1"].data_ptr(),
               d["w2"].data_ptr(), d["b2"].data_ptr(), d["grid"].data_ptr(), net.p_high, net.p_low,
               sched_dev.data_ptr(), d["dbg"].data_ptr(), torch.cuda.current_stream().cuda_stream)


def _as_f16_kv(net, K, V):
    K = torch.as_tensor(np.asarray(K) if not isinstance(K, torch.Tensor) else K)
    V = torch.as_tensor(np.asarray(V) if not isinstance(V, torch.Tensor) else V)
    _check_kv(net, K, V)
    return K.to("cuda", torch.float16).contiguous(), V.to("cuda", torch.float16).contiguous()


def class_logits(net: SchedulerNet, K, V) -> np.ndarray:
    """Class scores of the MLP (learnsched.py:146-148), computed on the device from f16 K/V."""
    K16, V16 = _as_f16_kv(net, K, V)
    T = torch.tensor([K16.shape[0]], dtype=torch.int32, device="cuda")
    table = torch.zeros(16, dtype=torch.int32, device="cuda")
    device_predict(net, K16, V16, net.d_k, T, K16.shape[0], table)
    return net.device()["dbg"].double().cpu().numpy()


def predict_schedule(net: SchedulerNet, cache, p_prefill: int | None = None) -> PrecisionSchedule:
    """Map a prefilled cache to a valid two-precision schedule (learnsched.py:151-160).

    ``cache`` is a device ``KVCache`` (the prediction reads its f16 rows in place)
    or any object with ``layer_kv(layer) -> (K, V)``.
    """
    table = torch.zeros(16, dtype=torch.int32, device="cuda")
    if hasattr(cache, "device_kv"):
        K16, V16, T_dev, cap = cache.device_kv(net.feature_block)
        device_predict(net, K16, V16, K16.stride(0), T_dev, cap, table)
    else:
        K, V = cache.layer_kv(net.feature_block)
        K16, V16 = _as_f16_kv(net, K, V)
        T = torch.tensor([K16.shape[0]], dtype=torch.int32, device="cuda")
        device_predict(net, K16, V16, net.d_k, T, K16.shape[0], table)
    switch = int(table[3].item())
    return PrecisionSchedule.two_phase(net.p_high, net.p_low, switch, net.grid.horizon, p_prefill)


def pool_kv(net: SchedulerNet, K, V) -> np.ndarray:
    """Attention-pooled value vector (learnsched.py:140-143), float64 on the host side of the API."""
    K16, V16 = _as_f16_kv(net, K, V)
    s = (K16.float() @ net.device()["q"]) / float(np.sqrt(net.d_k))
    a = torch.softmax(s, dim=0)
    return (a @ V16.float()).double().cpu().numpy()


class LearnedScheduler:
    """Adapter giving the generation loop a per-prompt predicted schedule (learnsched.py:163-175).

    ``resolve_device`` is the hot-path entry: it enqueues the predictor so the
    schedule lands in the device table with no host synchronisation.
    """

    def __init__(self, net: SchedulerNet, p_prefill: int | None = None):
        self.net = net
        self.p_prefill = net.p_high if p_prefill is None else int(p_prefill)

    @property
    def horizon(self) -> int:
        return self.net.grid.horizon

    def resolve(self, cache) -> PrecisionSchedule:
        return predict_schedule(self.net, cache, self.p_prefill)

    def resolve_device(self, cache, sched_dev: torch.Tensor) -> None:
        K16, V16, T_dev, cap = cache.device_kv(self.net.feature_block)
        device_predict(self.net, K16, V16, K16.stride(0), T_dev, cap, sched_dev)

    def schedule_from_table(self, table_host) -> PrecisionSchedule:
        return PrecisionSchedule.two_phase(self.net.p_high, self.net.p_low, int(table_host[3]), self.horizon,
                                           self.p_prefill)
