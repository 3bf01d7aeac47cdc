"""Device-resident LLaMA-style decoder with per-token weight precision (drop-in for ``pmpd.tinylm``).

Same public names, arguments, validation and error classes as the reference
(pkg/src/pmpd/tinylm.py), re-designed for the B200:

* weights stay in HBM as nested bit planes (``quant.QuantizedTensor``), packed
  once into the GEMV's tile layout; q|k|v are fused into one GEMV;
* every linear layer is ``pmpd_gemv`` reading only planes ``0..p-1`` with ``p``
  read from device memory; glue (RMSNorm, RoPE, attention, SiLU, argmax) is
  CUDA in ``model.cu``; the residual stream is f32, the KV cache f16;
* ``generate`` resolves the schedule on device (static table upload or the
  learned predictor) and replays ONE CUDA graph per decode step whose first
  node is the precision hook ``pmpd_sched_step`` — no host sync per token;
* precision 16 is the fp16 baseline (cuBLAS), as the paper's fp16 runs.

Results match the reference CPU implementation within the north-star
tolerances (tests/test_gpu_model.py): logits rel-L2 <= 1e-2, identical greedy
tokens where the reference's top-2 margin exceeds the f16/f32 error.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import threading
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _capi
from .errors import ConfigError, ContractViolation, FormatError, InputError
from .linear import Workspace, gemm, gemv, gemv_fused, raise_device_status, workspace_bytes
from .quant import BitPlaneStore, PrecisionSet, QuantizedTensor, dequantize, quantize_tensor, read_model, \
    write_model
from .schedule import PrecisionSchedule
from .util import named_rng

FULL_PRECISION = 16
BYTE_EOS_ID = 256
BYTE_VOCAB_SIZE = 257
INIT_SCHEME = "gaussian-inv-sqrt-dmodel"
GEMV_MAX_ROWS = 8


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass(frozen=True)
class ModelConfig:
    """tinylm.py:86-116."""
    n_layers: int
    n_heads: int
    d_model: int
    d_ff: int
    vocab_size: int = BYTE_VOCAB_SIZE
    max_context: int = 512
    rope_theta: float = 10000.0

    def __post_init__(self):
        if self.d_model % self.n_heads != 0:
            raise ConfigError(f"d_model {self.d_model} not divisible by n_heads {self.n_heads}")
        if (self.d_model // self.n_heads) % 2 != 0:
            raise ConfigError("head width must be even for rotary embeddings")
        if self.max_context < 2:
            raise ConfigError(f"max_context must be >= 2, got {self.max_context}")
        if self.vocab_size < 2:
            raise ConfigError(f"vocab_size must be >= 2, got {self.vocab_size}")
        if min(self.n_layers, self.d_ff) < 1:
            raise ConfigError("n_layers and d_ff must be >= 1")

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads

    def to_json(self) -> dict:
        return {"n_layers": self.n_layers, "n_heads": self.n_heads, "d_model": self.d_model, "d_ff": self.d_ff,
                "vocab_size": self.vocab_size, "max_context": self.max_context, "rope_theta": self.rope_theta}


def _weight_shapes(cfg: ModelConfig):
    d, ff = cfg.d_model, cfg.d_ff
    shapes = [("embed", (cfg.vocab_size, d))]
    for i in range(cfg.n_layers):
        shapes += [(f"layers.{i}.wq", (d, d)), (f"layers.{i}.wk", (d, d)), (f"layers.{i}.wv", (d, d)),
                   (f"layers.{i}.wo", (d, d)), (f"layers.{i}.w_up", (d, 2 * ff)), (f"layers.{i}.w_down", (ff, d))]
    shapes.append(("head", (d, cfg.vocab_size)))
    return shapes


def _norm_names(cfg: ModelConfig):
    names = []
    for i in range(cfg.n_layers):
        names += [f"layers.{i}.norm_attn", f"layers.{i}.norm_mlp"]
    names.append("final_norm")
    return names


def random_weights(cfg: ModelConfig, seed: int, std: float | None = None):
    """Seeded Gaussian weights (tinylm.py:138-145): same RNG stream and order as the reference;
    ``std`` overrides the 1/sqrt(d_model) scale (BASELINE configs use 0.02)."""
    rng = named_rng(seed, "weights")
    scale = 1.0 / math.sqrt(cfg.d_model) if std is None else float(std)
    weights = {name: rng.normal(0.0, scale, shape).astype(np.float32) for name, shape in _weight_shapes(cfg)}
    norms = {name: np.ones(cfg.d_model, dtype=np.float32) for name in _norm_names(cfg)}
    return weights, norms


class SeededFullWeights:
    """Precision-16 originals of a model saved with its init seed (tinylm.py:244-257 regenerates
    them with ``random_weights``), produced lazily on first use, tensor by tensor in the reference's
    RNG order and kept on the device: the host never holds more than one f32 tensor."""

    def __init__(self, config: ModelConfig, seed: int, std: float | None = None):
        self.config, self.seed, self.std = config, int(seed), std
        self._dev = None
        self._lock = threading.Lock()

    def _materialize(self) -> dict:
        with self._lock:
            if self._dev is None:
                rng = named_rng(self.seed, "weights")
                scale = 1.0 / math.sqrt(self.config.d_model) if self.std is None else float(self.std)
                dev = {}
                for name, shape in _weight_shapes(self.config):
                    w = rng.normal(0.0, scale, shape).astype(np.float32)
                    dev[name] = torch.from_numpy(w).to("cuda")
                    del w
                self._dev = dev
            return self._dev

    def __getitem__(self, name):
        return self._materialize()[name]

    def items(self):
        return self._materialize().items()


def _concat_cols(parts: list) -> QuantizedTensor:
    """Column-concatenate quantized matrices whose group boundaries align (e.g. wq|wk|wv)."""
    codes = torch.cat([t.codes for t in parts], dim=1).contiguous()
    mins = torch.cat([t.mins for t in parts], dim=1)
    dels = torch.cat([t.deltas for t in parts], dim=1)
    t0 = parts[0]
    store = BitPlaneStore.from_codes(codes, t0.p_max)
    return QuantizedTensor(t0.rows, codes.shape[1], t0.group_size, t0.p_max, mins, dels, store)


class _DeviceWeights:
    """Runtime view of a ModelVariants: packed GEMV layouts, norms, RoPE tables, fp16 baseline."""

    def __init__(self, mv: "ModelVariants"):
        cfg = mv.config
        self.cfg = cfg
        gs = mv.group_size
        self.embed = mv.tensors["embed"].packed(_capi.LAYOUT_REF)
        self.layers = []
        fuse = cfg.d_model % gs == 0
        for i in range(cfg.n_layers):
            t = lambda n: mv.tensors[f"layers.{i}.{n}"]  # noqa: E731
            qkv = [_concat_cols([t("wq"), t("wk"), t("wv")]).packed(_capi.LAYOUT_KN)] if fuse else \
                [t(n).packed(_capi.LAYOUT_KN) for n in ("wq", "wk", "wv")]
            self.layers.append({"qkv": qkv, "wo": t("wo").packed(_capi.LAYOUT_KN),
                                "w_up": t("w_up").packed(_capi.LAYOUT_KN),
                                "w_down": t("w_down").packed(_capi.LAYOUT_KN),
                                "norm_attn": torch.tensor(mv.norms[f"layers.{i}.norm_attn"], device="cuda"),
                                "norm_mlp": torch.tensor(mv.norms[f"layers.{i}.norm_mlp"], device="cuda")})
        self.head = mv.tensors["head"].packed(_capi.LAYOUT_KN)
        self.final_norm = torch.tensor(mv.norms["final_norm"], device="cuda")
        half = cfg.d_head // 2
        inv = cfg.rope_theta ** (-np.arange(0, cfg.d_head, 2) / cfg.d_head)
        ang = np.arange(cfg.max_context, dtype=np.float64)[:, None] * inv[None, :]
        self.cos = torch.tensor(np.cos(ang), dtype=torch.float32, device="cuda").reshape(cfg.max_context, half)
        self.sin = torch.tensor(np.sin(ang), dtype=torch.float32, device="cuda").reshape(cfg.max_context, half)
        pks = [self.head] + [pk for lay in self.layers for pk in lay["qkv"] + [lay["wo"], lay["w_up"],
                                                                              lay["w_down"]]]
        self.ws_bytes = max(workspace_bytes(pk, GEMV_MAX_ROWS) for pk in pks)
        self.fp16 = None
        self._kp = (-(-cfg.d_model // 64) * 64, -(-cfg.d_ff // 64) * 64)
        if mv.full_weights is not None:
            self.fp16 = {n: torch.as_tensor(w, device="cuda").half() for n, w in mv.full_weights.items()}
            # fused q|k|v weight of the fp16 baseline, concatenated once (not per call)
            for i in range(cfg.n_layers):
                names = [f"layers.{i}.{nm}" for nm in ("wq", "wk", "wv")]
                self.fp16["+".join(names)] = torch.cat([self.fp16.pop(nm) for nm in names], dim=1).contiguous()


    def fusable(self, n: int) -> bool:
        """Whether the fused RMSNorm/SwiGLU decode GEMVs accept n rows (the staged-activation path)."""
        return all(kp <= 12288 if n == 1 else n * kp <= 32768 for kp in self._kp)


class ModelVariants:
    """One quantized weight store readable at any precision in its set (tinylm.py:151-263), resident in HBM."""

    def __init__(self, config: ModelConfig, precisions: PrecisionSet, tensors: dict, norms: dict,
                 full_weights: dict | None = None, init_info: dict | None = None, dequant_budget: int = 256 << 20):
        self.config = config
        self.precisions = precisions
        self.tensors = tensors
        self.norms = {k: np.asarray(v, dtype=np.float32) for k, v in norms.items()}
        self.full_weights = full_weights
        self.init_info = init_info
        self._budget = dequant_budget
        self._lock = threading.Lock()
        self._dev = None
        self._engine = None
        for name, shape in dict(_weight_shapes(config)).items():
            t = tensors.get(name)
            if t is None or (t.rows, t.cols) != shape:
                raise ConfigError(f"tensor '{name}' missing or mis-shaped for this config")
        for name in _norm_names(config):
            if name not in self.norms or self.norms[name].shape != (config.d_model,):
                raise ConfigError(f"norm gain '{name}' missing or mis-shaped for this config")
        ps = {t.p_max for t in tensors.values()}
        if ps != {precisions.p_max}:
            raise ConfigError("tensors must be quantized at the precision set's p_max")

    @classmethod
    def from_random(cls, config: ModelConfig, precisions: PrecisionSet, seed: int, group_size: int = 64,
                    std: float | None = None, **kwargs) -> "ModelVariants":
        """tinylm.py:184-192: host-seeded weights (identical to the reference's), device-quantized."""
        full, norms = random_weights(config, seed, std)
        tensors = {name: quantize_tensor(w, precisions.p_max, group_size) for name, w in full.items()}
        info = {"scheme": INIT_SCHEME, "seed": int(seed)} if std is None else None
        return cls(config, precisions, tensors, norms, full_weights=full, init_info=info, **kwargs)

    @property
    def group_size(self) -> int:
        return next(iter(self.tensors.values())).group_size

    def norm(self, name: str) -> np.ndarray:
        return self.norms[name].astype(np.float64)

    def device(self) -> _DeviceWeights:
        with self._lock:
            if self._dev is None:
                self._dev = _DeviceWeights(self)
            return self._dev

    def weights(self, name: str, p: int) -> torch.Tensor:
        """Weights of ``name`` at precision ``p`` as a device f32 (d_in, d_out) tensor; 16 = originals."""
        if p == FULL_PRECISION:
            if self.full_weights is None:
                raise ConfigError("full-precision weights unavailable: model was loaded without "
                                  "an init seed and cannot serve precision 16")
            return torch.as_tensor(self.full_weights[name], device="cuda").clone()
        if p not in self.precisions:
            raise ContractViolation(f"precision {p} not in declared set {list(self.precisions)}")
        return dequantize(self.tensors[name], p)

    def save(self, path) -> None:
        """tinylm.py:233-241: the PMPD v1 file, written tensor by tensor (quant.write_model)."""
        meta = {"config": self.config.to_json(), "precisions": list(self.precisions.precisions),
                "norms": {k: [float(x) for x in v] for k, v in self.norms.items()}}
        if self.init_info is not None:
            meta["init"] = self.init_info
        write_model(path, self.tensors, meta)

    @classmethod
    def load(cls, path, dequant_budget: int = 256 << 20) -> "ModelVariants":
        """tinylm.py:243-257: the file is streamed tensor by tensor into HBM (quant.read_model);
        precision-16 originals of a seeded model are regenerated lazily, on the device."""
        tensors, meta = read_model(path)
        try:
            config = ModelConfig(**meta["config"])
            precisions = PrecisionSet(tuple(meta["precisions"]))
            norms = {k: np.asarray(v, dtype=np.float32) for k, v in meta["norms"].items()}
        except (KeyError, TypeError) as exc:
            raise FormatError(f"weight file metadata incomplete: {exc}") from exc
        full = None
        init = meta.get("init")
        if init is not None and init.get("scheme") == INIT_SCHEME:
            full = SeededFullWeights(config, int(init["seed"]))
        return cls(config, precisions, tensors, norms, full_weights=full, init_info=init,
                   dequant_budget=dequant_budget)

    def allowed_precisions(self) -> set:
        allowed = set(self.precisions.precisions)
        if self.full_weights is not None:
            allowed.add(FULL_PRECISION)
        return allowed


class KVCache:
    """Per-layer post-RoPE K and V rows of every processed token (tinylm.py:272-286), f16 in HBM.

    ``T`` is mirrored on the host for validation; the kernels read the device
    counter ``T_dev`` so a decode step can be replayed as a CUDA graph.
    """

    def __init__(self, n_layers: int, width: int, capacity: int):
        self.k = torch.zeros((n_layers, capacity, width), dtype=torch.float16, device="cuda")
        self.v = torch.zeros((n_layers, capacity, width), dtype=torch.float16, device="cuda")
        self.T_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.T = 0

    @property
    def capacity(self) -> int:
        return self.k.shape[1]

    def layer_kv(self, layer: int):
        """(K, V) of shape [T, width] for one layer as float64 host arrays (reference view)."""
        return (self.k[layer, :self.T].double().cpu().numpy(), self.v[layer, :self.T].double().cpu().numpy())

    def device_kv(self, layer: int):
        """(K, V, T_dev, capacity) device views of one layer for on-device consumers."""
        return self.k[layer], self.v[layer], self.T_dev, self.capacity

    def reset(self) -> None:
        self.T = 0
        self.T_dev.zero_()

    @classmethod
    def batch(cls, n: int, n_layers: int, width: int, capacity: int) -> list:
        """n caches carved from one allocation ([n][layers][capacity][width] f16 K and V, lengths
        int32[n]) so a batched decode step attends over all of them in one launch."""
        k = torch.zeros((n, n_layers, capacity, width), dtype=torch.float16, device="cuda")
        v = torch.zeros_like(k)
        T = torch.zeros(n, dtype=torch.int32, device="cuda")
        out = []
        for j in range(n):
            c = cls.__new__(cls)
            c.k, c.v, c.T_dev, c.T = k[j], v[j], T[j:j + 1], 0
            c.group = (k, v, T, j)
            out.append(c)
        return out


# ---------------------------------------------------------------------------
# forward pass
# ---------------------------------------------------------------------------

class _Buffers:
    """Activation scratch for up to ``rows`` tokens (static addresses: graph-capturable)."""

    def __init__(self, cfg: ModelConfig, rows: int, ws_bytes: int):
        d, ff, V = cfg.d_model, cfg.d_ff, cfg.vocab_size
        dev = "cuda"
        self.rows = rows
        self.x = torch.zeros((rows, d), dtype=torch.float32, device=dev)
        self.h = torch.zeros((rows, d), dtype=torch.float16, device=dev)
        self.qkv = torch.zeros((rows, 3 * d), dtype=torch.float32, device=dev)
        self.q = torch.zeros((rows, d), dtype=torch.float32, device=dev)
        self.ctx = torch.zeros((rows, d), dtype=torch.float16, device=dev)
        self.u = torch.zeros((rows, 2 * ff), dtype=torch.float32, device=dev)
        self.a = torch.zeros((rows, ff), dtype=torch.float16, device=dev)
        self.logits = torch.zeros((rows, V), dtype=torch.float32, device=dev)
        self.ids = torch.zeros(rows, dtype=torch.int32, device=dev)
        self.p = torch.zeros(1, dtype=torch.int32, device=dev)
        self.bad = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ws = Workspace(ws_bytes)


def _linear(dw: _DeviceWeights, pks: list, name16: list, x16: torch.Tensor, out: torch.Tensor, p_dev, p_host,
            ws: Workspace, accumulate: bool) -> None:
    """out (+)= x16 @ W_p for rows of x16: the decode GEMV for up to 8 rows (decode steps), the
    tcgen05 dequant GEMM for longer row blocks (prefill, prompt-length M)."""
    n = x16.shape[0]
    if p_host == FULL_PRECISION:
        y = (x16 @ dw.fp16["+".join(name16)]).float()
        if accumulate:
            out.add_(y)
        else:
            out.copy_(y)
        return
    col = 0
    for pk in pks:
        width = pk.desc.n
        if n > GEMV_MAX_ROWS:
            gemm(pk, x16, p_dev, out=out[:n, col:col + width], accumulate=accumulate)
        else:
            gemv(pk, x16, p_dev, ws, out=out[:n, col:col + width], accumulate=accumulate)
        col += width


_FUSE_DECODE = os.environ.get("PMPD_FUSE_DECODE", "0") == "1"  # fused norm/SwiGLU GEMVs: measured slower, off


# prefill rows from which causal self-attention over an empty cache goes through torch SDPA
_SDPA_MIN_ROWS = int(os.environ.get("PMPD_SDPA_MIN_ROWS", "256"))
# the same inside a graphed prefill, where the library call's host overhead is paid once at capture
_SDPA_MIN_ROWS_GRAPHED = int(os.environ.get("PMPD_SDPA_MIN_ROWS_GRAPHED", "16"))


def _fused_linear(pks: list, mode: int, xf: torch.Tensor, gain, u_off: int, out: torch.Tensor, buf: _Buffers,
                  accumulate: bool) -> None:
    """out (+)= op(xf) @ W_p with op = RMSNorm*gain or SwiGLU fused into the decode GEMV staging."""
    col = 0
    for pk in pks:
        width = pk.desc.n
        gemv_fused(pk, mode, xf, buf.p, buf.ws, out[:, col:col + width], gain=gain, eps=1e-6, u_off=u_off,
                   accumulate=accumulate)
        col += width


def _run_layers(model: ModelVariants, dw: _DeviceWeights, buf: _Buffers, n: int, cache: KVCache, p_host,
                seq_caches: list | None = None, sdpa_min_rows: int | None = None) -> None:
    """Embedding + all blocks + final norm + head for n tokens in buf.ids; logits -> buf.logits[:n].
    ``seq_caches``: the n rows are the next tokens of n independent sequences (batched decode),
    row j attending over seq_caches[j]; the linear layers run as one n-row GEMV."""
    cfg = model.config
    d, ff, dh = cfg.d_model, cfg.d_ff, cfg.d_head
    s = _stream()
    x, h, qkv, q, ctx, u, a, logits = (buf.x[:n], buf.h[:n], buf.qkv[:n], buf.q[:n], buf.ctx[:n], buf.u[:n],
                                       buf.a[:n], buf.logits[:n])
    if p_host == FULL_PRECISION:
        x.copy_(dw.fp16["embed"][buf.ids[:n].long()].float())
    else:
        _capi.call("pmpd_gather_rows", dw.embed.ref(), buf.ids.data_ptr(), n, buf.p.data_ptr(), x.data_ptr(), s)
    scale = 1.0 / math.sqrt(dh)
    # decode steps: RMSNorm and SwiGLU run inside the GEMV's activation staging (one launch each
    # instead of two) when the fused path accepts the shape
    fuse = p_host != FULL_PRECISION and n <= GEMV_MAX_ROWS and dw.fusable(n) and _FUSE_DECODE
    for i, lay in enumerate(dw.layers):
        pre = f"layers.{i}."
        if fuse:
            _fused_linear(lay["qkv"], _capi.GEMV_IN_RMSNORM, x, lay["norm_attn"], 0, qkv, buf, False)
        else:
            _capi.call("pmpd_rmsnorm", x.data_ptr(), d, lay["norm_attn"].data_ptr(), n, d, 1e-6, h.data_ptr(), d, s)
            _linear(dw, lay["qkv"], [pre + "wq", pre + "wk", pre + "wv"], h, qkv, buf.p, p_host, buf.ws, False)
        if seq_caches is not None:
            g = getattr(seq_caches[0], "group", None)
            if g is not None and dh % 32 == 0 and dh <= 256 and \
                    all(getattr(c, "group", (None,))[0] is g[0] and c.group[3] == j for j, c in enumerate(seq_caches)):
                # caches carved from one allocation (KVCache.batch): every sequence in one launch
                kb, vb, Tb, _ = g
                _capi.call("pmpd_attention_rope_batch", qkv.data_ptr(), qkv.stride(0), n, d, dh, dw.cos.data_ptr(),
                           dw.sin.data_ptr(), Tb.data_ptr(), kb.shape[2], scale, kb[0, i].data_ptr(),
                           vb[0, i].data_ptr(), kb.stride(0), ctx.data_ptr(), s)
            else:
                for j, c in enumerate(seq_caches):
                    _attend_one(dw, qkv[j], ctx[j], q[j], c, i, d, dh, scale, s)
        elif n == 1 and dh % 32 == 0 and dh <= 256:  # decode: RoPE + KV append fused into the attention
            _capi.call("pmpd_attention_rope", qkv.data_ptr(), d, dh, dw.cos.data_ptr(), dw.sin.data_ptr(),
                       cache.T_dev.data_ptr(), cache.capacity, scale, cache.k[i].data_ptr(), cache.v[i].data_ptr(),
                       ctx.data_ptr(), s)
        else:
            _capi.call("pmpd_rope_kv", qkv.data_ptr(), 3 * d, n, d, dh, dw.cos.data_ptr(), dw.sin.data_ptr(),
                       cache.T_dev.data_ptr(), cache.capacity, q.data_ptr(), cache.k[i].data_ptr(),
                       cache.v[i].data_ptr(), s)
            if n >= (_SDPA_MIN_ROWS if sdpa_min_rows is None else sdpa_min_rows) and cache.T == 0:
                # long-prompt prefill from an empty cache (>= 256 rows; below that the per-query kernel
                # wins over the library call overhead): causal attention of the n new rows over
                # themselves (tinylm.py:349-358) through torch's fused SDPA (a library kernel, like
                # cuBLAS; attention is runner glue, not the quantized hot path).  4-D (batch, heads,
                # rows, dh) inputs: with 3-D ones SDPA has no fused kernel and falls back to f32 math
                H = cfg.n_heads
                qh = q[:n].view(n, H, dh).transpose(0, 1).half().unsqueeze(0)
                kh = cache.k[i][:n].view(n, H, dh).transpose(0, 1).unsqueeze(0)
                vh = cache.v[i][:n].view(n, H, dh).transpose(0, 1).unsqueeze(0)
                o = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True, scale=scale)
                ctx.copy_(o[0].transpose(0, 1).reshape(n, d))
            else:
                _capi.call("pmpd_attention", q.data_ptr(), n, d, dh, cache.k[i].data_ptr(), cache.v[i].data_ptr(),
                           cache.T_dev.data_ptr(), cache.capacity, scale, ctx.data_ptr(), s)
        _linear(dw, [lay["wo"]], [pre + "wo"], ctx, x, buf.p, p_host, buf.ws, True)
        if fuse:
            _fused_linear([lay["w_up"]], _capi.GEMV_IN_RMSNORM, x, lay["norm_mlp"], 0, u, buf, False)
            _fused_linear([lay["w_down"]], _capi.GEMV_IN_SWIGLU, u, None, ff, x, buf, True)
        else:
            _capi.call("pmpd_rmsnorm", x.data_ptr(), d, lay["norm_mlp"].data_ptr(), n, d, 1e-6, h.data_ptr(), d, s)
            _linear(dw, [lay["w_up"]], [pre + "w_up"], h, u, buf.p, p_host, buf.ws, False)
            _capi.call("pmpd_silu_mul", u.data_ptr(), 2 * ff, n, ff, a.data_ptr(), ff, s)
            _linear(dw, [lay["w_down"]], [pre + "w_down"], a, x, buf.p, p_host, buf.ws, True)
    if fuse:
        _fused_linear([dw.head], _capi.GEMV_IN_RMSNORM, x, dw.final_norm, 0, logits, buf, False)
    else:
        _capi.call("pmpd_rmsnorm", x.data_ptr(), d, dw.final_norm.data_ptr(), n, d, 1e-6, h.data_ptr(), d, s)
        _linear(dw, [dw.head], ["head"], h, logits, buf.p, p_host, buf.ws, False)


def _attend_one(dw: _DeviceWeights, qkv_row, ctx_row, q_row, cache: KVCache, layer: int, d: int, dh: int,
                scale: float, s: int) -> None:
    """One new token of one sequence: RoPE, KV append at cache.T_dev, attention -> ctx_row."""
    if dh % 32 == 0 and dh <= 256:
        _capi.call("pmpd_attention_rope", qkv_row.data_ptr(), d, dh, dw.cos.data_ptr(), dw.sin.data_ptr(),
                   cache.T_dev.data_ptr(), cache.capacity, scale, cache.k[layer].data_ptr(),
                   cache.v[layer].data_ptr(), ctx_row.data_ptr(), s)
    else:
        _capi.call("pmpd_rope_kv", qkv_row.data_ptr(), 3 * d, 1, d, dh, dw.cos.data_ptr(), dw.sin.data_ptr(),
                   cache.T_dev.data_ptr(), cache.capacity, q_row.data_ptr(), cache.k[layer].data_ptr(),
                   cache.v[layer].data_ptr(), s)
        _capi.call("pmpd_attention", q_row.data_ptr(), 1, d, dh, cache.k[layer].data_ptr(), cache.v[layer].data_ptr(),
                   cache.T_dev.data_ptr(), cache.capacity, scale, ctx_row.data_ptr(), s)


def _check_precision(model: ModelVariants, p: int) -> None:
    if p not in model.allowed_precisions():
        raise ContractViolation(f"precision {p} not in the model's set {sorted(model.allowed_precisions())}")


def _forward(model: ModelVariants, p: int, tokens: Sequence[int], cache: KVCache) -> torch.Tensor:
    """Run ``tokens`` at precision p, extending the cache; device logits [n, V] (tinylm.py:322-368)."""
    cfg = model.config
    n, T0 = len(tokens), cache.T
    if T0 + n > cfg.max_context:
        raise InputError(f"sequence length {T0 + n} exceeds max_context {cfg.max_context}")
    ids = np.asarray(tokens, dtype=np.int64)
    if ids.size and (ids.min() < 0 or ids.max() >= cfg.vocab_size):
        raise InputError(f"token id outside vocabulary of size {cfg.vocab_size}")
    dw = model.device()
    if T0 == 0 and n > 1 and _PREFILL_GRAPH:
        return _prefill_graphed(model, dw, p, ids, cache)
    buf = _Buffers(cfg, n, dw.ws_bytes)
    buf.ids.copy_(torch.from_numpy(ids.astype(np.int32)))
    buf.p.fill_(p if p != FULL_PRECISION else 0)
    _run_layers(model, dw, buf, n, cache, p)
    _capi.call("pmpd_add_i32", cache.T_dev.data_ptr(), n, _stream())
    cache.T = T0 + n
    return buf.logits[:n]


_PREFILL_GRAPH = os.environ.get("PMPD_PREFILL_GRAPH", "1") == "1"
_PREFILL_GRAPHS_KEPT = 4


class _PrefillGraph:
    """A prompt pass of n rows at precision p from an empty cache as ONE CUDA graph (the ~10
    launches per layer of `_run_layers` are ctypes calls at ~5 µs of host time each, so an eager
    short-prompt prefill is host-bound). The graph runs on its own static buffers and an n-row KV
    cache; a replay is followed by copying those rows into the caller's cache."""

    def __init__(self, model: ModelVariants, dw: _DeviceWeights, p: int, n: int):
        cfg = model.config
        self.n, self.p = n, p
        self.buf = _Buffers(cfg, n, dw.ws_bytes)
        self.buf.p.fill_(p if p != FULL_PRECISION else 0)
        self.cache = KVCache(cfg.n_layers, cfg.d_model, n)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up pass: lazy attributes, tensor maps, library handles
            _run_layers(model, dw, self.buf, n, self.cache, p, sdpa_min_rows=_SDPA_MIN_ROWS_GRAPHED)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            _run_layers(model, dw, self.buf, n, self.cache, p, sdpa_min_rows=_SDPA_MIN_ROWS_GRAPHED)
        torch.cuda.synchronize()
        self.graph = g

    def run(self, ids: np.ndarray, cache: KVCache) -> torch.Tensor:
        n = self.n
        self.buf.ids.copy_(torch.from_numpy(ids.astype(np.int32)), non_blocking=False)
        self.graph.replay()
        cache.k[:, :n].copy_(self.cache.k)
        cache.v[:, :n].copy_(self.cache.v)
        # the static buffers are reused by the next replay: hand the caller its own logits
        return self.buf.logits[:n].clone()


def _prefill_graphed(model: ModelVariants, dw: _DeviceWeights, p: int, ids: np.ndarray,
                     cache: KVCache) -> torch.Tensor:
    n = int(ids.size)
    # (the graphs' static buffers are shared by every caller of the model: one prompt pass at a
    # time, enqueued on the caller's current stream)
    lock = model.__dict__.setdefault("_prefill_lock", threading.Lock())
    with lock:
        graphs = model.__dict__.setdefault("_prefill_graphs", {})
        key = (n, p, id(dw))
        pg = graphs.pop(key, None)
        if pg is None:
            while len(graphs) >= _PREFILL_GRAPHS_KEPT:  # keep the most recently used shapes
                graphs.pop(next(iter(graphs)))
            pg = _PrefillGraph(model, dw, p, n)
        graphs[key] = pg
        logits = pg.run(ids, cache)
    _capi.call("pmpd_add_i32", cache.T_dev.data_ptr(), n, _stream())
    cache.T = n
    return logits


def prefill(model: ModelVariants, p: int, prompt: Sequence[int], collect_attn: list | None = None):
    """Causal pass over the prompt; last-position logits (device f32 [V]) plus the cache (tinylm.py:377-388)."""
    if collect_attn is not None:
        raise ConfigError("collect_attn (attention-map capture) is not available on the device path")
    if not prompt:
        raise InputError("prompt is empty")
    if len(prompt) >= model.config.max_context:
        raise InputError(f"prompt length {len(prompt)} must be < max_context {model.config.max_context}")
    _check_precision(model, p)
    cfg = model.config
    cache = KVCache(cfg.n_layers, cfg.d_model, cfg.max_context)
    logits = _forward(model, p, prompt, cache)
    return logits[-1], cache


def decode_step(model: ModelVariants, p: int, token: int, cache: KVCache):
    """One autoregressive step on top of the cache (tinylm.py:391-400)."""
    if cache.T < 1:
        raise InputError("decode_step requires a prefilled cache")
    if cache.T >= model.config.max_context:
        raise InputError(f"context window full at {cache.T} tokens")
    _check_precision(model, p)
    logits = _forward(model, p, [token], cache)
    return logits[-1], cache


def forward_full(model: ModelVariants, p: int, tokens: Sequence[int]) -> torch.Tensor:
    """From-scratch causal pass returning logits at every position (tinylm.py:403-408)."""
    _check_precision(model, p)
    cfg = model.config
    return _forward(model, p, tokens, KVCache(cfg.n_layers, cfg.d_model, cfg.max_context))


# ---------------------------------------------------------------------------
# sampling & generation
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SamplerConfig:
    mode: str = "greedy"  # "greedy" | "temperature"
    temperature: float = 1.0
    seed: int = 0


def sample(logits, cfg: SamplerConfig, rng: np.random.Generator | None = None) -> int:
    """Greedy argmax on device (lowest index on ties) or seeded temperature sampling (tinylm.py:422-436)."""
    if cfg.mode == "greedy":
        t = logits if isinstance(logits, torch.Tensor) else torch.as_tensor(np.asarray(logits, dtype=np.float64))
        t = t.to("cuda", torch.float32).reshape(1, -1).contiguous()
        out = torch.zeros(1, dtype=torch.int32, device="cuda")
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        _capi.call("pmpd_argmax", t.data_ptr(), t.shape[1], 1, t.shape[1], out.data_ptr(), bad.data_ptr(), _stream())
        if int(bad.item()):
            raise InputError("logits contain non-finite values")
        return int(out.item())
    lg = logits.double().cpu().numpy() if isinstance(logits, torch.Tensor) else np.asarray(logits, np.float64)
    if not np.all(np.isfinite(lg)):
        raise InputError("logits contain non-finite values")
    if cfg.mode == "temperature":
        if cfg.temperature <= 0:
            raise ConfigError(f"temperature must be > 0, got {cfg.temperature}")
        z = lg / cfg.temperature
        e = np.exp(z - z.max())
        probs = e / e.sum()
        rng = rng if rng is not None else named_rng(cfg.seed, "sampler")
        return int(rng.choice(len(probs), p=probs))
    raise ConfigError(f"unknown sampler mode {cfg.mode!r}")


def _logits_hash(logits: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(logits, dtype="<f8").tobytes()).hexdigest()[:16]


@dataclass
class GenerationTrace:
    """Everything needed to reproduce and audit one generation (tinylm.py:443-472)."""

    prompt_tokens: list
    output_tokens: list
    precisions: list
    logits_hashes: list
    termination: str  # "eos" | "length"
    p_prefill: int
    schedule: PrecisionSchedule | None = None
    logits: object = None  # device f32 [len, V] when generate(..., record_logits=True)

    def to_json(self) -> dict:
        obj = {"prompt_tokens": self.prompt_tokens, "output_tokens": self.output_tokens,
               "precisions": self.precisions, "logits_hashes": self.logits_hashes,
               "termination": self.termination, "p_prefill": self.p_prefill}
        if self.schedule is not None:
            obj["schedule"] = self.schedule.to_json()
        return obj

    @classmethod
    def from_json(cls, obj: dict) -> "GenerationTrace":
        try:
            sched = obj.get("schedule")
            return cls(list(obj["prompt_tokens"]), list(obj["output_tokens"]), list(obj["precisions"]),
                       list(obj["logits_hashes"]), obj["termination"], obj["p_prefill"],
                       PrecisionSchedule.from_json(sched) if sched else None)
        except (KeyError, TypeError) as exc:
            raise InputError(f"malformed trace JSON: {exc}") from exc


class DecodeEngine:
    """Static device state of greedy generation: KV cache, token/step counters, the device
    schedule table and one CUDA graph per decode step (sched hook -> forward -> argmax -> push)."""

    def __init__(self, model: ModelVariants, capacity: int, p16: bool = False):
        cfg = model.config
        self.model = model
        self.dw = model.device()
        self.buf = _Buffers(cfg, GEMV_MAX_ROWS, self.dw.ws_bytes)
        self.cache = KVCache(cfg.n_layers, cfg.d_model, cfg.max_context)
        self.capacity = capacity
        self.tokens = torch.zeros(capacity, dtype=torch.int32, device="cuda")
        self.n = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.step = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.table = torch.zeros(16, dtype=torch.int32, device="cuda")
        self.hist = torch.zeros((capacity, cfg.vocab_size), dtype=torch.float32, device="cuda")
        self.p16 = p16
        self.graph = None
        self.program = None if p16 or os.environ.get("PMPD_DECODE_ENGINE", "1") == "0" else self._decoder_program()

    def _decoder_program(self):
        """The whole decode step (tinylm.py:334-368 for one token) as one persistent-engine program:
        per layer q|k|v (RMSNorm staged in) -> attention (RoPE + KV append) -> o (added into the
        residual) -> gate|up (RMSNorm) -> down (SwiGLU staged in, added into the residual); then the
        head (final RMSNorm).  None when the shapes are outside the engine (the per-op path runs)."""
        from .engine import IN_ATTN, IN_RMSNORM, AttnSpec, OpSpec, Program
        cfg, dw = self.model.config, self.dw
        d, ff, dh = cfg.d_model, cfg.d_ff, cfg.d_head
        if dh not in (32, 64, 128, 256) or d % 64 or ff % 4 or max(d, ff) > 12288 or \
                any(len(lay["qkv"]) != 1 for lay in dw.layers):
            return None
        x = self.buf.x[0]
        ops = []
        for i, lay in enumerate(dw.layers):
            q = len(ops)
            ops.append(OpSpec(lay["qkv"][0], in_mode=IN_RMSNORM, resid=x, gain=lay["norm_attn"], eps=1e-6))
            ops.append(OpSpec(None, src=q, attn=AttnSpec(cfg.n_heads, dh, self.cache.k[i], self.cache.v[i], dw.cos,
                                                         dw.sin, self.cache.T_dev, self.cache.capacity,
                                                         1.0 / math.sqrt(dh))))
            ops.append(OpSpec(lay["wo"], src=q + 1, in_mode=IN_ATTN, out=x))
            ops.append(OpSpec(lay["w_up"], in_mode=IN_RMSNORM, resid=x, gain=lay["norm_mlp"], eps=1e-6))
            ops.append(OpSpec(lay["w_down"], src=q + 3, act=1, act_off=ff, out=x))
        ops.append(OpSpec(dw.head, in_mode=IN_RMSNORM, resid=x, gain=dw.final_norm, eps=1e-6))
        try:
            return Program(ops)
        except ConfigError:
            return None

    def _step(self) -> None:
        s = _stream()
        if not self.p16:
            _capi.call("pmpd_sched_step", self.table.data_ptr(), 8, self.step.data_ptr(), self.buf.p.data_ptr(), 1, s)
        if self.program is not None and not self.p16:
            # embedding row at the step's precision -> residual stream, then one engine launch
            _capi.call("pmpd_gather_rows", self.dw.embed.ref(), self.buf.ids.data_ptr(), 1, self.buf.p.data_ptr(),
                       self.buf.x.data_ptr(), s)
            self.program.run(self.buf.x, self.buf.p, self.buf.logits)
        else:
            _run_layers(self.model, self.dw, self.buf, 1, self.cache, FULL_PRECISION if self.p16 else None)
        V = self.model.config.vocab_size
        _capi.call("pmpd_argmax", self.buf.logits.data_ptr(), V, 1, V, self.buf.ids.data_ptr(),
                   self.buf.bad.data_ptr(), s)
        _capi.call("pmpd_store_row", self.buf.logits.data_ptr(), self.hist.data_ptr(), self.n.data_ptr(), V,
                   self.capacity, s)
        _capi.call("pmpd_push_token", self.buf.ids.data_ptr(), self.tokens.data_ptr(), self.n.data_ptr(),
                   self.cache.T_dev.data_ptr(), self.capacity, s)

    def check_device(self) -> None:
        """Surface the device error words (one host sync): non-finite logits, a GEMV or engine
        status (precision outside the set -> ContractViolation, activations outside the
        fixed-point range -> InputError), as the reference's checks would raise them."""
        flags = torch.stack([self.buf.bad[0],
                             self.buf.ws.buf[Workspace.STATUS_OFFSET:Workspace.STATUS_OFFSET + 4].view(torch.int32)[0],
                             self.program.status[0] if self.program is not None else self.buf.bad[0] * 0]).cpu()
        if int(flags[0]):
            raise InputError("logits contain non-finite values")
        raise_device_status(int(flags[1]), "decode GEMV", self.buf.ws.clear_status)
        if self.program is not None:
            raise_device_status(int(flags[2]), "decode engine", self.program.status.zero_)

    def capture(self) -> None:
        """Capture one decode step (after a prefill has set the counters)."""
        # snapshot the counters BEFORE the side stream is ordered after the current one: the
        # warm-up step below advances them and must not race with the copies
        saved = [t.clone() for t in (self.n, self.step, self.cache.T_dev, self.buf.ids, self.tokens)]
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._step()  # warm-up launch (lazy attributes, cuBLAS handles)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        for t, v in zip((self.n, self.step, self.cache.T_dev, self.buf.ids, self.tokens), saved):
            t.copy_(v)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step()
        torch.cuda.synchronize()
        self.graph = g


def generate(model: ModelVariants, prompt: Sequence[int], scheduler, sampler_cfg: SamplerConfig | None = None,
             eos_id: int | None = None, max_new: int = 64, record_logits: bool = False,
             check_every: int = 16) -> GenerationTrace:
    """Prefill once, then decode under the scheduler's precision switching (tinylm.py:475-523).

    Greedy decoding runs entirely on the device: the per-token precision is
    ``precision_at(step)`` evaluated by the device hook, the sampled token is
    fed back on device, and the host only checks for EOS every
    ``check_every`` tokens.  Temperature sampling uses the reference's host RNG.
    """
    cfg = sampler_cfg if sampler_cfg is not None else SamplerConfig()
    eos = model.config.vocab_size - 1 if eos_id is None else eos_id
    if max_new < 1:
        raise InputError(f"max_new must be >= 1, got {max_new}")
    if max_new > scheduler.horizon:
        raise InputError(f"max_new {max_new} exceeds the schedule horizon {scheduler.horizon}")
    if cfg.mode != "greedy":
        return _generate_host(model, prompt, scheduler, cfg, eos, max_new)
    if not prompt:
        raise InputError("prompt is empty")
    if len(prompt) >= model.config.max_context:
        raise InputError(f"prompt length {len(prompt)} must be < max_context {model.config.max_context}")
    _check_precision(model, scheduler.p_prefill)
    cap = max_new
    eng = DecodeEngine(model, cap, p16=False)
    # ---- prefill into the engine's cache
    logits = _forward(model, scheduler.p_prefill, prompt, eng.cache)
    # ---- schedule: learned predictor writes the device table, static ones upload theirs
    if hasattr(scheduler, "resolve_device"):
        scheduler.resolve_device(eng.cache, eng.table)
        sched = scheduler.schedule_from_table(eng.table.cpu().tolist())
    else:
        sched = scheduler.resolve(eng.cache)
    violations = sched.validate()
    if violations:
        raise ContractViolation("scheduler produced an invalid schedule: " + "; ".join(violations))
    allowed = model.allowed_precisions()
    for p in sched.precisions:
        if p not in allowed:
            raise ContractViolation(f"schedule uses precision {p} outside the model's set {sorted(allowed)}")
    p16 = FULL_PRECISION in sched.precisions.precisions
    if p16 and len(sched.precisions) > 1:
        raise ConfigError("mixing precision 16 with quantized precisions in one schedule is not supported on device")
    eng.p16 = p16
    if not hasattr(scheduler, "resolve_device"):
        eng.table.copy_(torch.tensor(sched.device_table(), dtype=torch.int32))
    # ---- token 0 from the prefill logits
    s = _stream()
    V = model.config.vocab_size
    last = logits[-1:].contiguous()
    _capi.call("pmpd_argmax", last.data_ptr(), V, 1, V, eng.buf.ids.data_ptr(), eng.buf.bad.data_ptr(), s)
    _capi.call("pmpd_store_row", last.data_ptr(), eng.hist.data_ptr(), eng.n.data_ptr(), V, cap, s)
    _capi.call("pmpd_push_token", eng.buf.ids.data_ptr(), eng.tokens.data_ptr(), eng.n.data_ptr(), 0, cap, s)
    eng.step.zero_()
    produced = 1
    # decode step i runs at T = len(prompt) + i and needs T < max_context (tinylm.py:394-397)
    limit = min(max_new, 1 + model.config.max_context - len(prompt))
    if max_new > 1:
        eng.capture()
    while True:
        eng.check_device()
        toks = eng.tokens[:produced].cpu().tolist()
        if eos in toks or produced >= limit:
            break
        k = min(check_every, limit - produced)
        for _ in range(k):
            eng.graph.replay()
        produced += k
    toks = eng.tokens[:produced].cpu().tolist()
    if eos in toks:
        toks = toks[:toks.index(eos) + 1]
    elif produced < max_new:  # the reference's next decode_step would raise
        raise InputError(f"context window full at {model.config.max_context} tokens")
    eng.cache.T = len(prompt) + len(toks) - 1
    hist = eng.hist[:len(toks)]
    hashes = [_logits_hash(r) for r in hist.double().cpu().numpy()] if record_logits else [""] * len(toks)
    term = "eos" if toks[-1] == eos else "length"
    trace = GenerationTrace(list(prompt), toks, [sched.precision_at(j) for j in range(len(toks))], hashes, term,
                            scheduler.p_prefill, sched, hist if record_logits else None)
    return trace


def _generate_host(model, prompt, scheduler, cfg, eos, max_new) -> GenerationTrace:
    """Temperature sampling: device forward passes, host-side seeded sampling (reference RNG)."""
    rng = named_rng(cfg.seed, "sampler")
    logits, cache = prefill(model, scheduler.p_prefill, prompt)
    sched = scheduler.resolve(cache)
    violations = sched.validate()
    if violations:
        raise ContractViolation("scheduler produced an invalid schedule: " + "; ".join(violations))
    tokens, precisions, hashes = [], [], []

    def push(tok, lg):
        tokens.append(tok)
        precisions.append(sched.precision_at(len(tokens) - 1))
        hashes.append(_logits_hash(lg.double().cpu().numpy()))

    push(sample(logits, cfg, rng), logits)
    while tokens[-1] != eos and len(tokens) < max_new:
        step = len(tokens) - 1
        logits, cache = decode_step(model, sched.precision_at(step), tokens[-1], cache)
        push(sample(logits, cfg, rng), logits)
    term = "eos" if tokens[-1] == eos else "length"
    return GenerationTrace(list(prompt), tokens, precisions, hashes, term, scheduler.p_prefill, sched)


# ---------------------------------------------------------------------------
# batched generation (offline schedule search)
# ---------------------------------------------------------------------------

class _BatchDecoder:
    """Static device state of up to 8 greedy generations that share one static schedule: one
    KV cache per sequence, one CUDA graph per decode step (sched hook -> embedding gather ->
    n-row GEMVs with per-sequence attention -> n-row argmax -> per-sequence token push)."""

    def __init__(self, model: ModelVariants, caches: list, capacity: int, record: bool):
        cfg = model.config
        self.model, self.dw, self.caches, self.capacity = model, model.device(), caches, capacity
        self.M = len(caches)
        self.buf = _Buffers(cfg, GEMV_MAX_ROWS, self.dw.ws_bytes)
        self.tokens = torch.zeros((self.M, capacity), dtype=torch.int32, device="cuda")
        self.n = torch.zeros(self.M, dtype=torch.int32, device="cuda")
        self.step = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.table = torch.zeros(16, dtype=torch.int32, device="cuda")
        self.hist = torch.zeros((self.M, capacity, cfg.vocab_size), dtype=torch.float32, device="cuda") \
            if record else None
        self.graph = None

    def _emit(self, logits_rows, s, advance: bool) -> None:
        """Greedy token of every row of logits_rows [M, V] -> buf.ids; history; token push (and,
        after a decode step, T += 1 for the row the attention appended)."""
        V = self.model.config.vocab_size
        _capi.call("pmpd_argmax", logits_rows.data_ptr(), logits_rows.stride(0), self.M, V, self.buf.ids.data_ptr(),
                   self.buf.bad.data_ptr(), s)
        for j, c in enumerate(self.caches):
            if self.hist is not None:
                _capi.call("pmpd_store_row", logits_rows[j].data_ptr(), self.hist[j].data_ptr(),
                           self.n[j:].data_ptr(), V, self.capacity, s)
            _capi.call("pmpd_push_token", self.buf.ids[j:].data_ptr(), self.tokens[j].data_ptr(), self.n[j:].data_ptr(),
                       c.T_dev.data_ptr() if advance else 0, self.capacity, s)

    def _step(self) -> None:
        s = _stream()
        _capi.call("pmpd_sched_step", self.table.data_ptr(), 8, self.step.data_ptr(), self.buf.p.data_ptr(), 1, s)
        _run_layers(self.model, self.dw, self.buf, self.M, None, None, seq_caches=self.caches)
        self._emit(self.buf.logits[:self.M], s, True)

    def capture(self) -> None:
        state = (self.n, self.step, self.buf.ids, self.tokens) + tuple(c.T_dev for c in self.caches)
        saved = [t.clone() for t in state]  # before the side stream is ordered (see DecodeEngine.capture)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._step()  # warm-up launch
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        for t, v in zip(state, saved):
            t.copy_(v)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step()
        torch.cuda.synchronize()
        self.graph = g


def generate_batch(model: ModelVariants, prompts: Sequence[Sequence[int]], scheduler,
                   sampler_cfg: SamplerConfig | None = None, eos_id: int | None = None, max_new: int = 64,
                   record_logits: bool = False, check_every: int = 16) -> list:
    """``[generate(model, prompt, scheduler, ...) for prompt in prompts]`` for up to 8 prompts at
    once (tinylm.py:475-523 per prompt): the decode steps of all sequences run as one batch of
    n-row GEMVs, each sequence attending over its own cache.  This is the inner loop of the
    reference's offline schedule search (schedule.py:447-457 scores one candidate schedule by
    generating every validation prompt under StaticScheduler(schedule)).

    Greedy sampling and schedules that do not depend on the prompt (StaticScheduler /
    FixedScheduler) only; every trace equals the one ``generate`` returns for that prompt."""
    cfg = sampler_cfg if sampler_cfg is not None else SamplerConfig()
    eos = model.config.vocab_size - 1 if eos_id is None else eos_id
    prompts = [list(p) for p in prompts]
    if not 1 <= len(prompts) <= GEMV_MAX_ROWS:
        raise ConfigError(f"generate_batch takes 1..{GEMV_MAX_ROWS} prompts, got {len(prompts)}")
    if cfg.mode != "greedy":
        raise ConfigError("generate_batch supports greedy sampling only")
    if hasattr(scheduler, "resolve_device"):
        raise ConfigError("generate_batch needs a prompt-independent (static) scheduler")
    if max_new < 1:
        raise InputError(f"max_new must be >= 1, got {max_new}")
    if max_new > scheduler.horizon:
        raise InputError(f"max_new {max_new} exceeds the schedule horizon {scheduler.horizon}")
    mc = model.config.max_context
    for pr in prompts:
        if not pr:
            raise InputError("prompt is empty")
        if len(pr) >= mc:
            raise InputError(f"prompt length {len(pr)} must be < max_context {mc}")
        if len(pr) + max_new - 1 > mc:
            raise InputError(f"prompt length {len(pr)} + {max_new - 1} decode steps exceed max_context {mc}")
    _check_precision(model, scheduler.p_prefill)
    caches = KVCache.batch(len(prompts), model.config.n_layers, model.config.d_model, mc)
    sched = scheduler.resolve(caches[0])
    violations = sched.validate()
    if violations:
        raise ContractViolation("scheduler produced an invalid schedule: " + "; ".join(violations))
    allowed = model.allowed_precisions()
    for p in sched.precisions:
        if p not in allowed or p == FULL_PRECISION:
            raise ContractViolation(f"schedule uses precision {p} outside the batched decoder's set "
                                    f"{sorted(allowed - {FULL_PRECISION})}")
    bd = _BatchDecoder(model, caches, max_new, record_logits)
    bd.table.copy_(torch.tensor(sched.device_table(), dtype=torch.int32))
    V = model.config.vocab_size
    last = torch.zeros((bd.M, V), dtype=torch.float32, device="cuda")
    for j, (pr, c) in enumerate(zip(prompts, caches)):
        last[j].copy_(_forward(model, scheduler.p_prefill, pr, c)[-1])
    bd._emit(last, _stream(), False)  # token 0 of every sequence (caches already hold the prompts)
    produced = 1
    if max_new > 1:
        bd.capture()
    while True:
        if int(bd.buf.bad.item()):
            raise InputError("logits contain non-finite values")
        toks = bd.tokens[:, :produced].cpu().numpy()
        if produced >= max_new or all((row == eos).any() for row in toks):
            break
        k = min(check_every, max_new - produced)
        for _ in range(k):
            bd.graph.replay()
        produced += k
    out = []
    toks_all = bd.tokens[:, :produced].cpu().tolist()
    for j, (pr, c) in enumerate(zip(prompts, caches)):
        toks = toks_all[j]
        if eos in toks:
            toks = toks[:toks.index(eos) + 1]
        c.T = len(pr) + len(toks) - 1
        hist = bd.hist[j, :len(toks)] if record_logits else None
        hashes = [_logits_hash(r) for r in hist.double().cpu().numpy()] if record_logits else [""] * len(toks)
        term = "eos" if toks[-1] == eos else "length"
        out.append(GenerationTrace(pr, toks, [sched.precision_at(i) for i in range(len(toks))], hashes, term,
                                   scheduler.p_prefill, sched, hist))
    return out
