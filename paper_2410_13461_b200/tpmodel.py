"""Tensor-parallel decoder: the full model of SURVEY.md §8(e) config 5 sharded over ``tp`` ranks.

Every rank holds its Megatron shards of each decoder layer (``tp.plan_layer``):
q|k|v and gate|up column-split (by heads / by channel, gate and up cut at the
same offsets), o and down row-split, the head split by vocabulary.  Per layer
a rank runs the same device kernels as the 1-GPU model (``tinylm._run_layers``)
on its slices: RMSNorm (replicated residual stream), the q|k|v GEMV on its heads,
RoPE + attention over its heads' KV cache, the o GEMV (partial sums), an
all-reduce, the gate|up GEMV, SwiGLU, the down GEMV (partial sums), an
all-reduce.  The head logits stay sharded: greedy decoding takes each rank's
local argmax and combines (value, global index) pairs, lowest index on ties,
which is ``np.argmax`` over the concatenated logits (tinylm.py:422-429).

The learned scheduler (learnsched.py:151-160) needs the feature block's full K/V:
the ranks all-gather their head slices once per prompt (2·T·d f16) and every rank
runs the same device predictor.

The forward is a generator that yields at each collective ("sum": in-place
all-reduce of a tensor, "gather": every rank's copy of a tensor).  ``DistComm``
serves it with torch.distributed (NCCL on the GPU, one process per GPU);
``LocalComm`` drives all ranks of a TP group in one process on one device, in
lockstep, summing/gathering between the ranks' kernel sequences (no kernel ever
waits on another rank) — the 1-GPU validation of the sharded model.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch

from . import _capi
from . import tp as tpplan
from .errors import ConfigError, ContractViolation, InputError
from .linear import Workspace, workspace_bytes
from .tinylm import (FULL_PRECISION, GEMV_MAX_ROWS, GenerationTrace, KVCache, ModelVariants, _concat_cols,
                     _linear, _logits_hash, _stream)


class TPWeights:
    """Rank ``rank``'s shards of a ModelVariants, packed for the GEMV/GEMM (plus replicated glue)."""

    def __init__(self, model: ModelVariants, tp: int, rank: int):
        cfg = model.config
        gs = model.group_size
        if not 0 <= rank < tp:
            raise ConfigError(f"rank {rank} outside tensor-parallel degree {tp}")
        if cfg.d_model % gs:
            raise ConfigError(f"d_model {cfg.d_model} must be a multiple of the group size {gs} for TP")
        if cfg.n_heads % tp:
            raise ConfigError(f"{cfg.n_heads} heads do not split evenly over {tp} ranks")
        self.cfg, self.tp, self.rank = cfg, tp, rank
        self.plan = tpplan.plan_layer(cfg.d_model, cfg.n_heads, cfg.d_ff, tp, rank, gs)
        self.heads = self.plan.heads.size
        self.dq = self.heads * cfg.d_head
        self.ffl = self.plan.ff.size
        self.vocab = [tpplan.plan_head(cfg.vocab_size, tp, r, gs) for r in range(tp)]
        self.vs = self.vocab[rank]
        t = model.tensors
        self.embed = t["embed"].packed(_capi.LAYOUT_REF)
        self.layers = []
        for i in range(cfg.n_layers):
            pre = f"layers.{i}."
            qkv = _concat_cols([t[pre + "wq"], t[pre + "wk"], t[pre + "wv"]])
            self.layers.append({
                "qkv": tpplan.shard_columns(qkv, self.plan.qkv_cols).packed(_capi.LAYOUT_KN),
                "wo": tpplan.shard_rows(t[pre + "wo"], self.plan.o_rows).packed(_capi.LAYOUT_KN),
                "w_up": tpplan.shard_columns(t[pre + "w_up"], self.plan.up_cols).packed(_capi.LAYOUT_KN),
                "w_down": tpplan.shard_rows(t[pre + "w_down"], self.plan.down_rows).packed(_capi.LAYOUT_KN),
                "norm_attn": torch.tensor(model.norms[pre + "norm_attn"], device="cuda"),
                "norm_mlp": torch.tensor(model.norms[pre + "norm_mlp"], device="cuda")})
        self.head = tpplan.shard_columns(t["head"], [self.vs]).packed(_capi.LAYOUT_KN)
        self.final_norm = torch.tensor(model.norms["final_norm"], device="cuda")
        dh = cfg.d_head
        inv = cfg.rope_theta ** (-np.arange(0, dh, 2) / dh)
        ang = np.arange(cfg.max_context, dtype=np.float64)[:, None] * inv[None, :]
        self.cos = torch.tensor(np.cos(ang), dtype=torch.float32, device="cuda")
        self.sin = torch.tensor(np.sin(ang), dtype=torch.float32, device="cuda")
        pks = [self.head] + [lay[k] for lay in self.layers for k in ("qkv", "wo", "w_up", "w_down")]
        self.ws_bytes = max(workspace_bytes(pk, GEMV_MAX_ROWS) for pk in pks)


class _Buffers:
    """One rank's activation scratch for up to ``rows`` tokens (static addresses)."""

    def __init__(self, w: TPWeights, rows: int):
        d, dq, ffl = w.cfg.d_model, w.dq, w.ffl
        vmax = max(s.size for s in w.vocab)
        z = lambda *s, dt=torch.float32: torch.zeros(s, dtype=dt, device="cuda")  # noqa: E731
        self.rows = rows
        self.x, self.y, self.h = z(rows, d), z(rows, d), z(rows, d, dt=torch.float16)
        self.qkv, self.q, self.ctx = z(rows, 3 * dq), z(rows, dq), z(rows, dq, dt=torch.float16)
        self.u, self.a = z(rows, 2 * ffl), z(rows, ffl, dt=torch.float16)
        self.logits = z(rows, vmax)  # padded to the widest vocabulary shard (gather shape)
        self.ids = z(rows, dt=torch.int32)
        self.p = z(1, dt=torch.int32)
        self.loc = z(1, dt=torch.int32)
        self.bad = z(1, dt=torch.int32)
        self.pair = z(3)
        self.ws = Workspace(w.ws_bytes)


def _layers(w: TPWeights, buf: _Buffers, n: int, cache: KVCache, T0: int):
    """Generator: one rank's forward of the n tokens in buf.ids (tinylm.py:327-368 on the rank's
    shards); yields ("sum", t) where the row-parallel partials are all-reduced in place.
    Local head logits -> buf.logits[:n, :vs.size]."""
    cfg = w.cfg
    d, dh, dq, ffl = cfg.d_model, cfg.d_head, w.dq, w.ffl
    s = _stream()
    x, y, h, qkv, q, ctx, u, a = (buf.x[:n], buf.y[:n], buf.h[:n], buf.qkv[:n], buf.q[:n], buf.ctx[:n], buf.u[:n],
                                  buf.a[:n])
    _capi.call("pmpd_gather_rows", w.embed.ref(), buf.ids.data_ptr(), n, buf.p.data_ptr(), x.data_ptr(), s)
    scale = 1.0 / math.sqrt(dh)
    for i, lay in enumerate(w.layers):
        _capi.call("pmpd_rmsnorm", x.data_ptr(), d, lay["norm_attn"].data_ptr(), n, d, 1e-6, h.data_ptr(), d, s)
        _linear(None, [lay["qkv"]], [], h, qkv, buf.p, None, buf.ws, False)
        if n == 1 and dh % 32 == 0 and dh <= 256:
            _capi.call("pmpd_attention_rope", qkv.data_ptr(), dq, dh, w.cos.data_ptr(), w.sin.data_ptr(),
                       cache.T_dev.data_ptr(), cache.capacity, scale, cache.k[i].data_ptr(), cache.v[i].data_ptr(),
                       ctx.data_ptr(), s)
        else:
            _capi.call("pmpd_rope_kv", qkv.data_ptr(), 3 * dq, n, dq, dh, w.cos.data_ptr(), w.sin.data_ptr(),
                       cache.T_dev.data_ptr(), cache.capacity, q.data_ptr(), cache.k[i].data_ptr(),
                       cache.v[i].data_ptr(), s)
            if n >= 256 and T0 == 0:  # long prompt from an empty cache: library SDPA (as tinylm)
                H = w.heads
                qh = q.view(n, H, dh).transpose(0, 1).half().unsqueeze(0)
                kh = cache.k[i][:n].view(n, H, dh).transpose(0, 1).unsqueeze(0)
                vh = cache.v[i][:n].view(n, H, dh).transpose(0, 1).unsqueeze(0)
                o = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True, scale=scale)
                ctx.copy_(o[0].transpose(0, 1).reshape(n, dq))
            else:
                _capi.call("pmpd_attention", q.data_ptr(), n, dq, dh, cache.k[i].data_ptr(), cache.v[i].data_ptr(),
                           cache.T_dev.data_ptr(), cache.capacity, scale, ctx.data_ptr(), s)
        _linear(None, [lay["wo"]], [], ctx, y, buf.p, None, buf.ws, False)  # partial sums of ctx @ wo
        yield "sum", y
        x.add_(y)
        _capi.call("pmpd_rmsnorm", x.data_ptr(), d, lay["norm_mlp"].data_ptr(), n, d, 1e-6, h.data_ptr(), d, s)
        _linear(None, [lay["w_up"]], [], h, u, buf.p, None, buf.ws, False)
        _capi.call("pmpd_silu_mul", u.data_ptr(), 2 * ffl, n, ffl, a.data_ptr(), ffl, s)
        _linear(None, [lay["w_down"]], [], a, y, buf.p, None, buf.ws, False)
        yield "sum", y
        x.add_(y)
    _capi.call("pmpd_rmsnorm", x.data_ptr(), d, w.final_norm.data_ptr(), n, d, 1e-6, h.data_ptr(), d, s)
    _linear(None, [w.head], [], h, buf.logits[:n, :w.vs.size], buf.p, None, buf.ws, False)


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------

class DistComm:
    """The ranks of a torch.distributed group, one per process (NCCL over NVLink on B200s)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    @property
    def ranks(self) -> list:
        return [self.rank]

    def exchange(self, op: str, ts: list) -> list:
        (t,) = ts
        if op == "sum":
            self.dist.all_reduce(t, group=self.group)
            return [None]
        if op == "gather":
            out = [torch.empty_like(t) for _ in range(self.world)]
            self.dist.all_gather(out, t.contiguous(), group=self.group)
            return [out]
        raise ConfigError(f"unknown collective {op!r}")


class LocalComm:
    """All ``world`` ranks of a TP group driven by this process on one device, in lockstep."""

    def __init__(self, world: int):
        self.world = world

    @property
    def ranks(self) -> list:
        return list(range(self.world))

    def exchange(self, op: str, ts: list) -> list:
        if op == "sum":
            tot = ts[0].clone()
            for t in ts[1:]:
                tot += t
            for t in ts:
                t.copy_(tot)
            return [None] * len(ts)
        if op == "gather":
            snap = [t.clone() for t in ts]
            return [snap] * len(ts)
        raise ConfigError(f"unknown collective {op!r}")


def lockstep(gens: list, comm) -> list:
    """Run one generator per local rank to completion, serving each round of yields with one
    collective (every rank must yield the same op in the same order)."""
    sends = [None] * len(gens)
    results = [None] * len(gens)
    while True:
        reqs, done = [], 0
        for i, g in enumerate(gens):
            try:
                reqs.append(g.send(sends[i]))
            except StopIteration as stop:
                results[i] = stop.value
                reqs.append(None)
                done += 1
        if done == len(gens):
            return results
        if done or len({r[0] for r in reqs}) != 1:
            raise ContractViolation("tensor-parallel ranks diverged in their collective sequence")
        sends = comm.exchange(reqs[0][0], [r[1] for r in reqs])


def combine_argmax(pairs: torch.Tensor):
    """Greedy token from per-rank (max value, global index of the lowest local argmax, bad flag)
    rows: the max over ranks, the LOWEST global index among ranks attaining it (ranks own
    ascending index ranges, so this is np.argmax of the concatenated logits, tinylm.py:429).
    Device tensors in, device tensors out (no host sync): (token int32 [1], bad int32 [1])."""
    vals, idx = pairs[:, 0], pairs[:, 1]
    best = vals.max()
    cand = torch.where(vals == best, idx, torch.full_like(idx, float("inf"))).min()
    cand = torch.where(torch.isfinite(cand), cand, torch.zeros_like(cand))
    return cand.reshape(1).to(torch.int32), (pairs[:, 2].max() > 0).reshape(1).to(torch.int32)


# ---------------------------------------------------------------------------
# public API
# ---------------------------------------------------------------------------

class TPModel:
    """A ModelVariants served by a tensor-parallel group: ``prefill`` / ``decode_step`` /
    ``generate`` with the reference's semantics (tinylm.py:377-400,475-523).

    ``comm`` is a DistComm (this process is one rank) or a LocalComm (this process runs every
    rank).  Each local rank owns its shards, its head-sliced KV cache and its buffers."""

    def __init__(self, model: ModelVariants, tp: int, comm):
        cfg = model.config
        if comm.world != tp:
            raise ConfigError(f"communicator has {comm.world} ranks, tensor-parallel degree is {tp}")
        self.model, self.tp, self.comm = model, tp, comm
        self.w = [TPWeights(model, tp, r) for r in comm.ranks]
        self.caches = [KVCache(cfg.n_layers, w.dq, cfg.max_context) for w in self.w]
        self.T = 0

    # -- forward ------------------------------------------------------------
    def _forward(self, p: int, tokens: Sequence[int]) -> torch.Tensor:
        """Extend every rank's cache by ``tokens`` at precision p; full logits [n, V] (gathered)."""
        cfg = self.model.config
        if p == FULL_PRECISION:
            raise ConfigError("precision 16 (fp16 baseline) is not served by the tensor-parallel model")
        if p not in self.model.allowed_precisions():
            raise ContractViolation(f"precision {p} not in the model's set {sorted(self.model.allowed_precisions())}")
        n = len(tokens)
        if self.T + n > cfg.max_context:
            raise InputError(f"sequence length {self.T + n} exceeds max_context {cfg.max_context}")
        ids = np.asarray(tokens, dtype=np.int64)
        if ids.size and (ids.min() < 0 or ids.max() >= cfg.vocab_size):
            raise InputError(f"token id outside vocabulary of size {cfg.vocab_size}")
        bufs = [_Buffers(w, n) for w in self.w]
        for b in bufs:
            b.ids.copy_(torch.from_numpy(ids.astype(np.int32)))
            b.p.fill_(p)
        lockstep([_layers(w, b, n, c, self.T) for w, b, c in zip(self.w, bufs, self.caches)], self.comm)
        full = self._gather_logits(bufs, n)
        for c in self.caches:
            _capi.call("pmpd_add_i32", c.T_dev.data_ptr(), n, _stream())
            c.T = self.T + n
        self.T += n
        return full

    def _gather_logits(self, bufs: list, n: int) -> torch.Tensor:
        def gen(b):
            parts = yield "gather", b.logits[:n]
            return torch.cat([pt[:, :s.size] for pt, s in zip(parts, self.w[0].vocab)], dim=1)
        return lockstep([gen(b) for b in bufs], self.comm)[0]

    def reset(self) -> None:
        for c in self.caches:
            c.reset()
        self.T = 0

    def prefill(self, p: int, prompt: Sequence[int]) -> torch.Tensor:
        """Fresh caches, causal pass over the prompt; last-position logits (device f32 [V])."""
        if not prompt:
            raise InputError("prompt is empty")
        if len(prompt) >= self.model.config.max_context:
            raise InputError(f"prompt length {len(prompt)} must be < max_context {self.model.config.max_context}")
        self.reset()
        return self._forward(p, prompt)[-1]

    def decode_step(self, p: int, token: int) -> torch.Tensor:
        if self.T < 1:
            raise InputError("decode_step requires a prefilled cache")
        if self.T >= self.model.config.max_context:
            raise InputError(f"context window full at {self.T} tokens")
        return self._forward(p, [token])[-1]

    def forward_full(self, p: int, tokens: Sequence[int]) -> torch.Tensor:
        self.reset()
        return self._forward(p, tokens)

    # -- scheduling ------------------------------------------------------------
    def _feature_kv(self, layer: int):
        """The feature block's K and V of all heads (T x d f16), all-gathered from the head slices."""
        def gen(c):
            T = self.T
            ks = yield "gather", c.k[layer][:T]
            vs = yield "gather", c.v[layer][:T]
            return torch.cat(ks, dim=1).contiguous(), torch.cat(vs, dim=1).contiguous()
        return lockstep([gen(c) for c in self.caches], self.comm)

    def _resolve(self, scheduler, tables: list):
        if hasattr(scheduler, "resolve_device"):
            from .learnsched import device_predict
            net = scheduler.net
            for (K, V), c, tab in zip(self._feature_kv(net.feature_block), self.caches, tables):
                device_predict(net, K, V, K.stride(0), c.T_dev, K.shape[0], tab)
            return scheduler.schedule_from_table(tables[0].cpu().tolist())

        sched = scheduler.resolve(_LazyCache(self))
        for tab in tables:
            tab.copy_(torch.tensor(sched.device_table(), dtype=torch.int32))
        return sched

    # -- generation ------------------------------------------------------------
    def generate(self, prompt: Sequence[int], scheduler, eos_id: int | None = None, max_new: int = 64,
                 record_logits: bool = False, check_every: int = 16, graph: bool = True) -> GenerationTrace:
        """Greedy generation under the scheduler's precision switching (tinylm.py:475-523): the
        per-token precision comes from the device hook, the token from the distributed argmax,
        both on device; the host reads tokens back every ``check_every`` steps for EOS."""
        cfg = self.model.config
        eos = cfg.vocab_size - 1 if eos_id is None else eos_id
        if max_new < 1:
            raise InputError(f"max_new must be >= 1, got {max_new}")
        if max_new > scheduler.horizon:
            raise InputError(f"max_new {max_new} exceeds the schedule horizon {scheduler.horizon}")
        logits = self.prefill(scheduler.p_prefill, prompt)
        tables = [torch.zeros(16, dtype=torch.int32, device="cuda") for _ in self.w]
        sched = self._resolve(scheduler, tables)
        violations = sched.validate()
        if violations:
            raise ContractViolation("scheduler produced an invalid schedule: " + "; ".join(violations))
        allowed = self.model.allowed_precisions()
        for p in sched.precisions:
            if p not in allowed or p == FULL_PRECISION:
                raise ContractViolation(f"schedule uses precision {p} outside the TP model's set")
        V = cfg.vocab_size
        s = _stream()
        cap = max_new
        bufs = [_Buffers(w, 1) for w in self.w]
        tokens = [torch.zeros(cap, dtype=torch.int32, device="cuda") for _ in self.w]
        counts = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in self.w]
        steps = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in self.w]
        hist = torch.zeros((cap, V), dtype=torch.float32, device="cuda") if record_logits else None
        last = logits.reshape(1, V).contiguous()
        for b, tk, nn in zip(bufs, tokens, counts):
            _capi.call("pmpd_argmax", last.data_ptr(), V, 1, V, b.ids.data_ptr(), b.bad.data_ptr(), s)
            _capi.call("pmpd_push_token", b.ids.data_ptr(), tk.data_ptr(), nn.data_ptr(), 0, cap, s)
        if hist is not None:
            hist[0].copy_(logits)
        produced = 1
        # decode step i runs at T = len(prompt) + i and needs T < max_context (tinylm.py:394-397)
        limit = min(max_new, 1 + cfg.max_context - len(prompt))

        def step():
            self._decode_token(bufs, tables, steps, tokens, counts, cap, hist)
        if graph and max_new > 1:
            # one CUDA graph per decode step on every local rank (NCCL collectives are captured
            # too); the warm-up step's counter updates are undone before capturing
            state = [steps[i] for i in range(len(steps))] + tokens + counts + [b.ids for b in bufs] + \
                [b.bad for b in bufs] + [c.T_dev for c in self.caches]
            saved = [t.clone() for t in state]
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            for t, v in zip(state, saved):
                t.copy_(v)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            torch.cuda.synchronize()
            step = g.replay
        while True:
            if int(bufs[0].bad.item()):
                raise InputError("logits contain non-finite values")
            for b in bufs:
                b.ws.check("TP decode GEMV")
            toks = tokens[0][:produced].cpu().tolist()
            if eos in toks or produced >= limit:
                break
            for _ in range(min(check_every, limit - produced)):
                step()
                produced += 1
        toks = tokens[0][:produced].cpu().tolist()
        if eos in toks:
            toks = toks[:toks.index(eos) + 1]
        elif produced < max_new:  # the reference's next decode_step would raise
            raise InputError(f"context window full at {cfg.max_context} tokens")
        self.T = len(prompt) + len(toks) - 1
        for c in self.caches:
            c.T = self.T
        hashes = [_logits_hash(r) for r in hist[:len(toks)].double().cpu().numpy()] if record_logits \
            else [""] * len(toks)
        term = "eos" if toks[-1] == eos else "length"
        return GenerationTrace(list(prompt), toks, [sched.precision_at(j) for j in range(len(toks))], hashes, term,
                               scheduler.p_prefill, sched, hist[:len(toks)] if record_logits else None)

    def _decode_token(self, bufs, tables, steps, tokens, counts, cap, hist) -> None:
        """One greedy decode step on every local rank: sched hook -> sharded forward -> local
        argmax -> (value, index) exchange -> token push (all on device)."""
        s = _stream()
        for b, tab, st in zip(bufs, tables, steps):
            _capi.call("pmpd_sched_step", tab.data_ptr(), 8, st.data_ptr(), b.p.data_ptr(), 1, s)
        lockstep([_layers(w, b, 1, c, 1) for w, b, c in zip(self.w, bufs, self.caches)], self.comm)

        def gen(w, b):
            vl = w.vs.size
            _capi.call("pmpd_argmax", b.logits.data_ptr(), vl, 1, vl, b.loc.data_ptr(), b.bad.data_ptr(), s)
            li = b.loc.long()
            b.pair[0:1].copy_(b.logits[0].index_select(0, li))
            b.pair[1:2].copy_(li.float() + w.vs.start)
            b.pair[2:3].copy_(b.bad.float())
            pairs = yield "gather", b.pair
            tok, bad = combine_argmax(torch.stack(pairs))
            b.ids[:1].copy_(tok)
            b.bad.copy_(bad)
            if hist is not None:
                full = yield "gather", b.logits[:1]
                return torch.cat([pt[:, :sl.size] for pt, sl in zip(full, w.vocab)], dim=1)
            return None
        out = lockstep([gen(w, b) for w, b in zip(self.w, bufs)], self.comm)
        if hist is not None:  # row = tokens produced so far (device counter: graph-capturable)
            full = out[0].contiguous()
            _capi.call("pmpd_store_row", full.data_ptr(), hist.data_ptr(), counts[0].data_ptr(), full.shape[1], cap, s)
        for b, tk, nn, c in zip(bufs, tokens, counts, self.caches):
            _capi.call("pmpd_push_token", b.ids.data_ptr(), tk.data_ptr(), nn.data_ptr(), c.T_dev.data_ptr(), cap, s)


class _LazyCache:
    """Reference-style cache view (``layer_kv``) over a TPModel's sharded caches: the feature
    block's K/V are gathered on first use (host-side schedulers, e.g. StaticScheduler ignore it)."""

    def __init__(self, m: TPModel):
        self._m = m
        self.T = m.T

    def layer_kv(self, layer: int):
        K, V = self._m._feature_kv(layer)[0]
        return K.double().cpu().numpy(), V.double().cpu().numpy()
