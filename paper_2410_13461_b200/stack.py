"""The decode-token linear stack of a Llama-shaped model, B200-resident.

This is the unit the headline metric is quoted on (BASELINE.json: "7B decode
linear-layer µs/token & HBM GB/s at 2/3/4-bit, batch 1"): for every layer the
fused q|k|v projection, o, the fused gate|up projection and down, then the
vocabulary head — exactly the linear call sites of one reference decode step
(pkg/src/pmpd/tinylm.py:341-343,359,362,364,368), each a GEMV over the nested
bit-plane weights at the precision chosen on device by the schedule hook.

The chain keeps the real data dependencies (each GEMV consumes the previous
output; q|k|v of layer i+1 reads down of layer i) and scales every output by
1/(std*sqrt(K)) so activations stay O(1) without the attention/norm glue.
One token = one CUDA-graph replay; the precision of token i is
``PrecisionSchedule.precision_at(i)`` evaluated by ``pmpd_sched_step``.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import _capi
from .engine import OpSpec, Program
from .errors import ConfigError
from .linear import Workspace, gemv, workspace_bytes
from .quant import QuantizedTensor, quantize_tensor


@dataclass(frozen=True)
class StackShape:
    n_layers: int
    d_model: int
    d_ff: int
    vocab: int

    @property
    def weights_per_token(self) -> int:
        d, f = self.d_model, self.d_ff
        return self.n_layers * (4 * d * d + 3 * d * f) + d * self.vocab


SCHED_CAPACITY = 8

LLAMA2_7B = StackShape(32, 4096, 11008, 32000)
MOBILELLAMA_1B4 = StackShape(24, 2048, 5632, 32000)


def algorithmic_bytes(shape: StackShape, p: int, m: int = 1, group_size: int = 64) -> int:
    """perf.py:96-101 accounting (p/8 bytes + 8 bytes of f32 min/step per group) plus activations."""
    w = shape.weights_per_token
    if p == 16:
        wb = 2 * w
    else:
        wb = w * p // 8 + 8 * w // group_size
    d, f, L = shape.d_model, shape.d_ff, shape.n_layers
    act = L * 2 * m * ((d + 3 * d) + (d + d) + (d + 2 * f) + (f + d)) + 2 * m * d + 4 * m * shape.vocab
    return wb + act


def _rand_kn(K: int, N: int, std: float, gen: torch.Generator) -> torch.Tensor:
    """Synthetic (K, N) weights of standard deviation ~std on the 4-bit quantization grid of each
    (row, 64-column group): odd codes from a discretised N(8, 3^2), one element at code 0 and one
    at code 15 (the group's min and max), w = (code - 8) * std / 3.25.

    Why not plain N(0, std^2): the reference's nested reconstruction at p < p_max uses the bucket
    centre c*2^m + 2^(m-1) (quant.py:212-215), on average 0.5 step above the codes it replaces.
    That bias is harmless in a model (RMSNorm every layer) but the linear stack chains 129 GEMVs
    with no normalisation: the common-mode shift grows ~10x per op and the chain overflows at
    p <= 3.  Odd codes make the p = 3 reconstruction exact and the p = 2 (and p = 1) errors
    zero-mean, so every precision stays finite; bytes, shapes and work are unchanged."""
    z = torch.randn((K, N), generator=gen, device="cuda", dtype=torch.float32)
    code = (torch.round((z * 3.0 + 7.0) / 2.0) * 2.0 + 1.0).clamp_(1.0, 15.0)
    G = N // 64
    if G:
        blk = code[:, :G * 64].view(K, G, 64)
        i0 = torch.randint(0, 64, (K, G, 1), generator=gen, device="cuda")
        i1 = (i0 + torch.randint(1, 64, (K, G, 1), generator=gen, device="cuda")) % 64
        blk.scatter_(2, i0, 0.0)
        blk.scatter_(2, i1, 15.0)
    return code.sub_(8.0).mul_(std / 3.25)


class LinearStack:
    """Quantized (nested 4/3/2-bit) weights of every decode linear layer, packed for the GEMV."""

    def __init__(self, shape: StackShape, p_max: int = 4, group_size: int = 64, seed: int = 0, std: float = 0.02,
                 m: int = 1, keep_fp16: bool = False):
        self.shape, self.p_max, self.m, self.std = shape, p_max, m, std
        d, f, V = shape.d_model, shape.d_ff, shape.vocab
        gen = torch.Generator(device="cuda")
        gen.manual_seed(seed)
        self.layers = []
        self.fp16 = [] if keep_fp16 else None

        def make(K, N):
            w = _rand_kn(K, N, std, gen)
            qt = quantize_tensor(w, p_max, group_size)
            pk = qt.packed(_capi.LAYOUT_KN)
            qt.drop_reference_copy()
            if keep_fp16:
                alpha = 1.0 / (std * math.sqrt(K))
                self.fp16.append((w.t().contiguous() * alpha).half())  # (N, K) for F.linear
            del w
            return qt, pk

        for _ in range(shape.n_layers):
            self.layers.append([make(d, 3 * d), make(d, d), make(d, 2 * f), make(f, d)])
        self.head = make(d, V)
        torch.cuda.synchronize()
        ws = max(workspace_bytes(pk, m) for lay in self.layers + [[self.head]] for _, pk in lay)
        self.ws = Workspace(ws)
        self.x0 = torch.randn((m, d), device="cuda", generator=gen).half()
        self.qkv = torch.empty((m, 3 * d), device="cuda", dtype=torch.float16)
        self.o = torch.empty((m, d), device="cuda", dtype=torch.float16)
        self.u = torch.empty((m, 2 * f), device="cuda", dtype=torch.float16)
        self.h = torch.empty((m, d), device="cuda", dtype=torch.float16)
        self.logits = torch.empty((m, V), device="cuda", dtype=torch.float32)
        self.p_dev = torch.full((1,), p_max, dtype=torch.int32, device="cuda")
        self.step = torch.zeros(1, dtype=torch.int32, device="cuda")
        # fixed-capacity device switch-point table (rewritten in place: graphs keep its address)
        self.sched = torch.zeros(2 * SCHED_CAPACITY, dtype=torch.int32, device="cuda")
        self.n_prec = SCHED_CAPACITY
        self.set_schedule({p_max: 0})

    # -------------------------------------------------------------- schedule
    def set_schedule(self, switch_points: dict) -> None:
        """Device switch-point table {p: first token index}; the step counter restarts at 0."""
        flat = [0] * (2 * SCHED_CAPACITY)
        for i, (p, st) in enumerate(sorted(switch_points.items(), reverse=True)):
            flat[2 * i], flat[2 * i + 1] = int(p), int(st)
        self.sched.copy_(torch.tensor(flat, dtype=torch.int32))
        self.step.zero_()

    def reset_step(self, value: int = 0) -> None:
        self.step.fill_(value)

    # -------------------------------------------------------------- one token
    def token(self) -> None:
        """Issue one decode token's linear stack on the current stream (graph-capturable)."""
        s = torch.cuda.current_stream().cuda_stream
        _capi.call("pmpd_sched_step", self.sched.data_ptr(), self.n_prec, self.step.data_ptr(),
                   self.p_dev.data_ptr(), 1, s)
        d, f = self.shape.d_model, self.shape.d_ff
        a_d = 1.0 / (self.std * math.sqrt(d))
        a_f = 1.0 / (self.std * math.sqrt(f))
        inp = self.x0
        for (_, wqkv), (_, wo), (_, wup), (_, wdn) in self.layers:
            gemv(wqkv, inp, self.p_dev, self.ws, out=self.qkv, alpha=a_d)
            gemv(wo, self.qkv[:, 2 * d:], self.p_dev, self.ws, out=self.o, alpha=a_d)
            gemv(wup, self.o, self.p_dev, self.ws, out=self.u, alpha=a_d)
            gemv(wdn, self.u[:, :f], self.p_dev, self.ws, out=self.h, alpha=a_f)
            inp = self.h
        gemv(self.head[1], inp, self.p_dev, self.ws, out=self.logits, alpha=a_d)

    def build_engine(self, paired: bool | None = None, groups: int = 4, cta_delta: list | None = None) -> Program:
        """The same chain as ``token`` as one persistent-engine program.

        paired (default: env PMPD_ENGINE_PAIRED, else off): each row-parallel op runs as `groups`
        k-slices, slice s on CTA group s, which also computes the source n-groups of that slice
        (the v columns of q|k|v feed o, the gate columns of gate|up feed down).  A slice then waits
        only on its own group, which has the rest of the column op (q|k columns, up columns) to do
        in between: two grid-wide exchanges per layer (down -> q|k|v, o -> gate|up) instead of four.
        Measured 16 % slower than the plain program (profiles/r02_paired.md): the sub-ops' partial
        stages, extra flushes and per-sub-op tails cost more than the two exchanges they remove."""
        if paired is None:
            paired = os.environ.get("PMPD_ENGINE_PAIRED", "0") == "1"
        if paired:
            return self._build_paired(groups)
        d, f = self.shape.d_model, self.shape.d_ff
        a_d = 1.0 / (self.std * math.sqrt(d))
        a_f = 1.0 / (self.std * math.sqrt(f))
        ops = []
        for i, ((_, wqkv), (_, wo), (_, wup), (_, wdn)) in enumerate(self.layers):
            base = 4 * i
            ops.append(OpSpec(wqkv, src=base - 1, src_col=0, in_alpha=a_f if i else 1.0))
            ops.append(OpSpec(wo, src=base, src_col=2 * d, in_alpha=a_d))
            ops.append(OpSpec(wup, src=base + 1, src_col=0, in_alpha=a_d))
            ops.append(OpSpec(wdn, src=base + 2, src_col=0, in_alpha=a_d))
        ops.append(OpSpec(self.head[1], src=len(ops) - 1, src_col=0, in_alpha=a_f))
        self.program = Program(ops, y_alpha=a_d, cta_delta=cta_delta)
        return self.program

    def _build_paired(self, S: int) -> Program:
        d, f = self.shape.d_model, self.shape.d_ff
        a_d = 1.0 / (self.std * math.sqrt(d))
        a_f = 1.0 / (self.std * math.sqrt(f))
        grid = _capi.lib().pmpd_engine_grid()
        if d % 64 or f % 64 or (d // 64) % S or (f // 64) % S or grid < S:
            raise ConfigError(f"paired engine program: {S} groups do not divide the shape / grid")
        ctas = [(grid * s // S, grid * (s + 1) // S) for s in range(S)]
        D, F = d // 64, f // 64  # n-groups of d and d_ff
        ops = []
        prev, prev_alpha = -1, 1.0
        for i, ((_, wqkv), (_, wo), (_, wup), (_, wdn)) in enumerate(self.layers):
            kq = wqkv.desc.k_tiles
            # q|k|v: the v columns (o's input) first, on every CTA in n-group order, so slice s of
            # them lands on group s; then the q|k columns
            iv = len(ops)
            ops.append(OpSpec(wqkv, src=prev, in_alpha=prev_alpha, part=(2 * D, 3 * D, 0, kq), share=f"qkv{i}"))
            ops.append(OpSpec(wqkv, src=prev, in_alpha=prev_alpha, part=(0, 2 * D, 0, kq), share=f"qkv{i}"))
            for s in range(S):
                ops.append(OpSpec(wo, src=iv, src_col=2 * d, in_alpha=a_d,
                                  part=(0, wo.desc.n_tiles, s * D // S, (s + 1) * D // S), ctas=ctas[s], share=f"o{i}"))
            io = len(ops) - 1
            ku = wup.desc.k_tiles
            ig = len(ops)
            ops.append(OpSpec(wup, src=io, in_alpha=a_d, part=(0, F, 0, ku), share=f"u{i}"))
            ops.append(OpSpec(wup, src=io, in_alpha=a_d, part=(F, wup.desc.n_tiles, 0, ku), share=f"u{i}"))
            for s in range(S):
                ops.append(OpSpec(wdn, src=ig, src_col=0, in_alpha=a_d,
                                  part=(0, wdn.desc.n_tiles, s * F // S, (s + 1) * F // S), ctas=ctas[s],
                                  share=f"dn{i}"))
            prev, prev_alpha = len(ops) - 1, a_f
        ops.append(OpSpec(self.head[1], src=prev, src_col=0, in_alpha=a_f))
        self.program = Program(ops, y_alpha=a_d)
        return self.program

    def token_engine(self) -> None:
        """One decode token's linear stack through the persistent engine (graph-capturable)."""
        s = torch.cuda.current_stream().cuda_stream
        _capi.call("pmpd_sched_step", self.sched.data_ptr(), self.n_prec, self.step.data_ptr(),
                   self.p_dev.data_ptr(), 1, s)
        self.program.run(self.x0, self.p_dev, self.logits)

    def token_fp16(self) -> None:
        """fp16 baseline of the same chain through cuBLAS (precision 16, tinylm.py:204-213)."""
        d, f = self.shape.d_model, self.shape.d_ff
        inp = self.x0
        L = self.shape.n_layers
        for i in range(L):
            wqkv, wo, wup, wdn = self.fp16[4 * i: 4 * i + 4]
            torch.matmul(inp, wqkv.t(), out=self.qkv)
            torch.matmul(self.qkv[:, 2 * d:], wo.t(), out=self.o)
            torch.matmul(self.o, wup.t(), out=self.u)
            torch.matmul(self.u[:, :f], wdn.t(), out=self.h)
            inp = self.h
        self.logits.copy_(F.linear(inp, self.fp16[-1]).float())

    def capture(self, fn) -> torch.cuda.CUDAGraph:
        """CUDA graph of one token (fn = self.token or self.token_fp16)."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()  # warm-up (workspace sizing, cuBLAS handles)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g

    def stream_bytes(self, p: int) -> int:
        """Bytes of packed weights the GEMVs actually fetch at precision p."""
        tot = 0
        for lay in self.layers + [[self.head]]:
            for _, pk in lay:
                tot += pk.stream_bytes(p)
        return tot


class TPLinearStack:
    """The decode linear stack tensor-parallel over ``world`` GPUs (one process per GPU, NCCL).

    Column-parallel q|k|v (by heads), gate|up (same offsets) and head (by vocabulary);
    row-parallel o and down, each followed by an NCCL all-reduce of the batch x d
    partial sums; the vocabulary shards are all-gathered.  All ranks draw the same
    full weights from the same seed, quantize them bit-exactly and keep their
    group-aligned sub-blocks (paper_2410_13461_b200.tp), so TP computes the same
    function as the 1-GPU stack.
    """

    def __init__(self, shape: StackShape, n_heads: int, rank: int, world: int, group, p_max: int = 4,
                 group_size: int = 64, seed: int = 0, std: float = 0.02, m: int = 1):
        from . import tp
        self.shape, self.rank, self.world, self.group, self.m, self.std = shape, rank, world, group, m, std
        d, f, V = shape.d_model, shape.d_ff, shape.vocab
        gen = torch.Generator(device="cuda")
        gen.manual_seed(seed)
        self.plan = tp.plan_layer(d, n_heads, f, world, rank, group_size)
        self.head_cols = tp.plan_head(V, world, rank, group_size)
        self.head_sizes = [tp.plan_head(V, world, r, group_size).size for r in range(world)]

        def make(K, N, cols=None, rows=None):
            w = _rand_kn(K, N, std, gen)
            qt = quantize_tensor(w, p_max, group_size)
            del w
            qt = tp.shard_columns(qt, cols) if cols is not None else tp.shard_rows(qt, rows)
            pk = qt.packed(_capi.LAYOUT_KN)
            qt.drop_reference_copy()
            return pk

        P = self.plan
        self.layers = []
        for _ in range(shape.n_layers):
            self.layers.append([make(d, 3 * d, cols=P.qkv_cols), make(d, d, rows=P.o_rows),
                                make(d, 2 * f, cols=P.up_cols), make(f, d, rows=P.down_rows)])
        self.head = make(d, V, cols=[self.head_cols])
        torch.cuda.synchronize()
        self.ws = Workspace(max(workspace_bytes(pk, m) for lay in self.layers for pk in lay))
        self.ws.ensure(workspace_bytes(self.head, m))
        hq = P.o_rows.size
        self.x16 = torch.randn((m, d), device="cuda", generator=gen).half()
        self.y32 = torch.zeros((m, d), device="cuda", dtype=torch.float32)  # row-parallel partial sums
        self.qkv = torch.empty((m, 3 * hq), device="cuda", dtype=torch.float16)
        self.u = torch.empty((m, 2 * P.ff.size), device="cuda", dtype=torch.float16)
        self.logits_loc = torch.zeros((m, max(self.head_sizes)), device="cuda", dtype=torch.float32)
        self.logits_all = torch.zeros((world, m, max(self.head_sizes)), device="cuda", dtype=torch.float32)
        self.p_dev = torch.full((1,), p_max, dtype=torch.int32, device="cuda")
        self.step = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.sched = torch.zeros(2 * SCHED_CAPACITY, dtype=torch.int32, device="cuda")
        self.set_schedule({p_max: 0})

    set_schedule = LinearStack.set_schedule
    reset_step = LinearStack.reset_step
    capture = LinearStack.capture

    def token(self) -> None:
        import torch.distributed as dist
        s = torch.cuda.current_stream().cuda_stream
        _capi.call("pmpd_sched_step", self.sched.data_ptr(), SCHED_CAPACITY, self.step.data_ptr(),
                   self.p_dev.data_ptr(), 1, s)
        d, f = self.shape.d_model, self.shape.d_ff
        a_d = 1.0 / (self.std * math.sqrt(d))
        a_f = 1.0 / (self.std * math.sqrt(f))
        hq = self.plan.o_rows.size
        ffl = self.plan.ff.size
        for wqkv, wo, wup, wdn in self.layers:
            gemv(wqkv, self.x16, self.p_dev, self.ws, out=self.qkv, alpha=a_d)
            # row-parallel partial sums are all-reduced in f32 (the residual path keeps full
            # precision across ranks), then rounded once to the next GEMV's f16 input
            gemv(wo, self.qkv[:, 2 * hq:], self.p_dev, self.ws, out=self.y32, alpha=a_d)   # row-parallel
            dist.all_reduce(self.y32, group=self.group)
            self.x16.copy_(self.y32)
            gemv(wup, self.x16, self.p_dev, self.ws, out=self.u, alpha=a_d)               # column-parallel
            gemv(wdn, self.u[:, :ffl], self.p_dev, self.ws, out=self.y32, alpha=a_f)      # row-parallel
            dist.all_reduce(self.y32, group=self.group)
            self.x16.copy_(self.y32)
        hs = self.head_cols.size
        gemv(self.head, self.x16, self.p_dev, self.ws, out=self.logits_loc[:, :hs], alpha=a_d)
        dist.all_gather_into_tensor(self.logits_all, self.logits_loc, group=self.group)

    def stream_bytes(self, p: int) -> int:
        return sum(pk.stream_bytes(p) for lay in self.layers for pk in lay) + self.head.stream_bytes(p)


class _ShapeOnly:
    """Another rank's shard in the distributed mode: only its shape (for the contributor counts)."""

    def __init__(self, rows: int, cols: int, group_size: int, p_max: int):
        self.desc = _capi.describe(rows, cols, group_size, p_max, _capi.LAYOUT_KN)

    def ref(self):
        import ctypes
        return ctypes.byref(self.desc)


class TPEngineStack:
    """The decode linear stack tensor-parallel over ``world`` ranks INSIDE the persistent engine.

    The same Megatron plan as ``TPLinearStack`` (column-parallel q|k|v by heads, gate|up at the same
    offsets in both halves, head by vocabulary; row-parallel o and down), but the row-parallel
    all-reduce is not an NCCL call between per-op kernels: every rank's o / down partials are added
    into every rank's copy of a counted fixed-point vector whose contributor counts sum all ranks'
    partitions (``engine.RankProgram``), so a rank's whole token is one engine launch and the
    reduction order never matters (bit-identical across runs).

    * ``group=None``: all ranks on this GPU, one launch (CTA groups; the emulation the B200
      profiling guide prescribes for kernels that wait on other ranks);
    * ``group``/``rank`` (one process per GPU under torch.distributed): this rank's shards only,
      the shared vectors in torch symmetric memory (peer copies over NVLink).
    Weights come from the same generator as ``LinearStack`` (all ranks draw the full matrices and
    keep their sub-blocks), so the 1-GPU stack is the reference for the sharded one.
    """

    def __init__(self, shape: StackShape, n_heads: int, world: int, p_max: int = 4, group_size: int = 64,
                 seed: int = 0, std: float = 0.02, group=None, rank: int | None = None):
        from . import tp
        from .engine import OpSpec, RankProgram
        self.shape, self.world, self.std = shape, world, std
        d, f, V = shape.d_model, shape.d_ff, shape.vocab
        gen = torch.Generator(device="cuda")
        gen.manual_seed(seed)
        plans = [tp.plan_layer(d, n_heads, f, world, r, group_size) for r in range(world)]
        heads = [tp.plan_head(V, world, r, group_size) for r in range(world)]
        self.head_slices = heads
        self.local = list(range(world)) if group is None else [rank]
        a_d = 1.0 / (std * math.sqrt(d))
        a_f = 1.0 / (std * math.sqrt(f))

        def make(K, N):
            w = _rand_kn(K, N, std, gen)
            qt = quantize_tensor(w, p_max, group_size)
            del w
            return qt

        def col(qt, slices, r):
            if r in self.local:
                return tp.shard_columns(qt, slices).packed(_capi.LAYOUT_KN)
            return _ShapeOnly(qt.rows, sum(sl.size for sl in slices), group_size, p_max)

        def row(qt, sl, r):
            if r in self.local:
                return tp.shard_rows(qt, sl).packed(_capi.LAYOUT_KN)
            return _ShapeOnly(sl.size, qt.cols, group_size, p_max)

        self.packs = []  # keeps the shards alive
        rank_ops = [[] for _ in range(world)]
        for i in range(shape.n_layers):
            qkv, o, up, dn = make(d, 3 * d), make(d, d), make(d, 2 * f), make(f, d)
            for r, P in enumerate(plans):
                pk = [col(qkv, P.qkv_cols, r), row(o, P.o_rows, r), col(up, P.up_cols, r), row(dn, P.down_rows, r)]
                self.packs.append(pk)
                base = 4 * i
                hq = P.o_rows.size
                ops = rank_ops[r]
                ops.append(OpSpec(pk[0], src=base - 1, src_col=0, in_alpha=a_f if i else 1.0))
                ops.append(OpSpec(pk[1], src=base, src_col=2 * hq, in_alpha=a_d, out=f"o{i}"))     # row-parallel
                ops.append(OpSpec(pk[2], src=base + 1, src_col=0, in_alpha=a_d))
                ops.append(OpSpec(pk[3], src=base + 2, src_col=0, in_alpha=a_d, out=f"down{i}"))  # row-parallel
            del qkv, o, up, dn
        head = make(d, V)
        for r in range(world):
            pk = col(head, [heads[r]], r)
            self.packs.append([pk])
            rank_ops[r].append(OpSpec(pk, src=len(rank_ops[r]) - 1, src_col=0, in_alpha=a_f))
        del head
        torch.cuda.synchronize()
        self.program = RankProgram(rank_ops, y_alpha=a_d, dist=None if group is None else (group, rank))
        self.x0 = torch.randn((1, d), device="cuda", generator=gen).half()
        self.y = torch.zeros((len(self.local), self.program.y_stride), device="cuda", dtype=torch.float32)
        self.p_dev = torch.full((1,), p_max, dtype=torch.int32, device="cuda")
        self.step = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.sched = torch.zeros(2 * SCHED_CAPACITY, dtype=torch.int32, device="cuda")
        self.n_prec = SCHED_CAPACITY
        self.set_schedule({p_max: 0})

    set_schedule = LinearStack.set_schedule
    reset_step = LinearStack.reset_step
    capture = LinearStack.capture

    def logits(self) -> torch.Tensor:
        """The vocabulary row from the head shards run here (all of them in the one-GPU mode)."""
        return torch.cat([self.y[j, :self.head_slices[r].size] for j, r in enumerate(self.local)])

    def token(self) -> None:
        """One token of the local rank(s) (graph-capturable): the precision hook, one engine launch."""
        _capi.call("pmpd_sched_step", self.sched.data_ptr(), self.n_prec, self.step.data_ptr(),
                   self.p_dev.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
        self.program.run(self.x0, self.p_dev, self.y)

    def stream_bytes(self, p: int) -> int:
        """HBM bytes of the shards run here at precision p."""
        return sum(pk.stream_bytes(p) for lay in self.packs for pk in lay if hasattr(pk, "buf"))
