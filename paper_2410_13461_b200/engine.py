"""Persistent decode engine (``pmpd_engine_run``): every quantized linear layer of one batch-1
decode token in one cooperative kernel, with the weight stream never waiting on activations.

A ``Program`` is a chain of GEMV ops over KN-packed tensors; op ``i`` consumes
``in_alpha * y_src[src_col:...]`` (optionally ``silu(g) * u``) of an earlier
op, or the external f16 input for ``src = -1``.  The CTAs sharing an n-group
add their split-K partials into the op's output vector at L2: in a linear-stack
program as counted 2^-24 fixed-point u64 words (deterministic, self-validating:
no grid-wide ticket between ops), in a decoder program as f32 (order not fixed).
The last op's output, scaled by ``y_alpha``, lands in ``y_out``.  The reference path this replaces is the
sequence of ``h @ model.weights(name, p)`` calls of one decode step
(pkg/src/pmpd/tinylm.py:341-368).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import _capi
from .errors import ConfigError
from .quant import PackedTensor


IN_SRC, IN_RMSNORM, IN_ATTN = 0, 2, 3  # engine.cu E_IN_*
SETS = 3  # buffer sets per counted vector (engine.cu kSets), used round-robin by launch


@dataclass
class AttnSpec:
    """A decode-attention op over one layer's KV cache (tinylm.py:344-358): RoPE of q and the new
    k at position *T_dev, append k and v to the cache, attend over rows 0..T."""
    n_heads: int
    d_head: int
    k_cache: torch.Tensor   # f16 [max_ctx, d]
    v_cache: torch.Tensor
    cos: torch.Tensor       # f32 [max_ctx, d_head / 2]
    sin: torch.Tensor
    T_dev: torch.Tensor     # int32 [1]: rows already cached
    max_ctx: int
    scale: float


@dataclass
class OpSpec:
    packed: PackedTensor | None
    src: int = -1       # index of the producing op, -1 = external input
    src_col: int = 0    # first output column of src used as input element 0
    act: int = 0        # 0 identity, 1 silu(g) * u with u at src_col + act_off
    act_off: int = 0
    in_alpha: float = 1.0
    # decoder-step extensions: input = rmsnorm(resid) * gain (IN_RMSNORM) or the combined
    # attention records of src (IN_ATTN); `out` = a persistent vector (the residual stream)
    # the op's output is added into (x += y), instead of a fresh per-launch vector
    in_mode: int = IN_SRC
    resid: torch.Tensor | None = None
    gain: torch.Tensor | None = None
    eps: float = 1e-6
    out: torch.Tensor | str | None = None  # decoder: residual op; RankProgram: shared (all-reduced) output key
    out_alpha: float = 1.0
    attn: AttnSpec | None = None
    # sub-ops (linear-stack programs): the op restricted to n-groups [ng0, ng1) x k-tiles [kt0, kt1)
    # of its tensor, partitioned over CTAs [c0, c1) only; sub-ops with the same `share` key add
    # into one output vector (the tensor's)
    part: tuple | None = None     # (ng0, ng1, kt0, kt1)
    ctas: tuple | None = None     # (c0, c1)
    share: str | None = None


class Program:
    """Device-resident op table, counted accumulators and the engine's epoch / counters.

    Every linear op gets a cost-balanced CTA partition and a counted fixed-point output (u64
    [2 parity sets][n_tiles * 64]; per n-group contributor counts from the partition).  In a
    decoder program the residual ops (``out`` set: o and down) instead add into ONE counted
    residual stream, into which the launch first adds the f32 embedding row ``x_in``; every
    RMSNorm op carries the static count each residual word has reached at that point."""

    def __init__(self, ops: list, y_alpha: float = 1.0, cta_delta: list | None = None):
        if not ops:
            raise ConfigError("engine program is empty")
        lib = _capi.lib()
        nbytes = lib.pmpd_engine_op_bytes()
        grid = lib.pmpd_engine_grid()
        self.ops = ops
        self.parts = []
        # decoder-step op kinds (attention, RMSNorm / attention-combine inputs, residual outputs)
        # run in the engine's decoder instantiation
        self.decoder = any(sp.attn is not None or sp.in_mode != IN_SRC or sp.out is not None or sp.out_alpha != 1.0
                           for sp in ops)
        self.R = None
        self.d_real = 0
        running = None   # decoder: contributions per residual n-group so far (x0 = 1)
        last_rms = -1
        if self.decoder:
            rms = [sp for sp in ops if sp.in_mode == IN_RMSNORM]
            if not rms:
                raise ConfigError("decoder program without an RMSNorm input op")
            self.d_real = rms[0].packed.desc.k
            d_tiles = rms[0].packed.desc.k_tiles
            self.R = torch.zeros(SETS * d_tiles * 64, dtype=torch.int64, device="cuda")
            running = [1] * d_tiles
        host = (ctypes.c_uint8 * (nbytes * len(ops)))()
        shared = {}  # share key -> [n_tiles, counts, [(addr, contrib, first)]]
        for i, spec in enumerate(ops):
            if spec.src >= i:
                raise ConfigError(f"op {i} reads op {spec.src}, which does not precede it")
            addr = ctypes.addressof(host) + i * nbytes
            if spec.attn is not None:
                at = spec.attn
                rec = torch.zeros(SETS * lib.pmpd_engine_attn_records(at.n_heads, at.d_head), dtype=torch.int64,
                                  device="cuda")
                self.parts.append((rec, at))
                _capi.call("pmpd_engine_make_attn_op", spec.src, at.n_heads, at.d_head, at.k_cache.data_ptr(),
                           at.v_cache.data_ptr(), at.cos.data_ptr(), at.sin.data_ptr(), at.T_dev.data_ptr(),
                           at.max_ctx, float(at.scale), rec.data_ptr(), addr)
                continue
            desc = spec.packed.desc
            sub = spec.part is not None or spec.ctas is not None or spec.share is not None
            if sub and self.decoder:
                raise ConfigError("sub-ops are supported in linear-stack programs")
            ng0, ng1, kt0, kt1 = spec.part if spec.part is not None else (0, desc.n_tiles, 0, desc.k_tiles)
            c0, c1 = spec.ctas if spec.ctas is not None else (0, grid)
            if not (0 <= c0 < c1 <= grid):
                raise ConfigError(f"op {i}: CTA range {spec.ctas} outside the grid of {grid}")
            nt = desc.n_tiles
            ns_host = (ctypes.c_uint8 * nt)()
            _capi.call("pmpd_engine_nslots", spec.packed.ref(), ctypes.addressof(ns_host))
            ns0 = torch.frombuffer(bytearray(ns_host), dtype=torch.uint8).cuda()
            part = torch.zeros(1, dtype=torch.float32, device="cuda")  # unused (op-table ABI)
            self.parts.append((part, ns0, spec.resid, spec.gain))
            _capi.call("pmpd_engine_make_op", spec.packed.ref(), spec.src, spec.src_col, spec.act, spec.act_off,
                       float(spec.in_alpha), part.data_ptr(), 1, ns0.data_ptr(), addr)
            if spec.part is not None:
                _capi.call("pmpd_engine_op_set_slice", addr, ng0, ng1, kt0, kt1)
            if spec.src >= 0 and ops[spec.src].packed is not None:
                width = spec.src_col + (spec.act_off if spec.act == 1 else 0) + desc.k_tiles * 64
                if width > ops[spec.src].packed.desc.n_tiles * 64:
                    raise ConfigError(f"op {i} reads past the end of op {spec.src}'s output")
            even = os.environ.get("PMPD_ENGINE_EVEN", "0") == "1"
            b_host = (ctypes.c_int32 * (grid + 1))()
            snt, skt = ng1 - ng0, kt1 - kt0
            if sub:
                # the slice's tiles over CTAs [c0, c1); the other CTAs get empty ranges
                g = c1 - c0
                sd = _capi.QTensorDesc.from_buffer_copy(desc)
                sd.n_tiles, sd.k_tiles = snt, skt
                sb = (ctypes.c_int32 * (g + 1))()
                _capi.call("pmpd_engine_partition_g", ctypes.byref(sd), g, ctypes.addressof(sb))
                for c in range(grid + 1):
                    b_host[c] = 0 if c <= c0 else (sb[c - c0] if c <= c1 else snt * skt)
            elif even:
                ntl = desc.n_tiles * desc.k_tiles
                for c in range(grid + 1):
                    b_host[c] = c * ntl // grid
            elif cta_delta is not None:
                # calibrated: CTAs measured slower get smaller budgets (calibrate_deltas)
                dl = (ctypes.c_int32 * grid)(*[int(v) for v in cta_delta])
                _capi.call("pmpd_engine_partition_w", spec.packed.ref(), grid, ctypes.addressof(dl),
                           ctypes.addressof(b_host))
            else:
                # cost-balanced CTA tile ranges (stage/segment aware) instead of an even tile split
                # (the 12-warp stage model; measured better for the 10-warp decoder kernel too)
                _capi.call("pmpd_engine_partition", spec.packed.ref(), ctypes.addressof(b_host))
            bounds = torch.frombuffer(bytearray(b_host), dtype=torch.int32).cuda()
            self.parts.append((bounds,))
            _capi.call("pmpd_engine_op_set_bounds", addr, bounds.data_ptr())
            # counted accumulation: contributors per n-group from the partition
            kt, cnt, contrib = skt, [0] * nt, 0
            for c in range(grid):
                t0, t1 = b_host[c], b_host[c + 1]
                if t1 > t0:
                    contrib += 1
                    for ng in range(t0 // kt, (t1 - 1) // kt + 1):
                        cnt[ng0 + ng] += 1
            if spec.share is not None:
                ent = shared.setdefault(spec.share, [nt, [0] * nt, []])
                if ent[0] != nt:
                    raise ConfigError(f"op {i}: shared output '{spec.share}' has another width")
                ent[1] = [a + b for a, b in zip(ent[1], cnt)]
                ent[2].append((addr, contrib))
                _capi.call("pmpd_engine_op_set_share", addr, int(len(ent[2]) == 1))
                continue
            if max(cnt) > 255 or min(cnt) < 1:
                raise ConfigError(f"op {i}: n-group contributor counts outside 1..255")
            cs = torch.tensor(cnt, dtype=torch.uint8, device="cuda")
            residual = self.decoder and spec.out is not None
            if residual:
                if nt != len(running):
                    raise ConfigError(f"op {i}: residual output width differs from the residual stream")
                acc = self.R
            else:
                acc = torch.zeros(SETS * nt * 64, dtype=torch.int64, device="cuda")
            self.parts.append((acc, cs))
            _capi.call("pmpd_engine_op_set_counted", addr, acc.data_ptr(), cs.data_ptr(), contrib)
            if spec.in_mode != IN_SRC or spec.out is not None or spec.out_alpha != 1.0:
                if spec.in_mode == IN_ATTN and (spec.src < 0 or ops[spec.src].attn is None):
                    raise ConfigError(f"op {i}: IN_ATTN needs an attention source op")
                _capi.call("pmpd_engine_op_set_io", addr, spec.in_mode, None,
                           spec.gain.data_ptr() if spec.gain is not None else None, float(spec.eps),
                           int(spec.out is not None), float(spec.out_alpha))
            if self.decoder and (spec.in_mode == IN_RMSNORM or residual):
                cum = None
                if spec.in_mode == IN_RMSNORM:
                    if desc.k_tiles != len(running):
                        raise ConfigError(f"op {i}: RMSNorm input width differs from the residual stream")
                    if max(running) > 1023:
                        raise ConfigError("residual stream: more than 1023 contributions per word")
                    cum = torch.tensor(running, dtype=torch.int32).to(torch.int16).cuda()
                    self.parts.append((cum,))
                _capi.call("pmpd_engine_op_set_residual", addr, cum.data_ptr() if cum is not None else None,
                           last_rms if residual else -1)
                if spec.in_mode == IN_RMSNORM:
                    last_rms = i
                if residual:
                    running = [a + b for a, b in zip(running, cnt)]
        self.cta_delta = cta_delta
        for key, (nt, cnt, members) in shared.items():
            if max(cnt) > 255 or min(cnt) < 1:
                raise ConfigError(f"shared output '{key}': n-group contributor counts outside 1..255")
            acc = torch.zeros(SETS * nt * 64, dtype=torch.int64, device="cuda")
            cs = torch.tensor(cnt, dtype=torch.uint8, device="cuda")
            self.parts.append((acc, cs))
            for addr, contrib in members:
                _capi.call("pmpd_engine_op_set_counted", addr, acc.data_ptr(), cs.data_ptr(), max(contrib, 1))
        _capi.call("pmpd_engine_link", ctypes.addressof(host), len(ops))
        self.table = torch.frombuffer(bytearray(host), dtype=torch.uint8).cuda()
        self.bar = torch.zeros(3 + 2 * len(ops), dtype=torch.int32, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.y_alpha = float(y_alpha)
        self.n_out = ops[-1].packed.desc.n

    def _launch(self, x_in, p_dev, y_out, trace):
        s = torch.cuda.current_stream().cuda_stream
        if self.decoder:
            if x_in.dtype != torch.float32 or x_in.shape[-1] < self.d_real:
                raise ConfigError("decoder program input must be the f32 embedding row")
            _capi.call("pmpd_engine_run_decoder", self.table.data_ptr(), len(self.ops), p_dev.data_ptr(),
                       x_in.data_ptr(), self.R.data_ptr(), self.R.numel() // SETS, self.d_real, y_out.data_ptr(),
                       self.y_alpha, self.bar.data_ptr(), self.status.data_ptr(), trace, s)
        elif trace is not None:
            _capi.call("pmpd_engine_run_traced", self.table.data_ptr(), len(self.ops), p_dev.data_ptr(),
                       x_in.data_ptr(), y_out.data_ptr(), self.y_alpha, self.bar.data_ptr(), self.status.data_ptr(),
                       trace, s)
        else:
            _capi.call("pmpd_engine_run", self.table.data_ptr(), len(self.ops), p_dev.data_ptr(), x_in.data_ptr(),
                       y_out.data_ptr(), self.y_alpha, self.bar.data_ptr(), self.status.data_ptr(), s)

    def run_traced(self, x_in, p_dev, y_out):
        """One pass recording the per-CTA per-op timeline; returns int64 [grid, n_ops, 8]: 4 timestamps (ns), warp-0 tile cycles, tile calls, loop cycles."""
        g = _capi.lib().pmpd_engine_grid()
        tr = torch.zeros((g, len(self.ops), 8), dtype=torch.int64, device="cuda")
        self._launch(x_in, p_dev, y_out, tr.data_ptr())
        torch.cuda.synchronize()
        return tr.cpu()

    def run(self, x_in: torch.Tensor, p_dev: torch.Tensor, y_out: torch.Tensor) -> None:
        """Enqueue one pass (graph-capturable): y_out = y_alpha * chain(x_in) at precision *p_dev
        (decoder programs: x_in = the f32 embedding row that starts the residual stream)."""
        self._launch(x_in, p_dev, y_out, None)


def calibrate_deltas(prog: Program, x_in, p_dev, y_out, runs: int = 3, unit_us: float = 0.25,
                     max_delta: int = 6) -> list:
    """Per-CTA budget reductions for ``Program(..., cta_delta=...)`` from traced launches of
    ``prog``: a CTA whose linear ops end later than the median CTA's (the same CTAs on every op:
    their SMs see inputs later and decode a little slower) gets roughly that lateness less work,
    in half tile-time units of ``unit_us`` (about 0.25 µs on B200 at p=2)."""
    import numpy as np
    lates = []
    for _ in range(runs):
        tr = prog.run_traced(x_in, p_dev, y_out).numpy().astype(np.float64)
        for i, spec in enumerate(prog.ops):
            if spec.attn is not None:
                continue
            staged, done = tr[:, i, 1], tr[:, i, 2]
            busy = done - staged > 0
            if busy.sum() < 0.8 * len(done):
                continue
            d = np.where(busy, done - np.median(done[busy]), np.nan)
            lates.append(d / 1e3)
    late = np.nanmean(np.array(lates), axis=0)
    late = np.nan_to_num(late, nan=0.0)
    return [int(v) for v in np.clip(np.round(late / unit_us), 0, max_delta)]


class RankProgram:
    """Tensor-parallel linear-stack program: ``rank_ops[r]`` is rank r's op chain (its Megatron
    shards, the same op sequence on every rank).  An op whose ``OpSpec.out`` is a string key is
    row-parallel: EVERY rank holds a copy of that output and every rank's op adds each partial into
    every copy, with contributor counts summing all ranks' partitions; each rank's consumers poll
    their own copy.  The cross-rank all-reduce is therefore the engine's own counted addition
    (deterministic, no collective call), the data flow of one GPU per rank over NVLink.

    * ``dist=None`` (one GPU): every rank is built here and all run in ONE launch
      (``pmpd_engine_run_ranks``, the grid split into ``len(rank_ops)`` CTA groups) -- the
      emulation the B200 profiling guide prescribes for kernels that wait on other ranks;
    * ``dist=(group, rank)``: this process runs rank ``rank`` of ``len(rank_ops)`` (only its own op
      table needs real tensors; the others provide shapes for the counts) and the shared copies are
      torch symmetric-memory buffers of the group, added into with system-scope atomics.
    ``y_out`` of ``run`` is [ranks, y_stride] f32: rank r writes its last op's output at row r (one
    row, this rank's, in the distributed mode)."""

    def __init__(self, rank_ops: list, y_alpha: float = 1.0, dist=None):
        W = len(rank_ops)
        if not 1 <= W <= 8 or any(len(ops) != len(rank_ops[0]) for ops in rank_ops) or not rank_ops[0]:
            raise ConfigError("rank programs need 1..8 ranks with the same non-empty op sequence")
        lib = _capi.lib()
        nbytes = lib.pmpd_engine_op_bytes()
        local = [dist[1]] if dist is not None else list(range(W))
        n_emul = len(local)
        G = lib.pmpd_engine_grid() // n_emul
        n_ops = len(rank_ops[0])
        self.n_ranks, self.n_emul, self.n_ops, self.parts = W, n_emul, n_ops, []
        counts, contribs, bounds = {}, {}, {}
        for r, ops in enumerate(rank_ops):
            for i, spec in enumerate(ops):
                if spec.attn is not None or spec.in_mode != IN_SRC or spec.act not in (0, 1):
                    raise ConfigError("rank programs run linear-stack ops only")
                if spec.src >= i:
                    raise ConfigError(f"op {i} reads op {spec.src}, which does not precede it")
                desc = spec.packed.desc
                b_host = (ctypes.c_int32 * (G + 1))()
                _capi.call("pmpd_engine_partition_g", ctypes.byref(desc), G, ctypes.addressof(b_host))
                kt, cnt, contrib = desc.k_tiles, [0] * desc.n_tiles, 0
                for c in range(G):
                    t0, t1 = b_host[c], b_host[c + 1]
                    if t1 > t0:
                        contrib += 1
                        for ng in range(t0 // kt, (t1 - 1) // kt + 1):
                            cnt[ng] += 1
                counts[(r, i)], contribs[(r, i)], bounds[(r, i)] = cnt, contrib, b_host
        # shared (row-parallel) outputs: contributor totals over the ranks, one copy per rank
        totals = {}
        for r, ops in enumerate(rank_ops):
            for i, spec in enumerate(ops):
                if isinstance(spec.out, str):
                    tot = totals.setdefault(spec.out, [0] * spec.packed.desc.n_tiles)
                    if len(tot) != spec.packed.desc.n_tiles:
                        raise ConfigError(f"shared output '{spec.out}' has different widths across ranks")
                    for ng, v in enumerate(counts[(r, i)]):
                        tot[ng] += v
        copies, peers, tot_dev, self.handles = {}, {}, {}, []
        for key, tot in totals.items():
            if max(tot) > 255:
                raise ConfigError(f"shared output '{key}': more than 255 contributors per n-group")
            tot_dev[key] = torch.tensor(tot, dtype=torch.uint8, device="cuda")
            n = SETS * len(tot) * 64
            if dist is None:
                copies[key] = {r: torch.zeros(n, dtype=torch.int64, device="cuda") for r in range(W)}
                peers[key] = [copies[key][r].data_ptr() for r in range(W)]
            else:
                import torch.distributed._symmetric_memory as symm_mem
                buf = symm_mem.empty(n, dtype=torch.int64, device="cuda")
                buf.zero_()
                hdl = symm_mem.rendezvous(buf, dist[0])
                self.handles.append((buf, hdl))
                copies[key] = {dist[1]: buf}
                peers[key] = [int(ptr) for ptr in hdl.buffer_ptrs]
        if dist is not None:
            torch.cuda.synchronize()
            import torch.distributed as tdist
            tdist.barrier(group=dist[0])  # every rank's copies are zero before anyone adds
        host = (ctypes.c_uint8 * (nbytes * n_ops * n_emul))()
        for slot, r in enumerate(local):
            ops = rank_ops[r]
            for i, spec in enumerate(ops):
                addr = ctypes.addressof(host) + (slot * n_ops + i) * nbytes
                desc = spec.packed.desc
                if spec.src >= 0:
                    width = spec.src_col + (spec.act_off if spec.act == 1 else 0) + desc.k_tiles * 64
                    if width > ops[spec.src].packed.desc.n_tiles * 64:
                        raise ConfigError(f"rank {r} op {i} reads past the end of op {spec.src}'s output")
                part = torch.zeros(1, dtype=torch.float32, device="cuda")  # unused (op-table ABI)
                ns0 = torch.tensor(counts[(r, i)], dtype=torch.uint8, device="cuda")
                self.parts.append((part, ns0))
                _capi.call("pmpd_engine_make_op", spec.packed.ref(), spec.src, spec.src_col, spec.act, spec.act_off,
                           float(spec.in_alpha), part.data_ptr(), 1, ns0.data_ptr(), addr)
                bd = torch.frombuffer(bytearray(bounds[(r, i)]), dtype=torch.int32).cuda()
                self.parts.append((bd,))
                _capi.call("pmpd_engine_op_set_bounds", addr, bd.data_ptr())
                key = spec.out if isinstance(spec.out, str) else None
                if key is not None:
                    acc, cs = copies[key][r], tot_dev[key]
                else:
                    acc, cs = torch.zeros(SETS * desc.n_tiles * 64, dtype=torch.int64, device="cuda"), ns0
                self.parts.append((acc, cs))
                _capi.call("pmpd_engine_op_set_counted", addr, acc.data_ptr(), cs.data_ptr(), max(1, contribs[(r, i)]))
                if key is not None:
                    arr = (ctypes.c_void_p * W)(*peers[key])
                    _capi.call("pmpd_engine_op_set_peers", addr, ctypes.cast(arr, ctypes.c_void_p), W,
                               int(dist is not None))
        self.copies = copies
        for r in range(n_emul):
            _capi.call("pmpd_engine_link", ctypes.addressof(host) + r * n_ops * nbytes, n_ops)
        self.table = torch.frombuffer(bytearray(host), dtype=torch.uint8).cuda()
        self.bar = torch.zeros(3 + 2 * n_ops, dtype=torch.int32, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.y_alpha = float(y_alpha)
        self.y_stride = max(ops[-1].packed.desc.n_tiles * 64 for ops in rank_ops)

    def run(self, x_in: torch.Tensor, p_dev: torch.Tensor, y_out: torch.Tensor) -> None:
        """Enqueue one token of every local rank (graph-capturable); y_out: f32 [ranks run here,
        >= y_stride]."""
        if y_out.dtype != torch.float32 or y_out.dim() != 2 or y_out.shape[0] < self.n_emul or \
                y_out.stride(0) < self.y_stride or y_out.stride(1) != 1:
            raise ConfigError(f"y_out must be f32 [{self.n_emul}, >= {self.y_stride}] with unit column stride")
        _capi.call("pmpd_engine_run_ranks", self.table.data_ptr(), self.n_ops, self.n_emul, p_dev.data_ptr(),
                   x_in.data_ptr(), y_out.data_ptr(), y_out.stride(0), self.y_alpha, self.bar.data_ptr(),
                   self.status.data_ptr(), torch.cuda.current_stream().cuda_stream)
