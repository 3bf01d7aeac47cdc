"""Persistent decode engine (``pmpd_engine_run``): every quantized linear layer of one batch-1
decode token in one cooperative kernel, with the weight stream never waiting on activations.

A ``Program`` is a chain of GEMV ops over KN-packed tensors; op ``i`` consumes
``in_alpha * y_src[src_col:...]`` (optionally ``silu(g) * u``) of an earlier
op, or the external f16 input for ``src = -1``.  Each op's output is an f32
vector in HBM into which the CTAs sharing an n-group add their split-K partials
(L2 atomics; summation order not fixed); the last op's output, scaled by
``y_alpha``, lands in ``y_out``.  The kernel re-zeroes the vectors on exit.  The reference path this replaces is the
sequence of ``h @ model.weights(name, p)`` calls of one decode step
(pkg/src/pmpd/tinylm.py:341-368).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _capi
from .errors import ConfigError
from .quant import PackedTensor


@dataclass
class OpSpec:
    packed: PackedTensor
    src: int = -1       # index of the producing op, -1 = external input
    src_col: int = 0    # first output column of src used as input element 0
    act: int = 0        # 0 identity, 1 silu(g) * u with u at src_col + act_off
    act_off: int = 0
    in_alpha: float = 1.0


class Program:
    """Device-resident op table + partial buffers + the engine's completion counters."""

    def __init__(self, ops: list, y_alpha: float = 1.0):
        if not ops:
            raise ConfigError("engine program is empty")
        lib = _capi.lib()
        nbytes = lib.pmpd_engine_op_bytes()
        self.ops = ops
        self.parts = []
        host = (ctypes.c_uint8 * (nbytes * len(ops)))()
        for i, spec in enumerate(ops):
            if spec.src >= i:
                raise ConfigError(f"op {i} reads op {spec.src}, which does not precede it")
            slots = 1  # one accumulation vector per op (the kernel adds split-K partials at L2)
            nt = spec.packed.desc.n_tiles
            part = torch.zeros(nt * 64, dtype=torch.float32, device="cuda")
            ns_host = (ctypes.c_uint8 * nt)()
            _capi.call("pmpd_engine_nslots", spec.packed.ref(), ctypes.addressof(ns_host))
            ns = torch.frombuffer(bytearray(ns_host), dtype=torch.uint8).cuda()
            self.parts.append((part, ns))
            _capi.call("pmpd_engine_make_op", spec.packed.ref(), spec.src, spec.src_col, spec.act, spec.act_off,
                       float(spec.in_alpha), part.data_ptr(), slots, ns.data_ptr(),
                       ctypes.addressof(host) + i * nbytes)
        self.table = torch.frombuffer(bytearray(host), dtype=torch.uint8).cuda()
        self.bar = torch.zeros(2, dtype=torch.int32, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.y_alpha = float(y_alpha)
        self.n_out = ops[-1].packed.desc.n

    def run_traced(self, x_in, p_dev, y_out):
        """One pass recording the per-CTA per-op timeline; returns int64 [grid, n_ops, 8]: 4 timestamps (ns), warp-0 tile cycles, tile calls, loop cycles."""
        g = _capi.lib().pmpd_engine_grid()
        tr = torch.zeros((g, len(self.ops), 8), dtype=torch.int64, device="cuda")
        _capi.call("pmpd_engine_run_traced", self.table.data_ptr(), len(self.ops), p_dev.data_ptr(),
                   x_in.data_ptr(), y_out.data_ptr(), self.y_alpha, self.bar.data_ptr(), self.status.data_ptr(),
                   tr.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        return tr.cpu()

    def run(self, x_in: torch.Tensor, p_dev: torch.Tensor, y_out: torch.Tensor) -> None:
        """Enqueue one pass (graph-capturable): y_out = y_alpha * chain(x_in) at precision *p_dev."""
        _capi.call("pmpd_engine_run", self.table.data_ptr(), len(self.ops), p_dev.data_ptr(), x_in.data_ptr(),
                   y_out.data_ptr(), self.y_alpha, self.bar.data_ptr(), self.status.data_ptr(),
                   torch.cuda.current_stream().cuda_stream)
