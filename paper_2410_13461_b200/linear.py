"""Quantized linear layer on the device: the replacement for ``h @ model.weights(name, p)``.

Reference call sites: ``pkg/src/pmpd/tinylm.py:334,341-343,359,362,364,368``
(``x @ W`` with ``W = ModelVariants.weights(name, p)``, tinylm.py:201-231).
Here the weights never leave their packed bit-plane form: the decode GEMV
reads planes ``0..p-1`` straight from HBM, with ``p`` read from device memory.
"""
from __future__ import annotations

import ctypes

import torch

from . import _capi
from .errors import InputError
from .quant import PackedTensor, QuantizedTensor


class Workspace:
    """Zero-initialised scratch for the GEMV's cross-CTA reduction (self-resetting counters).

    One workspace may be shared by every GEMV issued on ONE stream (all
    accesses happen after the kernel's dependency wait).  Do not share a
    workspace between concurrently running streams.
    """

    def __init__(self, nbytes: int = 1 << 20, device=None):
        self.buf = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8,
                               device=device if device is not None else torch.device("cuda"))

    @property
    def nbytes(self) -> int:
        return self.buf.numel()

    def ensure(self, nbytes: int) -> None:
        if nbytes > self.nbytes:
            self.buf = torch.zeros(int(nbytes), dtype=torch.uint8, device=self.buf.device)

    # byte offset of the status word (csrc/gemv.cu: kWsCounters u32 counters, then the status)
    STATUS_OFFSET = 16384 * 4

    def status(self) -> int:
        """Device status word: PMPD_ERR_CONTRACT after a GEMV saw a precision outside [1, p_max]
        (the kernel clamps it, so the error must be surfaced).  Reads device memory (a sync)."""
        if self.nbytes < self.STATUS_OFFSET + 4:
            return 0
        return int(self.buf[self.STATUS_OFFSET:self.STATUS_OFFSET + 4].view(torch.int32).item())

    def check(self, what: str = "decode GEMV") -> None:
        """Raise the error class of a nonzero status word (and clear it), errors.py taxonomy."""
        raise_device_status(self.status(), what, self.clear_status)

    def clear_status(self) -> None:
        if self.nbytes >= self.STATUS_OFFSET + 4:
            self.buf[self.STATUS_OFFSET:self.STATUS_OFFSET + 4].zero_()


def raise_device_status(code: int, what: str, clear=None) -> None:
    """Map a device status word to the reference error taxonomy (errors.py:8-25): CONTRACT ->
    ContractViolation (precision outside the declared set), INPUT -> InputError (non-finite or
    out-of-range activations)."""
    if code == 0:
        return
    if clear is not None:
        clear()
    msgs = {_capi.ERR_CONTRACT: "a kernel read a precision outside the model's set",
            _capi.ERR_INPUT: "non-finite or out-of-range activations"}
    raise _capi._ERRORS.get(code, _capi.PmpdError)(f"{what}: {msgs.get(code, f'device status {code}')}")


def workspace_bytes(pk: PackedTensor, m: int) -> int:
    out = ctypes.c_int64()
    _capi.call("pmpd_gemv_workspace_bytes", pk.ref(), m, ctypes.byref(out))
    return out.value


def gemv(pk: PackedTensor, x: torch.Tensor, p_dev: torch.Tensor, workspace: Workspace,
         out: torch.Tensor | None = None, out_dtype=torch.float32, alpha: float = 1.0,
         accumulate: bool = False) -> torch.Tensor:
    """``y = alpha * x @ W_p^T`` (+ ``y`` if accumulate) for a tiled PackedTensor; x is f16 [m, k]."""
    if x.dtype != torch.float16 or x.dim() != 2 or not x.is_cuda:
        raise InputError("gemv input must be a 2-D float16 CUDA tensor")
    m, k = x.shape
    d = pk.desc
    if k != d.k:
        raise InputError(f"input width {k} does not match the matrix's {d.k}")
    if x.stride(1) != 1:
        raise InputError("gemv input must be row-contiguous")
    if out is None:
        out = torch.empty((m, d.n), dtype=out_dtype, device=x.device)
    if out.stride(1) != 1 or tuple(out.shape) != (m, d.n):
        raise InputError("gemv output must be a row-contiguous [m, n] tensor")
    ydt = _capi.DTYPE_F32 if out.dtype == torch.float32 else _capi.DTYPE_F16
    need = workspace_bytes(pk, m)
    if need > workspace.nbytes:
        workspace.ensure(need)
    _capi.call("pmpd_gemv", pk.ref(), x.data_ptr(), x.stride(0), m, p_dev.data_ptr(), out.data_ptr(), ydt,
               out.stride(0), float(alpha), int(bool(accumulate)), workspace.buf.data_ptr(), workspace.nbytes,
               torch.cuda.current_stream().cuda_stream)
    return out


def gemv_fused(pk: PackedTensor, mode: int, xf: torch.Tensor, p_dev: torch.Tensor, workspace: Workspace,
               out: torch.Tensor, gain: torch.Tensor | None = None, eps: float = 1e-6, u_off: int = 0,
               alpha: float = 1.0, accumulate: bool = False) -> torch.Tensor:
    """``gemv`` with its producer op fused into the activation staging (one launch instead of two).

    mode ``_capi.GEMV_IN_RMSNORM``: the input is ``rmsnorm(xf) * gain`` of the f32 rows xf
    (tinylm.py:293-295); ``_capi.GEMV_IN_SWIGLU``: ``silu(xf[:, k]) * xf[:, k + u_off]``
    (tinylm.py:298,362-364).  Raises ConfigError when the shape is outside the staged path
    (callers then run the two ops separately).
    """
    if xf.dtype != torch.float32 or xf.dim() != 2 or not xf.is_cuda or xf.stride(1) != 1:
        raise InputError("fused gemv input must be a row-contiguous 2-D float32 CUDA tensor")
    m = xf.shape[0]
    d = pk.desc
    if out.stride(1) != 1 or tuple(out.shape) != (m, d.n):
        raise InputError("gemv output must be a row-contiguous [m, n] tensor")
    ydt = _capi.DTYPE_F32 if out.dtype == torch.float32 else _capi.DTYPE_F16
    need = workspace_bytes(pk, m)
    if need > workspace.nbytes:
        workspace.ensure(need)
    _capi.call("pmpd_gemv_fused", pk.ref(), int(mode), xf.data_ptr(), xf.stride(0), m,
               gain.data_ptr() if gain is not None else None, float(eps), int(u_off), p_dev.data_ptr(),
               out.data_ptr(), ydt, out.stride(0), float(alpha), int(bool(accumulate)), workspace.buf.data_ptr(),
               workspace.nbytes, torch.cuda.current_stream().cuda_stream)
    return out


def gemm(pk: PackedTensor, x: torch.Tensor, p_dev: torch.Tensor, out: torch.Tensor | None = None,
         out_dtype=torch.float32, alpha: float = 1.0, accumulate: bool = False,
         status: torch.Tensor | None = None) -> torch.Tensor:
    """Prefill ``y = alpha * x @ W_p^T`` (+ ``y``) on the tcgen05 tensor cores; x is f16 [m, k], any m >= 1.

    The prompt-length counterpart of ``gemv`` (the reference applies the same ``x @ W`` at every
    linear call site of prefill, tinylm.py:377-388 -> 334-368): each CTA dequantizes its weight
    tiles bit-exactly to f16 in shared memory once and streams 128 rows of x against them.
    """
    if x.dtype != torch.float16 or x.dim() != 2 or not x.is_cuda:
        raise InputError("gemm input must be a 2-D float16 CUDA tensor")
    m, k = x.shape
    d = pk.desc
    if k != d.k:
        raise InputError(f"input width {k} does not match the matrix's {d.k}")
    if x.stride(1) != 1:
        raise InputError("gemm input must be row-contiguous")
    if out is None:
        out = torch.empty((m, d.n), dtype=out_dtype, device=x.device)
    if out.stride(1) != 1 or tuple(out.shape) != (m, d.n):
        raise InputError("gemm output must be a row-contiguous [m, n] tensor")
    ydt = _capi.DTYPE_F32 if out.dtype == torch.float32 else _capi.DTYPE_F16
    _capi.call("pmpd_gemm", pk.ref(), x.data_ptr(), x.stride(0), m, p_dev.data_ptr(), out.data_ptr(), ydt,
               out.stride(0), float(alpha), int(bool(accumulate)), status.data_ptr() if status is not None else None,
               torch.cuda.current_stream().cuda_stream)
    return out


class QLinear:
    """A quantized matrix applied as ``x @ W`` (reference orientation, tinylm) at a device-selected precision."""

    def __init__(self, qt: QuantizedTensor, layout: int = _capi.LAYOUT_KN):
        self.qt = qt
        self.packed = qt.packed(layout)
        self.in_features = self.packed.desc.k
        self.out_features = self.packed.desc.n

    def __call__(self, x, p_dev, workspace, **kw):
        return gemv(self.packed, x, p_dev, workspace, **kw)
