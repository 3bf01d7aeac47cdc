"""Nested multi-precision weight format, B200-resident (drop-in for ``pmpd.quant``).

Same names, arguments and error behaviour as the reference
(``pkg/src/pmpd/quant.py``), but the arrays live in HBM as torch CUDA tensors
and every transformation runs in the CUDA library:

* :func:`quantize_tensor` — bit-exact device quantizer (quant.py:157-191);
* :class:`BitPlaneStore` — reference-layout planes (quant.py:71-109);
* :meth:`QuantizedTensor.packed` — the tiled, fragment-ordered HBM copy the
  decode GEMV streams (one region per bit plane, so precision ``p`` reads
  exactly planes ``0..p-1``);
* :func:`dequantize` — bit-exact f32 dequantization (quant.py:199-215).

The PMPD v1 file reader/writer (quant.py:237-318) is host I/O by nature and
is implemented here with ``struct``; its arrays are uploaded to the device.
"""
from __future__ import annotations

import ctypes
import json
import struct
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from .errors import ConfigError, FormatError, InputError

MAGIC = b"PMPD"
FORMAT_VERSION = 1


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2410_13461_b200 needs a CUDA device (B200); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _to_dev(a, dtype=None) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a))
    t = t.to(device=_device(), dtype=dtype if dtype is not None else t.dtype)
    return t.contiguous()


@dataclass(frozen=True)
class PrecisionSet:
    """Ordered set of supported weight bitwidths, highest first (quant.py:37-68)."""

    precisions: tuple

    def __post_init__(self):
        ps = tuple(int(p) for p in self.precisions)
        object.__setattr__(self, "precisions", ps)
        if not ps:
            raise ConfigError("precision set must be non-empty")
        if any(p < 1 or p > 8 for p in ps):
            raise ConfigError(f"precisions must lie in [1, 8], got {ps}")
        if any(a <= b for a, b in zip(ps, ps[1:])):
            raise ConfigError(f"precisions must be strictly descending, got {ps}")

    @property
    def p_max(self) -> int:
        return self.precisions[0]

    @property
    def p_min(self) -> int:
        return self.precisions[-1]

    def __iter__(self):
        return iter(self.precisions)

    def __len__(self):
        return len(self.precisions)

    def __contains__(self, p) -> bool:
        return p in self.precisions


def _plane_bytes(rows: int, cols: int) -> int:
    return (rows * cols + 7) // 8


def _groups_per_row(cols: int, group_size: int) -> int:
    return (cols + group_size - 1) // group_size


class BitPlaneStore:
    """MSB-first bit planes of one matrix in the reference byte layout, resident on the device."""

    def __init__(self, rows: int, cols: int, p_max: int, planes):
        planes = _to_dev(planes, torch.uint8)
        if tuple(planes.shape) != (p_max, _plane_bytes(rows, cols)):
            raise ConfigError(f"plane array shape {tuple(planes.shape)} does not match "
                              f"{p_max} planes of {_plane_bytes(rows, cols)} bytes")
        self.rows, self.cols, self.p_max = int(rows), int(cols), int(p_max)
        self.planes = planes

    @classmethod
    def from_codes(cls, codes, p_max: int) -> "BitPlaneStore":
        """quant.py:86-94 on the device."""
        c = _to_dev(codes, torch.uint8)
        if c.dim() != 2:
            raise InputError("codes must be a 2-D array")
        rows, cols = c.shape
        planes = torch.empty((p_max, _plane_bytes(rows, cols)), dtype=torch.uint8, device=c.device)
        _capi.call("pmpd_planes_from_codes", _ptr(c), rows, cols, p_max, _ptr(planes), _stream())
        return cls(rows, cols, p_max, planes)

    def prefix_codes(self, p: int) -> torch.Tensor:
        """Codes formed by the top ``p`` planes (quant.py:96-105); reads planes[0:p] only."""
        if not 1 <= p <= self.p_max:
            raise ConfigError(f"precision {p} outside [1, {self.p_max}]")
        d = _capi.describe(self.rows, self.cols, 1, self.p_max, _capi.LAYOUT_REF)
        # a REF descriptor whose planes are this store's buffer (scales unused here)
        buf = torch.empty(d.total_bytes, dtype=torch.uint8, device=self.planes.device)
        for j in range(self.p_max):
            buf[j * d.plane_bytes: j * d.plane_bytes + self.planes.shape[1]].copy_(self.planes[j])
        d.data = _ptr(buf)
        out = torch.empty((self.rows, self.cols), dtype=torch.uint8, device=self.planes.device)
        _capi.call("pmpd_prefix_codes", ctypes.byref(d), p, _ptr(out), _stream())
        return out

    @property
    def payload_bytes(self) -> int:
        return self.planes.numel()


class PackedTensor:
    """One matrix in a device layout (``pmpd_qtensor`` + its HBM buffer)."""

    def __init__(self, desc: _capi.QTensorDesc, buf: torch.Tensor):
        self.desc = desc
        self.buf = buf

    @property
    def layout(self) -> int:
        return self.desc.layout

    def ref(self):
        return ctypes.byref(self.desc)

    def stream_bytes(self, p: int) -> int:
        """HBM bytes one GEMV pass reads at precision p (planes 0..p-1 + scales)."""
        return p * self.desc.plane_bytes + self.desc.scale_bytes


class QuantizedTensor:
    """One matrix quantized at ``p_max`` with per-group f32 min/step scales (quant.py:116-139)."""

    def __init__(self, rows, cols, group_size, p_max, mins, deltas, store: BitPlaneStore):
        self.rows, self.cols = int(rows), int(cols)
        self.group_size, self.p_max = int(group_size), int(p_max)
        self.mins = _to_dev(mins, torch.float32)
        self.deltas = _to_dev(deltas, torch.float32)
        self.store = store
        gpr = _groups_per_row(self.cols, self.group_size)
        if tuple(self.mins.shape) != (self.rows, gpr) or tuple(self.deltas.shape) != (self.rows, gpr):
            raise ConfigError(f"scale arrays must have shape ({self.rows}, {gpr})")
        self._packed = {}
        self._lock = threading.Lock()

    @property
    def n_groups(self) -> int:
        return self.rows * _groups_per_row(self.cols, self.group_size)

    @property
    def codes(self) -> torch.Tensor:
        return self.store.prefix_codes(self.p_max)

    def packed(self, layout: int = _capi.LAYOUT_KN) -> PackedTensor:
        """Device copy in ``layout`` (created once, then cached)."""
        with self._lock:
            pk = self._packed.get(layout)
            if pk is None:
                d = _capi.describe(self.rows, self.cols, self.group_size, self.p_max, layout)
                buf = torch.empty(d.total_bytes, dtype=torch.uint8, device=self.mins.device)
                d.data = _ptr(buf)
                _capi.call("pmpd_pack", ctypes.byref(d), _ptr(self.store.planes), _ptr(self.mins),
                           _ptr(self.deltas), _stream())
                pk = PackedTensor(d, buf)
                self._packed[layout] = pk
            return pk

    def drop_reference_copy(self) -> None:
        """Free the reference-layout planes once a packed copy exists (saves HBM for 7B models)."""
        self.store.planes = torch.empty(0, dtype=torch.uint8, device=self.mins.device)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _capi.DTYPE_F32
    if t.dtype == torch.float64:
        return _capi.DTYPE_F64
    if t.dtype == torch.float16:
        return _capi.DTYPE_F16
    raise InputError(f"unsupported weight dtype {t.dtype}")


def quantize_tensor(weights, p_max: int, group_size: int) -> QuantizedTensor:
    """Asymmetric round-to-nearest quantization into the nested store (quant.py:157-191), on the device.

    Bit-identical to the reference: float64 group min/max, f32 scales, codes
    ``clip(floor((w - min32)/step32 + 0.5), 0, 2^p_max - 1)``.
    """
    if not 1 <= p_max <= 8:
        raise ConfigError(f"p_max must lie in [1, 8], got {p_max}")
    if group_size < 1:
        raise ConfigError(f"group_size must be >= 1, got {group_size}")
    if isinstance(weights, torch.Tensor):
        w = weights
    else:
        w = np.asarray(weights)
        if w.dtype not in (np.float16, np.float32, np.float64):
            w = w.astype(np.float64)
        w = torch.from_numpy(np.ascontiguousarray(w))
    if w.dim() != 2:
        raise InputError(f"expected a 2-D weight matrix, got shape {tuple(w.shape)}")
    if w.dtype not in (torch.float16, torch.float32, torch.float64):
        w = w.to(torch.float64)
    w = w.to(_device()).contiguous()
    rows, cols = w.shape
    gpr = _groups_per_row(cols, group_size)
    dev = w.device
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=dev)
    planes = torch.empty((p_max, _plane_bytes(rows, cols)), dtype=torch.uint8, device=dev)
    mins = torch.empty((rows, gpr), dtype=torch.float32, device=dev)
    deltas = torch.empty((rows, gpr), dtype=torch.float32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    _capi.call("pmpd_quantize", _ptr(w), _dtype_code(w), rows, cols, p_max, group_size, _ptr(codes),
               _ptr(planes), _ptr(mins), _ptr(deltas), _ptr(flag), _stream())
    if int(flag.item()) != 0:
        raise InputError("weights contain non-finite values")
    del codes
    return QuantizedTensor(rows, cols, group_size, p_max, mins, deltas, BitPlaneStore(rows, cols, p_max, planes))


def unpack_prefix(store: BitPlaneStore, p: int) -> torch.Tensor:
    """Codes formed by the top ``p`` bits of every weight (quant.py:194-196)."""
    return store.prefix_codes(p)


def dequantize(qt: QuantizedTensor, p: int, layout: int | None = None) -> torch.Tensor:
    """Reconstruct weights at precision ``p`` (quant.py:199-215) as f32 on the device.

    Equals ``float32(reference float64 result)`` bit for bit.  ``layout``
    selects which resident copy is decoded (default: the reference layout).
    """
    if not 1 <= p <= qt.p_max:
        raise ConfigError(f"precision {p} outside [1, {qt.p_max}]")
    pk = qt.packed(_capi.LAYOUT_REF if layout is None else layout)
    out = torch.empty((qt.rows, qt.cols), dtype=torch.float32, device=qt.mins.device)
    _capi.call("pmpd_dequant", pk.ref(), p, _ptr(out), _stream())
    return out


def max_reconstruction_error_bound(qt: QuantizedTensor, p: int) -> torch.Tensor:
    """Per-group worst-case |w - dequantize(p)| (quant.py:218-230), float64 on the device."""
    d = qt.deltas.double()
    storage = qt.mins.double().abs() * 2.0 ** -23
    if p == qt.p_max:
        return d / 2.0 + storage
    return d * float(1 << (qt.p_max - p)) / 2.0 + d / 2.0 + storage


def _host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def serialize_model(tensors: dict, meta: dict) -> bytes:
    """Weight file writer (quant.py:237-261); byte-identical to the reference."""
    if not tensors:
        raise InputError("no tensors to serialize")
    pms = {t.p_max for t in tensors.values()}
    if len(pms) != 1:
        raise InputError(f"tensors disagree on p_max: {sorted(pms)}")
    gss = {t.group_size for t in tensors.values()}
    if len(gss) != 1:
        raise InputError(f"tensors disagree on group_size: {sorted(gss)}")
    head = dict(meta)
    head["p_max"], head["group_size"] = pms.pop(), gss.pop()
    head["tensors"] = [{"name": n, "rows": t.rows, "cols": t.cols} for n, t in tensors.items()]
    blob = json.dumps(head, sort_keys=True, separators=(",", ":")).encode("utf-8")
    parts = [MAGIC, struct.pack("<II", FORMAT_VERSION, len(blob)), blob]
    for t in tensors.values():
        parts += [_host(t.mins).astype("<f4").tobytes(), _host(t.deltas).astype("<f4").tobytes(),
                  _host(t.store.planes).tobytes()]
    return b"".join(parts)


def parse_model(data: bytes):
    """Weight file reader (quant.py:264-318) with the same validation and messages; uploads to HBM."""
    if len(data) < 4 or data[:4] != MAGIC:
        raise FormatError(f"bad magic {data[:4]!r} at offset 0 (expected {MAGIC!r})")
    if len(data) < 12:
        raise FormatError(f"truncated header: {len(data)} bytes")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported format version {version} at offset 4")
    (meta_len,) = struct.unpack_from("<I", data, 8)
    off = 12
    if off + meta_len > len(data):
        raise FormatError(f"truncated metadata: need {meta_len} bytes at offset {off}")
    try:
        meta = json.loads(data[off:off + meta_len].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise FormatError(f"metadata is not valid JSON at offset {off}: {exc}") from exc
    off += meta_len
    for key in ("p_max", "group_size", "tensors"):
        if key not in meta:
            raise FormatError(f"metadata is missing required key '{key}'")
    p_max, group_size = int(meta["p_max"]), int(meta["group_size"])
    tensors = {}
    for entry in meta["tensors"]:
        try:
            name, rows, cols = entry["name"], int(entry["rows"]), int(entry["cols"])
        except (KeyError, TypeError, ValueError) as exc:
            raise FormatError(f"malformed tensor entry {entry!r} in metadata: {exc}") from exc
        gpr = _groups_per_row(cols, group_size)
        sb = rows * gpr * 4
        pb = _plane_bytes(rows, cols)
        chunks = []
        for nbytes, what in [(sb, "group mins"), (sb, "group steps")] + [(pb, f"plane {k}") for k in range(p_max)]:
            if off + nbytes > len(data):
                raise FormatError(f"truncated reading {what} of tensor '{name}' at offset {off}")
            chunks.append(data[off:off + nbytes])
            off += nbytes
        mins = np.frombuffer(chunks[0], dtype="<f4").reshape(rows, gpr)
        deltas = np.frombuffer(chunks[1], dtype="<f4").reshape(rows, gpr)
        planes = np.frombuffer(b"".join(chunks[2:]), dtype=np.uint8).reshape(p_max, pb)
        tensors[name] = QuantizedTensor(rows, cols, group_size, p_max, mins.copy(), deltas.copy(),
                                        BitPlaneStore(rows, cols, p_max, planes.copy()))
    if off != len(data):
        raise FormatError(f"{len(data) - off} trailing bytes after last tensor at offset {off}")
    return tensors, meta


# ---------------------------------------------------------------------------
# streaming PMPD v1 file I/O: one tensor on the host at a time
# ---------------------------------------------------------------------------

def write_model(path, tensors: dict, meta: dict) -> int:
    """``serialize_model`` (quant.py:237-261) written tensor by tensor to ``path``: the same bytes,
    with at most one tensor's planes and scales on the host.  Returns the file size."""
    if not tensors:
        raise InputError("no tensors to serialize")
    pms = {t.p_max for t in tensors.values()}
    if len(pms) != 1:
        raise InputError(f"tensors disagree on p_max: {sorted(pms)}")
    gss = {t.group_size for t in tensors.values()}
    if len(gss) != 1:
        raise InputError(f"tensors disagree on group_size: {sorted(gss)}")
    head = dict(meta)
    head["p_max"], head["group_size"] = pms.pop(), gss.pop()
    head["tensors"] = [{"name": n, "rows": t.rows, "cols": t.cols} for n, t in tensors.items()]
    blob = json.dumps(head, sort_keys=True, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC + struct.pack("<II", FORMAT_VERSION, len(blob)) + blob)
        for t in tensors.values():
            fh.write(_host(t.mins).astype("<f4").tobytes())
            fh.write(_host(t.deltas).astype("<f4").tobytes())
            if t.store.planes.numel() == 0:
                raise InputError("tensor's reference-layout planes were dropped (drop_reference_copy)")
            fh.write(_host(t.store.planes).tobytes())
        return fh.tell()


def read_model(path, on_tensor=None):
    """``parse_model`` (quant.py:264-318) streamed from ``path`` straight into HBM, same validation
    and messages: each tensor's scales and planes are read into one reusable pinned host buffer
    and copied to the device, so the host holds at most one tensor (``on_tensor(name, qt)`` may
    consume and drop each tensor, e.g. after packing it)."""
    with open(path, "rb") as fh:
        size = fh.seek(0, 2)
        fh.seek(0)
        head = fh.read(12)
        if len(head) < 4 or head[:4] != MAGIC:
            raise FormatError(f"bad magic {head[:4]!r} at offset 0 (expected {MAGIC!r})")
        if len(head) < 12:
            raise FormatError(f"truncated header: {len(head)} bytes")
        (version,) = struct.unpack_from("<I", head, 4)
        if version != FORMAT_VERSION:
            raise FormatError(f"unsupported format version {version} at offset 4")
        (meta_len,) = struct.unpack_from("<I", head, 8)
        off = 12
        if off + meta_len > size:
            raise FormatError(f"truncated metadata: need {meta_len} bytes at offset {off}")
        try:
            meta = json.loads(fh.read(meta_len).decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as exc:
            raise FormatError(f"metadata is not valid JSON at offset {off}: {exc}") from exc
        off += meta_len
        for key in ("p_max", "group_size", "tensors"):
            if key not in meta:
                raise FormatError(f"metadata is missing required key '{key}'")
        p_max, group_size = int(meta["p_max"]), int(meta["group_size"])
        entries = []
        for entry in meta["tensors"]:
            try:
                entries.append((entry["name"], int(entry["rows"]), int(entry["cols"])))
            except (KeyError, TypeError, ValueError) as exc:
                raise FormatError(f"malformed tensor entry {entry!r} in metadata: {exc}") from exc
        biggest = max([2 * r * _groups_per_row(c, group_size) * 4 + p_max * _plane_bytes(r, c)
                       for _, r, c in entries] + [1])
        stage = torch.empty(biggest, dtype=torch.uint8, pin_memory=torch.cuda.is_available())
        view = memoryview(stage.numpy())
        dev = _device()
        tensors = {}
        for name, rows, cols in entries:
            gpr = _groups_per_row(cols, group_size)
            sb, pb = rows * gpr * 4, _plane_bytes(rows, cols)
            parts = [(sb, "group mins"), (sb, "group steps")] + [(pb, f"plane {k}") for k in range(p_max)]
            pos = 0
            for nbytes, what in parts:
                if off + nbytes > size:
                    raise FormatError(f"truncated reading {what} of tensor '{name}' at offset {off}")
                got = fh.readinto(view[pos:pos + nbytes])
                if got != nbytes:
                    raise FormatError(f"truncated reading {what} of tensor '{name}' at offset {off}")
                off += nbytes
                pos += nbytes
            d = stage[:pos].to(dev, non_blocking=True)
            mins = d[:sb].view(torch.float32).reshape(rows, gpr).clone()
            deltas = d[sb:2 * sb].view(torch.float32).reshape(rows, gpr).clone()
            planes = d[2 * sb:].reshape(p_max, pb).clone()
            torch.cuda.current_stream().synchronize()  # the staging buffer is reused next
            qt = QuantizedTensor(rows, cols, group_size, p_max, mins, deltas, BitPlaneStore(rows, cols, p_max, planes))
            if on_tensor is not None:
                qt = on_tensor(name, qt)
            tensors[name] = qt
        if off != size:
            raise FormatError(f"{size - off} trailing bytes after last tensor at offset {off}")
    return tensors, meta
