"""Oracle restatement of the nested bit-plane weight format (reference ``pkg/src/pmpd/quant.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Plain numpy, float64
arithmetic exactly where the reference uses it, so that codes, f32 scales,
bit planes and dequantized values are bit-identical to the reference.
"""
from __future__ import annotations

import json
import struct

import numpy as np

from .errors import ConfigError, FormatError, InputError

MAGIC = b"PMPD"          # quant.py:33
VERSION = 1              # quant.py:34
_BIT_WEIGHTS = (1 << np.arange(8, dtype=np.uint16)).astype(np.uint8)  # LSB-first byte packing


def check_precisions(ps) -> tuple:
    """``PrecisionSet.__post_init__`` (quant.py:43-51): non-empty, each in [1,8], strictly descending."""
    ps = tuple(int(p) for p in ps)
    if len(ps) == 0:
        raise ConfigError("precision set must be non-empty")
    if min(ps) < 1 or max(ps) > 8:
        raise ConfigError(f"precisions must lie in [1, 8], got {ps}")
    for hi, lo in zip(ps[:-1], ps[1:]):
        if not hi > lo:
            raise ConfigError(f"precisions must be strictly descending, got {ps}")
    return ps


def plane_nbytes(rows: int, cols: int) -> int:
    """``_plane_bytes`` (quant.py:112-113)."""
    return -(-(rows * cols) // 8)


def groups_per_row(cols: int, group_size: int) -> int:
    """``_groups_per_row`` (quant.py:142-143)."""
    return -(-cols // group_size)


def spread_groups(per_group: np.ndarray, cols: int, group_size: int) -> np.ndarray:
    """Column-wise broadcast of per-group values (``_spread``, quant.py:150-154)."""
    col_group = np.arange(cols) // group_size
    return per_group[:, col_group]


def pack_planes(codes: np.ndarray, p_max: int) -> np.ndarray:
    """``BitPlaneStore.from_codes`` (quant.py:86-94).

    Plane ``j`` holds bit ``p_max-1-j`` of every code (MSB plane first); the
    flat row-major weight index ``i`` lives in byte ``i >> 3`` bit ``i & 7``
    (LSB-first, zero padded).
    """
    flat = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    n = flat.size
    nb = -(-n // 8)
    out = np.zeros((p_max, nb), dtype=np.uint8)
    for j in range(p_max):
        bits = np.zeros(nb * 8, dtype=np.uint8)
        bits[:n] = (flat >> np.uint8(p_max - 1 - j)) & np.uint8(1)
        out[j] = (bits.reshape(nb, 8) * _BIT_WEIGHTS).sum(axis=1, dtype=np.uint16).astype(np.uint8)
    return out


def prefix_codes(planes: np.ndarray, rows: int, cols: int, p_max: int, p: int) -> np.ndarray:
    """``BitPlaneStore.prefix_codes`` / ``unpack_prefix`` (quant.py:96-105, 194-196).

    Reads planes ``0..p-1`` only; the result equals ``code >> (p_max - p)``.
    """
    if p < 1 or p > p_max:
        raise ConfigError(f"precision {p} outside [1, {p_max}]")
    n = rows * cols
    acc = np.zeros(n, dtype=np.uint8)
    for j in range(p):
        raw = planes[j]
        bits = ((raw[:, None] >> np.arange(8, dtype=np.uint8)[None, :]) & 1).reshape(-1)[:n]
        acc = (acc << np.uint8(1)) | bits.astype(np.uint8)
    return acc.reshape(rows, cols)


class QTensor:
    """Container mirroring ``QuantizedTensor`` (quant.py:116-139)."""

    def __init__(self, rows, cols, group_size, p_max, mins, deltas, planes):
        self.rows, self.cols = int(rows), int(cols)
        self.group_size, self.p_max = int(group_size), int(p_max)
        self.mins = np.ascontiguousarray(mins, dtype=np.float32)
        self.deltas = np.ascontiguousarray(deltas, dtype=np.float32)
        self.planes = np.ascontiguousarray(planes, dtype=np.uint8)
        g = groups_per_row(self.cols, self.group_size)
        if self.mins.shape != (self.rows, g) or self.deltas.shape != (self.rows, g):
            raise ConfigError(f"scale arrays must have shape ({self.rows}, {g})")
        if self.planes.shape != (self.p_max, plane_nbytes(self.rows, self.cols)):
            raise ConfigError("plane array shape mismatch")

    @property
    def codes(self) -> np.ndarray:
        return prefix_codes(self.planes, self.rows, self.cols, self.p_max, self.p_max)


def quantize(weights, p_max: int, group_size: int) -> QTensor:
    """``quantize_tensor`` (quant.py:157-191).

    Per (row, group of ``group_size`` columns): f64 min/max; stored scales are
    ``f32(min)`` and ``f32((max-min)/(2^p_max-1))``; codes are
    ``clip(floor((w - min32)/delta32 + 0.5), 0, 2^p_max-1)`` computed in f64
    against the f32-rounded scales, with step-0 groups coded 0.
    """
    if not 1 <= p_max <= 8:
        raise ConfigError(f"p_max must lie in [1, 8], got {p_max}")
    if group_size < 1:
        raise ConfigError(f"group_size must be >= 1, got {group_size}")
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 2:
        raise InputError(f"expected a 2-D weight matrix, got shape {w.shape}")
    if not np.isfinite(w).all():
        raise InputError("weights contain non-finite values")
    rows, cols = w.shape
    ng = groups_per_row(cols, group_size)
    lo = np.empty((rows, ng))
    hi = np.empty((rows, ng))
    for g in range(ng):
        seg = w[:, g * group_size:(g + 1) * group_size]
        lo[:, g] = seg.min(axis=1)
        hi[:, g] = seg.max(axis=1)
    top = float((1 << p_max) - 1)
    mins32 = lo.astype(np.float32)
    deltas32 = ((hi - lo) / top).astype(np.float32)
    mn = spread_groups(mins32.astype(np.float64), cols, group_size)
    dl = spread_groups(deltas32.astype(np.float64), cols, group_size)
    pos = dl > 0
    t = np.zeros_like(w)
    t[pos] = (w[pos] - mn[pos]) / dl[pos]
    codes = np.clip(np.floor(t + 0.5), 0.0, top).astype(np.uint8)
    return QTensor(rows, cols, group_size, p_max, mins32, deltas32, pack_planes(codes, p_max))


def bucket_index(codes: np.ndarray, p_max: int, p: int) -> np.ndarray:
    """Integer grid index of the reconstruction (quant.py:212-215): the code
    itself at ``p_max``, else the bucket centre ``c*2^m + 2^(m-1)``, ``m=p_max-p``."""
    c = codes.astype(np.int64)
    if p == p_max:
        return c
    m = p_max - p
    return c * (1 << m) + (1 << (m - 1))


def dequantize(qt: QTensor, p: int) -> np.ndarray:
    """``dequantize`` (quant.py:199-215), float64 result."""
    if p < 1 or p > qt.p_max:
        raise ConfigError(f"precision {p} outside [1, {qt.p_max}]")
    codes = prefix_codes(qt.planes, qt.rows, qt.cols, qt.p_max, p).astype(np.float64)
    mn = spread_groups(qt.mins.astype(np.float64), qt.cols, qt.group_size)
    dl = spread_groups(qt.deltas.astype(np.float64), qt.cols, qt.group_size)
    if p == qt.p_max:
        return mn + codes * dl
    m = qt.p_max - p
    return mn + (codes * float(1 << m) + float(1 << (m - 1))) * dl


def error_bound(qt: QTensor, p: int) -> np.ndarray:
    """``max_reconstruction_error_bound`` (quant.py:218-230), per group."""
    d = qt.deltas.astype(np.float64)
    ulp = np.abs(qt.mins.astype(np.float64)) * 2.0 ** -23
    if p == qt.p_max:
        return d / 2.0 + ulp
    return d * float(1 << (qt.p_max - p)) / 2.0 + d / 2.0 + ulp


def serialize(tensors: dict, meta: dict) -> bytes:
    """``serialize_model`` (quant.py:237-261)."""
    if not tensors:
        raise InputError("no tensors to serialize")
    pm = sorted({t.p_max for t in tensors.values()})
    gs = sorted({t.group_size for t in tensors.values()})
    if len(pm) != 1:
        raise InputError(f"tensors disagree on p_max: {pm}")
    if len(gs) != 1:
        raise InputError(f"tensors disagree on group_size: {gs}")
    head = dict(meta)
    head["p_max"], head["group_size"] = pm[0], gs[0]
    head["tensors"] = [{"name": k, "rows": t.rows, "cols": t.cols} for k, t in tensors.items()]
    blob = json.dumps(head, sort_keys=True, separators=(",", ":")).encode("utf-8")
    out = bytearray(MAGIC)
    out += struct.pack("<II", VERSION, len(blob))
    out += blob
    for t in tensors.values():
        out += t.mins.astype("<f4").tobytes() + t.deltas.astype("<f4").tobytes() + t.planes.tobytes()
    return bytes(out)


def parse(data: bytes):
    """``parse_model`` (quant.py:264-318); returns ``(dict[name, QTensor], meta)``."""
    if len(data) < 4 or data[:4] != MAGIC:
        raise FormatError(f"bad magic {data[:4]!r} at offset 0 (expected {MAGIC!r})")
    if len(data) < 12:
        raise FormatError(f"truncated header: {len(data)} bytes")
    version, mlen = struct.unpack_from("<II", data, 4)
    if version != VERSION:
        raise FormatError(f"unsupported format version {version} at offset 4")
    pos = 12
    if pos + mlen > len(data):
        raise FormatError(f"truncated metadata: need {mlen} bytes at offset {pos}")
    try:
        meta = json.loads(data[pos:pos + mlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise FormatError(f"metadata is not valid JSON at offset {pos}: {exc}") from exc
    pos += mlen
    for key in ("p_max", "group_size", "tensors"):
        if key not in meta:
            raise FormatError(f"metadata is missing required key '{key}'")
    p_max, gsz = int(meta["p_max"]), int(meta["group_size"])
    out = {}
    for ent in meta["tensors"]:
        try:
            name, r, c = ent["name"], int(ent["rows"]), int(ent["cols"])
        except (KeyError, TypeError, ValueError) as exc:
            raise FormatError(f"malformed tensor entry {ent!r} in metadata: {exc}") from exc
        sb = r * groups_per_row(c, gsz) * 4
        pb = plane_nbytes(r, c)
        need = 2 * sb + p_max * pb
        if pos + need > len(data):
            raise FormatError(f"truncated reading tensor '{name}' at offset {pos}")
        g = groups_per_row(c, gsz)
        mins = np.frombuffer(data, "<f4", r * g, pos).reshape(r, g)
        dels = np.frombuffer(data, "<f4", r * g, pos + sb).reshape(r, g)
        planes = np.frombuffer(data, np.uint8, p_max * pb, pos + 2 * sb).reshape(p_max, pb)
        pos += need
        out[name] = QTensor(r, c, gsz, p_max, mins, dels, planes)
    if pos != len(data):
        raise FormatError(f"{len(data) - pos} trailing bytes after last tensor at offset {pos}")
    return out, meta
