"""Tensor-parallel sharding of the quantized linear layers (Megatron-style), north-star TP requirement.

Column-parallel: the fused q|k|v projection (split by heads), the fused gate|up
projection (gate and up cut at the SAME offsets so silu(gate)*up stays local)
and the vocabulary head.  Row-parallel: o and down, followed by an all-reduce
of the batch x d partial sums (NCCL over NVLink on the GPU; gloo in the CPU
tests).  Every shard boundary along a grouped axis is a multiple of the group
size, so each shard is an exact sub-block of the reference quantization
(codes, f32 min/step): per-shard dequantization stays bit-exact and the
sharded model computes the same function as the 1-GPU model.

The reference has no parallelism at all; parity for TP is
"TP output == 1-GPU output == oracle" (tests/test_tp_cpu.py, tests/test_gpu_tp.py).
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError


@dataclass(frozen=True)
class Slice:
    start: int
    stop: int

    @property
    def size(self) -> int:
        return self.stop - self.start


def split_aligned(n: int, parts: int, align: int) -> list:
    """Split [0, n) into ``parts`` contiguous slices whose boundaries are multiples of ``align``
    (the last slice absorbs a ragged tail); sizes differ by at most one ``align`` unit."""
    if parts < 1:
        raise ConfigError(f"tensor-parallel degree must be >= 1, got {parts}")
    units = -(-n // align)
    if units < parts:
        raise ConfigError(f"cannot split {n} into {parts} shards aligned to {align}")
    out, u0 = [], 0
    for r in range(parts):
        u1 = u0 + units // parts + (1 if r < units % parts else 0)
        out.append(Slice(min(u0 * align, n), min(u1 * align, n)))
        u0 = u1
    return out


@dataclass(frozen=True)
class LayerShards:
    """Per-rank pieces of one decoder layer (reference orientation: matrices are (d_in, d_out))."""
    heads: Slice          # attention heads owned by the rank
    qkv_cols: list        # column slices of the fused (d, 3d) q|k|v matrix: [q, k, v]
    o_rows: Slice         # rows of wo (d, d): the rank's head channels
    ff: Slice             # gate/up channels owned by the rank
    up_cols: list         # column slices of w_up (d, 2ff): [gate, up]
    down_rows: Slice      # rows of w_down (ff, d)


def plan_layer(d_model: int, n_heads: int, d_ff: int, tp: int, rank: int, group_size: int = 64) -> LayerShards:
    if d_model % n_heads:
        raise ConfigError("d_model must be divisible by n_heads")
    d_head = d_model // n_heads
    hs = split_aligned(n_heads, tp, 1)[rank]
    ch = Slice(hs.start * d_head, hs.stop * d_head)
    if ch.start % group_size or (ch.stop % group_size and ch.stop != d_model):
        raise ConfigError(f"head shard [{ch.start},{ch.stop}) is not aligned to group size {group_size}")
    ff = split_aligned(d_ff, tp, group_size)[rank]
    return LayerShards(heads=hs, qkv_cols=[Slice(ch.start + j * d_model, ch.stop + j * d_model) for j in range(3)],
                       o_rows=ch, ff=ff, up_cols=[ff, Slice(ff.start + d_ff, ff.stop + d_ff)], down_rows=ff)


def plan_head(vocab: int, tp: int, rank: int, group_size: int = 64) -> Slice:
    return split_aligned(vocab, tp, group_size)[rank]


def shard_columns_host(codes, mins, deltas, col_slices: list, group_size: int):
    """Gather column slices of a (rows, cols) quantized matrix (numpy/torch arrays, reference layout):
    codes[:, slices] and the matching per-group scales.  Slices must start on group boundaries."""
    import numpy as np
    lib = np if isinstance(codes, np.ndarray) else None
    cs, ms, ds = [], [], []
    for sl in col_slices:
        if sl.start % group_size:
            raise ConfigError(f"column slice start {sl.start} is not a multiple of the group size {group_size}")
        g0, g1 = sl.start // group_size, -(-sl.stop // group_size)
        cs.append(codes[:, sl.start:sl.stop])
        ms.append(mins[:, g0:g1])
        ds.append(deltas[:, g0:g1])
    if lib is not None:
        return np.concatenate(cs, 1), np.concatenate(ms, 1), np.concatenate(ds, 1)
    import torch
    return torch.cat(cs, 1).contiguous(), torch.cat(ms, 1).contiguous(), torch.cat(ds, 1).contiguous()


def shard_columns(qt, col_slices: list):
    """Device QuantizedTensor restricted to ``col_slices`` (concatenated) — an exact sub-block."""
    from .quant import BitPlaneStore, QuantizedTensor
    codes, mins, dels = shard_columns_host(qt.codes, qt.mins, qt.deltas, col_slices, qt.group_size)
    return QuantizedTensor(qt.rows, codes.shape[1], qt.group_size, qt.p_max, mins, dels,
                           BitPlaneStore.from_codes(codes, qt.p_max))


def shard_rows(qt, sl: Slice):
    """Device QuantizedTensor restricted to rows [start, stop) (groups run along columns: exact)."""
    from .quant import BitPlaneStore, QuantizedTensor
    codes = qt.codes[sl.start:sl.stop].contiguous()
    return QuantizedTensor(sl.size, qt.cols, qt.group_size, qt.p_max, qt.mins[sl.start:sl.stop],
                           qt.deltas[sl.start:sl.stop], BitPlaneStore.from_codes(codes, qt.p_max))
