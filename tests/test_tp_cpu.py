"""Tensor-parallel sharding logic on CPU with world_size-2 gloo process groups.

Each rank takes its Megatron shards of a quantized decoder layer chain
(paper_2410_13461_b200.tp), computes its partial products with the float64
oracle (the stand-in for the rank's GPU GEMVs), and all-reduces the row-split
outputs through torch.distributed (gloo).  The result must equal the unsharded
oracle chain: the shard planner, the group-aligned column cuts (gate and up cut at
the same offsets) and the reduction semantics are exact.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import quant as oq
from paper_2410_13461_b200 import tp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _deq_cols(qt, slices, p):
    codes, mins, dels = tp.shard_columns_host(qt.codes, qt.mins, qt.deltas, slices, qt.group_size)
    sub = oq.QTensor(qt.rows, codes.shape[1], qt.group_size, qt.p_max, mins, dels, oq.pack_planes(codes, qt.p_max))
    return oq.dequantize(sub, p)


def _deq_rows(qt, sl, p):
    codes = qt.codes[sl.start:sl.stop]
    sub = oq.QTensor(sl.size, qt.cols, qt.group_size, qt.p_max, qt.mins[sl.start:sl.stop],
                     qt.deltas[sl.start:sl.stop], oq.pack_planes(codes, qt.p_max))
    return oq.dequantize(sub, p)


def _model(d, H, ff, V, seed):
    rng = np.random.default_rng(seed)
    w = lambda *s: (0.05 * rng.standard_normal(s)).astype(np.float32)  # noqa: E731
    return {"qkv": oq.quantize(w(d, 3 * d), 4, 64), "wo": oq.quantize(w(d, d), 4, 64),
            "up": oq.quantize(w(d, 2 * ff), 4, 64), "down": oq.quantize(w(ff, d), 4, 64),
            "head": oq.quantize(w(d, V), 4, 64)}, rng.standard_normal((1, d))


def _reference(m, x, d, ff, p):
    qkv = x @ oq.dequantize(m["qkv"], p)
    h = x + qkv[:, 2 * d:] @ oq.dequantize(m["wo"], p)       # v -> o (stand-in for attention ctx)
    u = h @ oq.dequantize(m["up"], p)
    a = u[:, :ff] / (1 + np.exp(-u[:, :ff])) * u[:, ff:]
    h = h + a @ oq.dequantize(m["down"], p)
    return h @ oq.dequantize(m["head"], p)


def _worker(rank, world, port, d, H, ff, V, p, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, x = _model(d, H, ff, V, seed=3)
    plan = tp.plan_layer(d, H, ff, world, rank)
    qkv = x @ _deq_cols(m["qkv"], plan.qkv_cols, p)                   # column-parallel: local q|k|v heads
    v_loc = qkv[:, 2 * plan.o_rows.size:]
    part = v_loc @ _deq_rows(m["wo"], plan.o_rows, p)                 # row-parallel o
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    h = x + t.numpy()
    u = h @ _deq_cols(m["up"], plan.up_cols, p)                       # gate|up cut at the same offsets
    g, up = u[:, :plan.ff.size], u[:, plan.ff.size:]
    part = (g / (1 + np.exp(-g)) * up) @ _deq_rows(m["down"], plan.down_rows, p)
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    h = h + t.numpy()
    hs = tp.plan_head(V, world, rank)
    logits_loc = torch.from_numpy(np.ascontiguousarray(h @ _deq_cols(m["head"], [hs], p)))
    sizes = [tp.plan_head(V, world, r).size for r in range(world)]
    mx = max(sizes)
    padded = torch.zeros((1, mx), dtype=torch.float64)
    padded[:, :hs.size] = logits_loc
    gathered = [torch.zeros((1, mx), dtype=torch.float64) for _ in sizes]
    dist.all_gather(gathered, padded)   # shards are uneven by at most one group: pad, gather, trim
    if rank == 0:
        out.put(torch.cat([g[:, :s] for g, s in zip(gathered, sizes)], dim=1).numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,d,H,ff,V", [(2, 256, 4, 576, 320), (2, 128, 2, 192, 200), (4, 512, 8, 704, 1000)])
@pytest.mark.parametrize("p", [4, 2])
def test_tp_chain_equals_unsharded(world, d, H, ff, V, p):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, H, ff, V, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    m, x = _model(d, H, ff, V, seed=3)
    want = _reference(m, x, d, ff, p)
    assert np.allclose(got, want, rtol=1e-10, atol=1e-10)


def test_split_aligned_and_plans():
    sl = tp.split_aligned(11008, 8, 64)
    assert sl[0].start == 0 and sl[-1].stop == 11008
    assert all(s.start % 64 == 0 for s in sl) and all(b.start == a.stop for a, b in zip(sl, sl[1:]))
    assert max(s.size for s in sl) - min(s.size for s in sl) <= 64
    plan = tp.plan_layer(4096, 32, 11008, 8, 3)
    assert plan.heads.size == 4 and plan.o_rows == tp.Slice(1536, 2048)
    assert plan.qkv_cols[1] == tp.Slice(4096 + 1536, 4096 + 2048)
    assert plan.up_cols[1].start - plan.up_cols[0].start == 11008
    with pytest.raises(Exception):
        tp.split_aligned(100, 4, 64)


# ---------------------------------------------------------------------------
# tpmodel collective layer: DistComm + lockstep + distributed greedy argmax (gloo, world 2/4)
# ---------------------------------------------------------------------------

def _rank_logits(V, world, rank, seed):
    """Full logits with deliberate cross-shard ties; this rank's vocabulary slice."""
    rng = np.random.default_rng(seed)
    full = rng.standard_normal(V).astype(np.float32)
    top = full.max() + 1.0
    for j in (V - 1, V // 2, 3 * V // 4):  # the max appears in several shards
        full[j] = top
    sl = tp.plan_head(V, world, rank)
    return full, sl


def _argmax_worker(rank, world, port, V, seed, out):
    from paper_2410_13461_b200.tpmodel import DistComm, combine_argmax, lockstep
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = DistComm()
    full, sl = _rank_logits(V, world, rank, seed)
    loc = torch.from_numpy(full[sl.start:sl.stop].copy())

    def gen():
        y = torch.full((2, 3), float(rank + 1))
        yield "sum", y                          # in-place all-reduce
        li = int(torch.argmax(loc))             # first occurrence = lowest local index
        pair = torch.tensor([float(loc[li]), float(li + sl.start), 0.0])
        pairs = yield "gather", pair
        tok, bad = combine_argmax(torch.stack(pairs))
        return y, int(tok.item()), int(bad.item())
    (y, tok, bad), = lockstep([gen()], comm)
    if rank == 0:
        out.put((y.numpy(), tok, bad))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,V", [(2, 257), (4, 1000), (2, 32000)])
def test_tp_distributed_argmax_lowest_index_on_ties(world, V):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_argmax_worker, args=(r, world, port, V, 9, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    y, tok, bad = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    full, _ = _rank_logits(V, world, 0, 9)
    assert tok == int(np.argmax(full))          # np.argmax: lowest index among the tied maxima
    assert bad == 0
    assert np.array_equal(y, np.full((2, 3), world * (world + 1) / 2))


def test_combine_argmax_rules():
    from paper_2410_13461_b200.tpmodel import combine_argmax
    pairs = torch.tensor([[1.0, 5.0, 0.0], [3.0, 70.0, 0.0], [3.0, 130.0, 0.0], [2.0, 200.0, 0.0]])
    tok, bad = combine_argmax(pairs)
    assert int(tok) == 70 and int(bad) == 0
    pairs[3, 2] = 1.0
    assert int(combine_argmax(pairs)[1]) == 1
    pairs = torch.tensor([[float("nan"), 5.0, 1.0], [3.0, 70.0, 0.0]])
    tok, bad = combine_argmax(pairs)
    assert int(bad) == 1  # non-finite logits are flagged (the caller raises InputError)


def test_lockstep_detects_diverged_ranks():
    from paper_2410_13461_b200.errors import ContractViolation
    from paper_2410_13461_b200.tpmodel import LocalComm, lockstep

    def g(op):
        yield op, torch.zeros(1)
    with pytest.raises(ContractViolation):
        lockstep([g("sum"), g("gather")], LocalComm(2))
    a, b = torch.ones(2), torch.full((2,), 2.0)

    def h(t):
        yield "sum", t
        return t.clone()
    r = lockstep([h(a), h(b)], LocalComm(2))
    assert torch.equal(r[0], torch.full((2,), 3.0)) and torch.equal(r[1], r[0])
