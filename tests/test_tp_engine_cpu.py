"""Host side of tensor parallelism inside the engine (no GPU; gloo for the multi-process part).

Every rank of ``engine.RankProgram`` must derive the SAME contributor totals for a row-parallel
output (the sum over ranks of each rank's partition counts): the counted words are complete when
their count reaches that total, on every rank's copy.  The partitions come from the library's host
function (no GPU needed)."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_13461_b200 import _capi, tp


def _counts(rows, cols, G):
    import ctypes
    d = _capi.describe(rows, cols, 64, 4, _capi.LAYOUT_KN)
    b = (ctypes.c_int32 * (G + 1))()
    _capi.call("pmpd_engine_partition_g", ctypes.byref(d), G, ctypes.addressof(b))
    kt, cnt = d.k_tiles, [0] * d.n_tiles
    for c in range(G):
        if b[c + 1] > b[c]:
            for ng in range(b[c] // kt, (b[c + 1] - 1) // kt + 1):
                cnt[ng] += 1
    assert b[0] == 0 and b[G] == d.n_tiles * d.k_tiles and all(b[c] <= b[c + 1] for c in range(G))
    return cnt


def _row_totals(world, G, d=4096, f=11008, heads=32):
    """Totals of the o and down outputs (d wide) over the ranks' row shards."""
    plans = [tp.plan_layer(d, heads, f, world, r) for r in range(world)]
    o = [sum(v) for v in zip(*[_counts(p.o_rows.size, d, G) for p in plans])]
    dn = [sum(v) for v in zip(*[_counts(p.down_rows.size, d, G) for p in plans])]
    return o, dn


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_row_parallel_totals(world):
    G = 148 // world
    o, dn = _row_totals(world, G)
    assert len(o) == len(dn) == 64
    assert 1 <= min(o) and max(o) <= 255 and 1 <= min(dn) and max(dn) <= 255
    # each rank contributes at least one CTA to every n-group of its row shard's output
    assert min(o) >= world and min(dn) >= world


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    G = 148  # one GPU per rank in the distributed form
    o, dn = _row_totals(world, G)
    t = torch.tensor(o + dn, dtype=torch.int64)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    out[rank] = all(torch.equal(g, gathered[0]) for g in gathered)
    dist.destroy_process_group()


def test_totals_agree_across_processes():
    """Two processes (gloo) derive identical totals independently: no exchange of counts is needed
    when the program is built, every rank computes all ranks' partitions itself."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, 29631, out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
