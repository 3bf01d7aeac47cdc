"""GPU TP path (single-rank NCCL group on the one available B200): the sharded stack with
world=1 must reproduce the unsharded stack; multi-rank sharding logic is covered by
tests/test_tp_cpu.py (gloo, world_size 2/4)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

from paper_2410_13461_b200 import tp
from paper_2410_13461_b200.stack import LinearStack, StackShape, TPLinearStack
from pmpd_testutil import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_tp1_matches_single_gpu_stack(nccl_group):
    shape = StackShape(2, 512, 1024, 2048)
    ref = LinearStack(shape, seed=5)
    t = TPLinearStack(shape, 8, 0, 1, nccl_group, seed=5)
    t.x16.copy_(ref.x0)
    for p in (4, 2):
        ref.set_schedule({p: 0})
        t.set_schedule({p: 0})
        x_in = ref.x0.clone()
        ref.token()
        t.x16.copy_(x_in)
        t.token()
        torch.cuda.synchronize()
        got = t.logits_all[0, :, :shape.vocab].cpu().numpy()
        assert rel_l2(got, ref.logits.cpu().numpy()) < 5e-3, p


def test_shard_rows_and_columns_are_exact_subblocks():
    import numpy as np
    from paper_2410_13461_b200.quant import dequantize, quantize_tensor
    w = np.random.default_rng(0).standard_normal((256, 640)).astype(np.float32)
    qt = quantize_tensor(w, 4, 64)
    full = dequantize(qt, 3).cpu().numpy()
    cols = [tp.Slice(64, 192), tp.Slice(384, 640)]
    sub = dequantize(tp.shard_columns(qt, cols), 3).cpu().numpy()
    assert np.array_equal(sub, np.concatenate([full[:, 64:192], full[:, 384:640]], axis=1))
    rows = dequantize(tp.shard_rows(qt, tp.Slice(100, 200)), 3).cpu().numpy()
    assert np.array_equal(rows, full[100:200])
