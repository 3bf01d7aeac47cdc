"""Tensor parallelism inside the persistent engine (reference sites tinylm.py:359,364).

``TPEngineStack`` shards the 7B-width linear stack over 2 / 4 / 8 ranks (Megatron: q|k|v by heads,
gate|up at matching offsets, head by vocabulary; o and down by rows) and runs every rank's token in
the engine, the row-parallel all-reduce being the counted fixed-point addition of all ranks'
partials.  With one GPU the ranks are CTA groups of one launch.  The sharded stack must compute the
1-GPU stack's function (same weights, same generator) and be bit-reproducible."""
import pytest
import torch

from paper_2410_13461_b200.stack import LinearStack, StackShape, TPEngineStack
from pmpd_testutil import rel_l2

pytestmark = pytest.mark.gpu

SHAPE = StackShape(1, 4096, 11008, 32000)


@pytest.fixture(scope="module")
def single():
    st = LinearStack(SHAPE, seed=7)
    st.build_engine()
    out = {}
    for p in (4, 2):
        st.set_schedule({p: 0})
        st.token_engine()
        out[p] = st.logits[0].clone()
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("world", [2, 4, 8])
def test_tp_engine_matches_single_gpu(single, world):
    tp = TPEngineStack(SHAPE, n_heads=32, world=world, seed=7)
    for p in (4, 2):
        tp.set_schedule({p: 0})
        runs = []
        for _ in range(3):
            tp.token()
            runs.append(tp.logits().clone())
        torch.cuda.synchronize()
        for r in runs[1:]:
            assert torch.equal(r, runs[0]), (world, p)
        err = rel_l2(runs[0].cpu().numpy(), single[p].cpu().numpy())
        assert err < 3e-3, (world, p, err)
    assert int(tp.program.status.item()) == 0


def test_tp_engine_distributed_form_world1(single, tmp_path):
    """The one-process-per-GPU form at world 1: the shared vectors are torch symmetric-memory
    buffers added into with system-scope atomics and polled with system-scope loads."""
    import os
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tp = TPEngineStack(SHAPE, n_heads=32, world=1, seed=7, group=dist.group.WORLD, rank=0)
        for p in (4, 2):
            tp.set_schedule({p: 0})
            tp.token()
            tp.token()
            torch.cuda.synchronize()
            err = rel_l2(tp.logits().cpu().numpy(), single[p].cpu().numpy())
            assert err < 3e-3, (p, err)
    finally:
        dist.destroy_process_group()
