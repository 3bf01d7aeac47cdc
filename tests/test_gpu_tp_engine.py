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
        tp.p_dev.fill_(p)
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
