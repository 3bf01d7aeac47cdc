"""GPU parity of the persistent decode engine: the whole chained linear stack in one kernel
vs the per-op GEMV chain and vs the float64 oracle."""
import math

import numpy as np
import pytest
import torch

from oracle import quant as oq
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.engine import OpSpec, Program
from paper_2410_13461_b200.quant import quantize_tensor
from paper_2410_13461_b200.stack import LinearStack, StackShape
from pmpd_testutil import rel_l2

pytestmark = pytest.mark.gpu


def _pdev(p):
    return torch.tensor([p], dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("shape", [StackShape(1, 4096, 11008, 32000)])
def test_engine_matches_per_op_chain(shape):
    st = LinearStack(shape, seed=3)
    st.build_engine()
    for p in (4, 3, 2):
        st.set_schedule({p: 0})
        st.token()
        ref = st.logits.clone()
        st.set_schedule({p: 0})
        st.logits.zero_()
        st.token_engine()
        torch.cuda.synchronize()
        err = rel_l2(st.logits.cpu().numpy(), ref.cpu().numpy())
        assert err < 3e-3, (shape, p, err)
        assert int(st.program.bar[:2].sum().item()) == 0  # ticket / done counters self-reset
        assert int(st.program.status.item()) == 0


def _chain_f64(st, p):
    """The LinearStack chain in float64 from bit-exact dequantized weights (test-only reference)."""
    from paper_2410_13461_b200.quant import dequantize
    d, f = st.shape.d_model, st.shape.d_ff
    a_d, a_f = 1.0 / (st.std * math.sqrt(d)), 1.0 / (st.std * math.sqrt(f))
    W = lambda qt: dequantize(qt, p, layout=_capi.LAYOUT_KN).double()  # noqa: E731
    h = st.x0.double()
    for (q1, _), (q2, _), (q3, _), (q4, _) in st.layers:
        qkv = (a_d * (h @ W(q1))).half().double()
        o = (a_d * (qkv[:, 2 * d:] @ W(q2))).half().double()
        u = (a_d * (o @ W(q3))).half().double()
        h = (a_f * (u[:, :f] @ W(q4))).half().double()
    return a_d * (h @ W(st.head[0]))


@pytest.mark.parametrize("shape", [StackShape(2, 256, 512, 1000), StackShape(1, 512, 1376, 2048)])
def test_engine_and_per_op_chain_vs_f64(shape):
    st = LinearStack(shape, seed=3)
    st.build_engine()
    for p in (4, 2):
        ref = _chain_f64(st, p).cpu().numpy()
        st.set_schedule({p: 0})
        st.token()
        per_op = st.logits.clone().cpu().numpy()
        st.set_schedule({p: 0})
        st.token_engine()
        torch.cuda.synchronize()
        eng = st.logits.cpu().numpy()
        assert rel_l2(per_op, ref) < 1e-2, ("per-op", shape, p, rel_l2(per_op, ref))
        assert rel_l2(eng, ref) < 1e-2, ("engine", shape, p, rel_l2(eng, ref))


def test_engine_two_layer_chain_vs_oracle():
    rng = np.random.default_rng(0)
    K, N1, N2 = 320, 384, 200
    w1 = (0.02 * rng.standard_normal((K, N1))).astype(np.float32)
    w2 = (0.02 * rng.standard_normal((N1 - 64, N2))).astype(np.float32)
    x = rng.standard_normal((1, K)).astype(np.float16)
    q1, q2 = quantize_tensor(w1, 4, 64), quantize_tensor(w2, 4, 64)
    a1 = 1.0 / (0.02 * math.sqrt(K))
    prog = Program([OpSpec(q1.packed(_capi.LAYOUT_KN)),
                    OpSpec(q2.packed(_capi.LAYOUT_KN), src=0, src_col=64, in_alpha=a1)], y_alpha=0.5)
    y = torch.zeros(N2, device="cuda")
    xd = torch.from_numpy(x).cuda()
    r1, r2 = oq.quantize(w1, 4, 64), oq.quantize(w2, 4, 64)
    for p in (4, 3, 2):
        prog.run(xd, _pdev(p), y)
        h = a1 * (x.astype(np.float64) @ oq.dequantize(r1, p))
        h16 = h[:, 64:].astype(np.float16).astype(np.float64)
        want = 0.5 * (h16 @ oq.dequantize(r2, p))
        assert rel_l2(y.cpu().numpy(), want[0]) < 3e-3, p


def test_engine_silu_input_transform():
    rng = np.random.default_rng(1)
    K, F, N = 256, 192, 128
    wu = (0.05 * rng.standard_normal((K, 2 * F))).astype(np.float32)
    wd = (0.05 * rng.standard_normal((F, N))).astype(np.float32)
    x = rng.standard_normal((1, K)).astype(np.float16)
    qu, qd = quantize_tensor(wu, 4, 64), quantize_tensor(wd, 4, 64)
    prog = Program([OpSpec(qu.packed(_capi.LAYOUT_KN)),
                    OpSpec(qd.packed(_capi.LAYOUT_KN), src=0, src_col=0, act=1, act_off=F, in_alpha=1.0)])
    y = torch.zeros(N, device="cuda")
    prog.run(torch.from_numpy(x).cuda(), _pdev(4), y)
    u = x.astype(np.float64) @ oq.dequantize(oq.quantize(wu, 4, 64), 4)
    g, up = u[:, :F], u[:, F:]
    a = (g / (1 + np.exp(-g)) * up).astype(np.float16).astype(np.float64)
    want = a @ oq.dequantize(oq.quantize(wd, 4, 64), 4)
    assert rel_l2(y.cpu().numpy(), want[0]) < 3e-3


def test_engine_counted_accumulation_is_deterministic():
    """Split-K partials land in any order, but the counted fixed-point sums are integer adds:
    every launch (both parity sets, several epochs) gives bit-identical logits, equal to the
    per-op chain within the usual tolerance (same input -> same logits)."""
    st = LinearStack(StackShape(1, 4096, 11008, 32000), seed=4)
    st.build_engine()
    counts = [t for part in st.program.parts if len(part) == 2 for t in part[1:]]
    assert max(int(c.max()) for c in counts) >= 2  # n-groups really are shared by several CTAs
    for p in (4, 2):
        st.set_schedule({p: 0})
        outs = []
        for _ in range(5):
            st.token_engine()
            outs.append(st.logits.clone())
        torch.cuda.synchronize()
        for o in outs[1:]:
            assert torch.equal(o, outs[0]), p
        st.token()
        assert rel_l2(outs[0].cpu().numpy(), st.logits.cpu().numpy()) < 3e-3
    assert int(st.program.status.item()) == 0


def test_engine_flags_out_of_range_partials():
    """A partial outside the fixed-point range (|v| >= 2^23, far beyond f16) still counts, adds
    zero and sets the status word (InputError class), so no consumer waits forever."""
    rng = np.random.default_rng(2)
    K, N = 256, 128
    w = (50.0 * rng.standard_normal((K, N))).astype(np.float32)
    prog = Program([OpSpec(quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN))])
    y = torch.zeros(N, device="cuda")
    prog.run(torch.full((1, K), 60000.0, dtype=torch.float16, device="cuda"), _pdev(4), y)
    torch.cuda.synchronize()
    assert int(prog.status.item()) == _capi.ERR_INPUT
    prog.status.zero_()
    prog.run(torch.full((1, K), 1.0, dtype=torch.float16, device="cuda"), _pdev(4), y)
    torch.cuda.synchronize()
    assert int(prog.status.item()) == 0
    want = np.ones(K) @ oq.dequantize(oq.quantize(w, 4, 64), 4)
    assert rel_l2(y.cpu().numpy(), want) < 2e-3


@pytest.mark.parametrize("scale", [100.0, 1000.0])
def test_engine_outlier_activations(scale):
    """Outlier input channels through the engine's int16 activation path (one scale per op)."""
    rng = np.random.default_rng(5)
    K, N = 4096, 4096
    w = (0.02 * rng.standard_normal((K, N))).astype(np.float32)
    x = rng.standard_normal((1, K))
    x[0, rng.choice(K, 6, replace=False)] *= scale
    x = x.astype(np.float16)
    prog = Program([OpSpec(quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN))])
    y = torch.zeros(N, device="cuda")
    for p in (4, 2):
        prog.run(torch.from_numpy(x).cuda(), _pdev(p), y)
        want = x.astype(np.float64) @ oq.dequantize(oq.quantize(w, 4, 64), p)
        assert rel_l2(y.cpu().numpy(), want[0]) < 5e-3, (scale, p)  # measured ~1.5e-3


@pytest.mark.parametrize("groups", [2, 4])
def test_paired_program_vs_f64(groups):
    """Sub-op program (k-sliced row-parallel ops on CTA groups, shared counted outputs, reused
    input staging): same chain as the plain program, checked against the float64 chain and for
    bit-reproducibility."""
    st = LinearStack(StackShape(2, 512, 1536, 2048), seed=5)
    prog = st.build_engine(paired=True, groups=groups)
    assert len(prog.ops) == 2 * (4 + 2 * groups) + 1
    for p in (4, 3, 2):
        ref = _chain_f64(st, p).cpu().numpy()
        st.set_schedule({p: 0})
        st.token_engine()
        first = st.logits.clone()
        st.token_engine()
        torch.cuda.synchronize()
        assert torch.equal(first, st.logits), p
        assert rel_l2(st.logits.cpu().numpy(), ref) < 1e-2, (groups, p)
    assert int(prog.status.item()) == 0
    assert int(prog.bar[:2].sum().item()) == 0


def test_paired_program_matches_plain_at_7b_width():
    st = LinearStack(StackShape(1, 4096, 11008, 32000), seed=3)
    out = {}
    for paired in (False, True):
        st.build_engine(paired=paired)
        for p in (4, 2):
            st.set_schedule({p: 0})
            st.token_engine()
            torch.cuda.synchronize()
            out[(paired, p)] = st.logits.cpu().numpy()
        assert int(st.program.status.item()) == 0
    for p in (4, 2):
        assert rel_l2(out[(True, p)], out[(False, p)]) < 3e-3, p
