"""GPU parity of the tcgen05 prefill GEMM (pmpd_gemm) against a float64 reference built from the
bit-exact dequantized weights (quant.py:199-215), and against the decode GEMV."""
import numpy as np
import pytest
import torch

from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.linear import Workspace, gemm, gemv
from paper_2410_13461_b200.quant import dequantize, quantize_tensor
from pmpd_testutil import rel_l2

pytestmark = pytest.mark.gpu


def _pdev(p):
    return torch.tensor([p], dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("K,N", [(64, 64), (256, 192), (512, 1000), (1024, 384)])
@pytest.mark.parametrize("M", [1, 77, 128, 300])
def test_gemm_vs_f64(K, N, M):
    g = torch.Generator(device="cuda").manual_seed(K * 7 + N + M)
    w = torch.randn((K, N), generator=g, device="cuda") * 0.02
    qt = quantize_tensor(w, 4, 64)
    pk = qt.packed(_capi.LAYOUT_KN)
    x = torch.randn((M, K), generator=g, device="cuda").half()
    for p in (4, 3, 2):
        W = dequantize(qt, p, layout=_capi.LAYOUT_KN).double()  # (K, N), bit-exact reference dequant
        ref = (x.double() @ W).cpu().numpy()
        y = gemm(pk, x, _pdev(p)).double().cpu().numpy()
        # f16 weights x f16 activations, f32 accumulation
        assert rel_l2(y, ref) < 2e-3, (K, N, M, p, rel_l2(y, ref))


def test_gemm_matches_gemv_and_accumulates():
    g = torch.Generator(device="cuda").manual_seed(5)
    K, N, M = 4096, 4096, 512
    w = torch.randn((K, N), generator=g, device="cuda") * 0.02
    pk = quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN)
    x = torch.randn((M, K), generator=g, device="cuda").half()
    ws = Workspace()
    for p in (4, 2):
        y = gemm(pk, x, _pdev(p), alpha=0.5)
        y2 = torch.empty_like(y)
        for r0 in range(0, M, 8):
            gemv(pk, x[r0:r0 + 8], _pdev(p), ws, out=y2[r0:r0 + 8], alpha=0.5)
        assert rel_l2(y.cpu().numpy(), y2.cpu().numpy()) < 2e-3
        y3 = y.clone()
        gemm(pk, x, _pdev(p), out=y3, alpha=0.5, accumulate=True)
        assert rel_l2(y3.cpu().numpy(), 2 * y.cpu().numpy()) < 1e-6
    yh = gemm(pk, x, _pdev(4), out_dtype=torch.float16)
    assert yh.dtype == torch.float16 and rel_l2(yh.float().cpu().numpy(), gemm(pk, x, _pdev(4)).cpu().numpy()) < 1e-3


@pytest.mark.parametrize("split", [2, 4])
@pytest.mark.parametrize("K,N,M", [(4096, 4096, 512), (11008, 512, 300), (640, 320, 77)])
def test_gemm_split_k(split, K, N, M, monkeypatch):
    """Split-K (S CTAs per output tile, partials added at L2 into f32 y) == the unsplit GEMM, with and
    without accumulate, and with a strided y (ldy > n)."""
    g = torch.Generator(device="cuda").manual_seed(K + N + M + split)
    w = torch.randn((K, N), generator=g, device="cuda") * 0.02
    pk = quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN)
    x = torch.randn((M, K), generator=g, device="cuda").half()
    monkeypatch.setenv("PMPD_GEMM_SPLITK", "1")
    ref = gemm(pk, x, _pdev(3), alpha=0.75)
    monkeypatch.setenv("PMPD_GEMM_SPLITK", str(split))
    big = torch.full((M, N + 8), 7.0, device="cuda")
    y = big[:, :N]
    gemm(pk, x, _pdev(3), out=y, alpha=0.75)
    torch.cuda.synchronize()
    assert rel_l2(y.cpu().numpy(), ref.cpu().numpy()) < 1e-4  # f32 summation order only
    assert torch.all(big[:, N:] == 7.0)  # the zeroing before the split-K adds stays inside y
    gemm(pk, x, _pdev(3), out=y, alpha=0.75, accumulate=True)
    assert rel_l2(y.cpu().numpy(), 2 * ref.cpu().numpy()) < 1e-4


def test_gemm_split_k_is_bit_reproducible():
    """Split-K partials are added in split order (a per-tile turn counter), not by atomics: the
    same input gives bit-identical outputs every launch, with and without accumulation."""
    import os
    from paper_2410_13461_b200 import _capi, quant
    from paper_2410_13461_b200.linear import gemm
    w = torch.randn(4096, 1024, device="cuda") * 0.02
    pk = quant.quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN)
    x = torch.randn(512, 4096, device="cuda").half()
    pd = torch.tensor([4], dtype=torch.int32, device="cuda")
    old = os.environ.get("PMPD_GEMM_SPLITK")
    os.environ["PMPD_GEMM_SPLITK"] = "4"
    try:
        outs = [gemm(pk, x, pd, out=torch.empty(512, 1024, device="cuda")) for _ in range(4)]
        base = torch.randn(512, 1024, device="cuda")
        accs = []
        for _ in range(3):
            y = base.clone()
            gemm(pk, x, pd, out=y, accumulate=True)
            accs.append(y)
    finally:
        if old is None:
            os.environ.pop("PMPD_GEMM_SPLITK")
        else:
            os.environ["PMPD_GEMM_SPLITK"] = old
    ref = (x.float() @ quant.dequantize(quant.quantize_tensor(w, 4, 64), 4, layout=_capi.LAYOUT_KN))
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    for a in accs[1:]:
        assert torch.equal(a, accs[0])
    assert float((outs[0] - ref).norm() / ref.norm()) < 2e-3
    assert float((accs[0] - base - ref).norm() / ref.norm()) < 2e-3


@pytest.mark.parametrize("split", [2, 4])
@pytest.mark.parametrize("M,K,N", [(512, 4096, 1024), (77, 1024, 1000), (300, 2048, 384)])
def test_gemm_split_k_dsmem_equals_workspace(split, M, K, N, monkeypatch):
    """Split-K reduced on chip (the splits of a tile form a cluster and sum their partial tiles
    through distributed shared memory) gives the same bits as the global-workspace reduction, with
    and without accumulate, into a strided y."""
    g = torch.Generator(device="cuda").manual_seed(M + K + N + split)
    pk = quantize_tensor(torch.randn((K, N), generator=g, device="cuda") * 0.02, 4, 64).packed(_capi.LAYOUT_KN)
    x = torch.randn((M, K), generator=g, device="cuda").half()
    base = torch.randn((M, N + 8), generator=g, device="cuda")
    monkeypatch.setenv("PMPD_GEMM_SPLITK", str(split))
    outs = {}
    for dsm in ("0", "1"):
        monkeypatch.setenv("PMPD_GEMM_DSM", dsm)
        y0 = gemm(pk, x, _pdev(3), alpha=0.5)
        big = base.clone()
        gemm(pk, x, _pdev(3), out=big[:, :N], alpha=0.5, accumulate=True)
        outs[dsm] = (y0, big)
    torch.cuda.synchronize()
    assert torch.equal(outs["0"][0], outs["1"][0])
    assert torch.equal(outs["0"][1], outs["1"][1])
    assert torch.equal(outs["1"][1][:, N:], base[:, N:])
