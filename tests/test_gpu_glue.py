"""Decoder glue kernels (csrc/model.cu) against plain torch fp32 restatements of
tinylm.py:293-295 (RMSNorm) and tinylm.py:349-358 (causal attention over the cache).

Covers the cluster-split attention (head dims 32/64/128/256, contexts shorter than
the split, ragged chunks, prefill rows with causal lengths) and the generic
fallback (head dim 48), plus the vectorised and generic RMSNorm paths."""
import math

import pytest
import torch

from paper_2410_13461_b200 import _capi

pytestmark = pytest.mark.gpu


def _ref_attention(q, kc, vc, T, d, dh, scale):
    m = q.shape[0]
    H = d // dh
    out = torch.empty(m, d, dtype=torch.float64)
    for i in range(m):
        L = T + i + 1
        for h in range(H):
            qh = q[i, h * dh:(h + 1) * dh].double()
            k = kc[:L, h * dh:(h + 1) * dh].double()
            v = vc[:L, h * dh:(h + 1) * dh].double()
            a = torch.softmax((k @ qh) * scale, dim=0)
            out[i, h * dh:(h + 1) * dh] = a @ v
    return out


@pytest.mark.parametrize("dh,H,T,m", [(32, 2, 0, 1), (32, 2, 5, 1), (64, 4, 77, 1), (128, 16, 130, 1),
                                      (128, 32, 1023, 1), (256, 2, 300, 1), (128, 4, 0, 37), (32, 2, 9, 20),
                                      (48, 2, 50, 3)])
def test_attention_vs_torch(dh, H, T, m):
    torch.manual_seed(dh + H + T + m)
    d = dh * H
    cap = T + m + 3
    kc = (torch.randn(cap, d, device="cuda") * 0.5).half()
    vc = torch.randn(cap, d, device="cuda").half()
    q = torch.randn(m, d, device="cuda") * 0.5
    out = torch.zeros(m, d, dtype=torch.float16, device="cuda")
    T_dev = torch.tensor([T], dtype=torch.int32, device="cuda")
    scale = 1.0 / math.sqrt(dh)
    _capi.call("pmpd_attention", q.data_ptr(), m, d, dh, kc.data_ptr(), vc.data_ptr(), T_dev.data_ptr(), cap, scale,
               out.data_ptr(), None)
    torch.cuda.synchronize()
    ref = _ref_attention(q.cpu(), kc.float().cpu(), vc.float().cpu(), T, d, dh, scale)
    got = out.double().cpu()
    rel = ((got - ref).norm() / ref.norm()).item()
    assert rel < 2e-3, rel
    assert torch.isfinite(got).all()


@pytest.mark.parametrize("m,d", [(1, 64), (3, 512), (1, 2048), (5, 4096), (2, 8192), (1, 10000), (2, 66)])
def test_rmsnorm_vs_torch(m, d):
    torch.manual_seed(m * d)
    x = torch.randn(m, d, device="cuda") * 3
    g = torch.rand(d, device="cuda") + 0.5
    out = torch.zeros(m, d, dtype=torch.float16, device="cuda")
    _capi.call("pmpd_rmsnorm", x.data_ptr(), d, g.data_ptr(), m, d, 1e-6, out.data_ptr(), d, None)
    torch.cuda.synchronize()
    xd = x.double()
    ref = xd / torch.sqrt((xd * xd).mean(dim=1, keepdim=True) + 1e-6) * g.double()
    torch.testing.assert_close(out.double(), ref, rtol=2e-3, atol=2e-3)


@pytest.mark.parametrize("dh,H,T", [(32, 2, 0), (32, 4, 13), (64, 4, 77), (128, 32, 500), (256, 2, 9)])
def test_attention_rope_matches_two_kernels(dh, H, T):
    """pmpd_attention_rope == pmpd_rope_kv + pmpd_attention for one decode query: same output and
    the same cache row T."""
    torch.manual_seed(dh * H + T)
    d = dh * H
    cap = T + 4
    half = dh // 2
    ang = torch.arange(cap, dtype=torch.float64)[:, None] * (1e4 ** (-torch.arange(0, dh, 2, dtype=torch.float64) / dh))
    cos_t, sin_t = torch.cos(ang).float().cuda().contiguous(), torch.sin(ang).float().cuda().contiguous()
    assert cos_t.shape == (cap, half)
    k0 = (torch.randn(cap, d, device="cuda") * 0.5).half()
    v0 = torch.randn(cap, d, device="cuda").half()
    qkv = torch.randn(1, 3 * d, device="cuda")
    T_dev = torch.tensor([T], dtype=torch.int32, device="cuda")
    scale = 1.0 / math.sqrt(dh)
    # reference: two kernels
    k1, v1 = k0.clone(), v0.clone()
    q = torch.zeros(1, d, device="cuda")
    out1 = torch.zeros(1, d, dtype=torch.float16, device="cuda")
    _capi.call("pmpd_rope_kv", qkv.data_ptr(), 3 * d, 1, d, dh, cos_t.data_ptr(), sin_t.data_ptr(), T_dev.data_ptr(),
               cap, q.data_ptr(), k1.data_ptr(), v1.data_ptr(), None)
    _capi.call("pmpd_attention", q.data_ptr(), 1, d, dh, k1.data_ptr(), v1.data_ptr(), T_dev.data_ptr(), cap, scale,
               out1.data_ptr(), None)
    # fused
    k2, v2 = k0.clone(), v0.clone()
    out2 = torch.zeros(1, d, dtype=torch.float16, device="cuda")
    _capi.call("pmpd_attention_rope", qkv.data_ptr(), d, dh, cos_t.data_ptr(), sin_t.data_ptr(), T_dev.data_ptr(), cap,
               scale, k2.data_ptr(), v2.data_ptr(), out2.data_ptr(), None)
    torch.cuda.synchronize()
    assert torch.equal(v1, v2)
    assert (k1.float() - k2.float()).abs().max().item() <= 1e-3 * k1.float().abs().max().item()
    rel = ((out1.float() - out2.float()).norm() / out1.float().norm()).item()
    assert rel < 2e-3, rel


@pytest.mark.parametrize("m,ff,pad", [(1, 5632, 0), (512, 11008, 0), (3, 13, 1), (7, 96, 3)])
def test_silu_mul_matches_torch(m, ff, pad):
    """out = f16(silu(u[:, :ff]) * u[:, ff:]) (tinylm.py:362-364), vectorised and ragged/unaligned rows."""
    from paper_2410_13461_b200 import _capi
    ldu = 2 * ff + pad
    u = torch.randn(m, ldu, device="cuda") * 3
    out = torch.zeros(m, ff + pad, dtype=torch.float16, device="cuda")
    _capi.call("pmpd_silu_mul", u.data_ptr(), ldu, m, ff, out.data_ptr(), ff + pad, torch.cuda.current_stream().cuda_stream)
    g, up = u[:, :ff].double(), u[:, ff:2 * ff].double()
    want = g / (1 + torch.exp(-g)) * up
    got = out[:, :ff].double()
    assert torch.allclose(got, want, rtol=2e-3, atol=2e-3)
    assert torch.all(out[:, ff:] == 0)
