import torch, time
from torch.nn.attention import sdpa_kernel, SDPBackend
n, H, dh = 512, 32, 128
q = torch.randn(n, H * dh, device="cuda")
k = torch.randn(n, H * dh, device="cuda").half()
v = torch.randn(n, H * dh, device="cuda").half()
qh = q.view(n, H, dh).transpose(0, 1).half(); kh = k.view(n, H, dh).transpose(0, 1); vh = v.view(n, H, dh).transpose(0, 1)
def t(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 20 * 1e3
ref = torch.nn.functional.scaled_dot_product_attention(qh.float(), kh.float(), vh.float(), is_causal=True, scale=0.088)
for name, args in (("3D", (qh, kh, vh)), ("4D", (qh.unsqueeze(0), kh.unsqueeze(0), vh.unsqueeze(0)))):
    print(name, "default us", round(t(lambda: torch.nn.functional.scaled_dot_product_attention(*args, is_causal=True, scale=0.088)), 1))
    for be in (SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.CUDNN_ATTENTION):
        try:
            with sdpa_kernel(be):
                o = torch.nn.functional.scaled_dot_product_attention(*args, is_causal=True, scale=0.088)
                us = t(lambda: torch.nn.functional.scaled_dot_product_attention(*args, is_causal=True, scale=0.088))
            err = float((o.float().reshape(ref.shape) - ref).norm() / ref.norm())
            print(" ", be, round(us, 1), "us err", err)
        except Exception as e:
            print(" ", be, "fails:", str(e).split("\n")[0][:150])
