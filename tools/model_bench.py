"""End-to-end decoder timing on the device model runner (BASELINE configs 2 and 3).

config 2: MobileLLaMA-1.4B shape (24 x d2048, 16 heads, ff 5632, V 32000), prompt 128, 256 tokens,
          schedule 3-bit for tokens 0..63 then 2-bit, 4-bit prefill.
config 3: Llama-2-7B shape (32 x d4096, 32 heads, ff 11008, V 32000), prompt 512, 512 tokens,
          progressive 4->3->2 switching at tokens 32 and 128, 4-bit prefill.
Each is compared with uniform 4-bit and fp16 (precision 16) decoding of the same random-init model
(weights N(0, 0.02^2), seeded; prompt ids uniform).  Prefill runs through the tcgen05 dequant GEMM;
each decode token is one CUDA-graph replay (device precision hook -> 4 GEMVs/layer + attention glue
-> head -> greedy argmax -> token push).  Prints one JSON line per run.

    python tools/model_bench.py [2|3] [--tokens N]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet
from paper_2410_13461_b200.schedule import PrecisionSchedule, avg_bitwidth

CONFIGS = {
    2: dict(cfg=dict(n_layers=24, n_heads=16, d_model=2048, d_ff=5632, vocab_size=32000), prompt=128, tokens=256,
            sched=((3, 2), 4, {3: 0, 2: 64})),
    3: dict(cfg=dict(n_layers=32, n_heads=32, d_model=4096, d_ff=11008, vocab_size=32000), prompt=512, tokens=512,
            sched=((4, 3, 2), 4, {4: 0, 3: 32, 2: 128})),
}


def run(model, prompt, sched, tokens, p16=False):
    """Prefill + timed decode replays; returns (prefill_ms, decode_us_per_token)."""
    cfg = model.config
    eng = tinylm.DecodeEngine(model, tokens + 1, p16=p16)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(True)
    t1 = torch.cuda.Event(True)
    p_pre = 16 if p16 else sched.p_prefill
    warm = tinylm.KVCache(cfg.n_layers, cfg.d_model, cfg.max_context)
    tinylm._forward(model, p_pre, prompt, warm)  # untimed: first-call library/handle setup
    del warm
    torch.cuda.synchronize()
    t0.record()
    logits = tinylm._forward(model, p_pre, prompt, eng.cache)
    t1.record()
    torch.cuda.synchronize()
    prefill_ms = t0.elapsed_time(t1)
    if not p16:
        eng.table.copy_(torch.tensor(sched.device_table(), dtype=torch.int32))
    from paper_2410_13461_b200 import _capi
    s = tinylm._stream()
    V = cfg.vocab_size
    last = logits[-1:].contiguous()
    _capi.call("pmpd_argmax", last.data_ptr(), V, 1, V, eng.buf.ids.data_ptr(), eng.buf.bad.data_ptr(), s)
    _capi.call("pmpd_push_token", eng.buf.ids.data_ptr(), eng.tokens.data_ptr(), eng.n.data_ptr(), 0, tokens + 1, s)
    eng.step.zero_()
    eng.capture()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = tokens - 1
    e0.record()
    for _ in range(n):
        eng.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return prefill_ms, e0.elapsed_time(e1) * 1e3 / n


def measure(config: int, tokens: int | None = None, verbose: bool = False) -> dict:
    """Progressive vs uniform-4 vs fp16 decode (and prefill) of one BASELINE model config."""
    c = CONFIGS[config]
    tokens = tokens or c["tokens"]
    mc = tinylm.ModelConfig(max_context=c["prompt"] + tokens + 8, **c["cfg"])
    t = time.time()
    model = tinylm.ModelVariants.from_random(mc, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
    model.device()
    build_s = time.time() - t
    rng = np.random.default_rng(7)
    prompt = rng.integers(0, mc.vocab_size, size=c["prompt"]).tolist()
    precs, p_pre, st = c["sched"]
    prog = PrecisionSchedule(precs, p_pre, st, tokens)
    uni4 = PrecisionSchedule((4,), 4, {4: 0}, tokens)
    res = {}
    for name, sched, p16 in (("progressive", prog, False), ("uniform4", uni4, False), ("fp16", uni4, True)):
        pre, dec = run(model, prompt, sched, tokens, p16=p16)
        res[name] = {"prefill_ms": pre, "decode_us_per_token": dec}
        if verbose:
            print(json.dumps({"config": config, "run": name, "prefill_ms": round(pre, 3),
                              "decode_us_per_token": round(dec, 2)}), flush=True)
    out = {"config": config, "shape": c["cfg"], "prompt": c["prompt"], "tokens": tokens,
           "schedule": {str(k): v for k, v in st.items()}, "avg_bits": avg_bitwidth(prog, tokens),
           "model_build_s": round(build_s, 1), "runs": res,
           "decode_speedup_vs_uniform4": res["uniform4"]["decode_us_per_token"] / res["progressive"]["decode_us_per_token"],
           "decode_speedup_vs_fp16": res["fp16"]["decode_us_per_token"] / res["progressive"]["decode_us_per_token"]}
    del model
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int, nargs="?", default=2, choices=[2, 3])
    ap.add_argument("--tokens", type=int, default=None)
    args = ap.parse_args()
    print(json.dumps(measure(args.config, args.tokens, verbose=True)), flush=True)


if __name__ == "__main__":
    main()
