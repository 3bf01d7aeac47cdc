"""Batched greedy generation (the offline schedule search's inner loop).

BASELINE config-2 model (MobileLLaMA-1.4B shape, random init N(0, 0.02^2), seeded), B prompts of
128 uniform ids, 256 greedy tokens each under the config-2 schedule (3-bit, 2-bit from token 64),
4-bit prefill.  Times ``tinylm.generate_batch`` (all B sequences per decode step: n-row GEMVs,
per-sequence attention) against B sequential ``tinylm.generate`` calls (one persistent-engine
launch per token), end to end from the host (prefills, schedule upload, EOS checks included).

    python tools/batch_bench.py [--batch 1 2 4 8] [--tokens 256]
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
from paper_2410_13461_b200.schedule import PrecisionSchedule, StaticScheduler


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--prompt", type=int, default=128)
    args = ap.parse_args()
    cfg = tinylm.ModelConfig(n_layers=24, n_heads=16, d_model=2048, d_ff=5632, vocab_size=32000,
                             max_context=args.prompt + args.tokens + 8)
    model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
    model.device()
    rng = np.random.default_rng(7)
    prompts = [rng.integers(0, cfg.vocab_size, size=args.prompt).tolist() for _ in range(max(args.batch))]
    sch = StaticScheduler(PrecisionSchedule((3, 2), 4, {3: 0, 2: 64}, args.tokens))
    tinylm.generate_batch(model, prompts[:2], sch, eos_id=-1, max_new=4)  # warm-up (handles, first calls)
    tinylm.generate(model, prompts[0], sch, eos_id=-1, max_new=4)
    for B in args.batch:
        ps = prompts[:B]
        batched, tb = timed(lambda: tinylm.generate_batch(model, ps, sch, eos_id=-1, max_new=args.tokens))
        seq, ts = timed(lambda: [tinylm.generate(model, p, sch, eos_id=-1, max_new=args.tokens) for p in ps])
        same = all(a.output_tokens == b.output_tokens for a, b in zip(batched, seq))
        toks = B * args.tokens
        print(json.dumps({"batch": B, "tokens_per_seq": args.tokens, "batched_s": round(tb, 3),
                          "sequential_s": round(ts, 3), "batched_tok_per_s": round(toks / tb, 1),
                          "sequential_tok_per_s": round(toks / ts, 1), "speedup": round(ts / tb, 2),
                          "traces_identical": same}), flush=True)
    # where traces part: first differing token and the top-2 logit margin there (near-ties of the
    # random-init model flip under f32 rounding differences between the engine and the GEMV path)
    B = max(args.batch)
    a = tinylm.generate_batch(model, prompts[:B], sch, eos_id=-1, max_new=args.tokens, record_logits=True)
    for j in range(B):
        b = tinylm.generate(model, prompts[j], sch, eos_id=-1, max_new=args.tokens, record_logits=True)
        ta, tb_ = a[j].output_tokens, b.output_tokens
        i = next((k for k in range(len(ta)) if ta[k] != tb_[k]), None)
        info = {"seq": j, "first_diff": i}
        if i is not None:
            la, lb = a[j].logits[i].double(), b.logits[i].double()
            top = torch.topk(lb, 2).values
            info.update(margin_ref=float(top[0] - top[1]), max_abs_logit_diff=float((la - lb).abs().max()),
                        logits_rel_l2_before=float(((a[j].logits[:i] - b.logits[:i]).norm() /
                                                    b.logits[:i].norm()).item()) if i else None)
        print(json.dumps(info), flush=True)


if __name__ == "__main__":
    main()
