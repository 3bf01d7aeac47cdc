"""Per-rank GEMV chain of the tensor-parallel 7B linear stack at world W, on ONE GPU.

Builds rank 0's shards of TPLinearStack for W = 1, 2, 4, 8 and times one token's 129 GEMVs (CUDA graph) with the
collectives stubbed out: the compute share of a rank's token at that TP degree.  The all-reduce latency (64 per
token) adds on top of it in the real multi-GPU run."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import torch.distributed as dist
from paper_2410_13461_b200.stack import LLAMA2_7B, TPLinearStack

dist.all_reduce = lambda *a, **k: None               # noqa: E731  (compute share only)
dist.all_gather_into_tensor = lambda *a, **k: None   # noqa: E731
for W in [int(w) for w in (sys.argv[1:] or ["1", "2", "4", "8"])]:
    st = TPLinearStack(LLAMA2_7B, 32, 0, W, None, seed=1)
    g = st.capture(st.token)
    res = {}
    for p in (4, 3, 2):
        st.set_schedule({p: 0})
        for _ in range(5):
            g.replay()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[p] = round(e0.elapsed_time(e1) * 1e3 / 50, 1)
    print(json.dumps({"world": W, "rank0_gemv_chain_us_per_token": res}), flush=True)
    del st, g
    torch.cuda.empty_cache()
