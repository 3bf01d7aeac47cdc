"""Time the 7B linear stack's prefill (129 GEMMs at M=512, p=4) as bench.py does."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2410_13461_b200.stack import LLAMA2_7B, LinearStack
st = LinearStack(LLAMA2_7B, seed=1234)
for _ in range(2):
    print(bench.bench_prefill(st, LLAMA2_7B))
