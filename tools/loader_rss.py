"""RSS of the streaming loader at each stage (debug for tests/test_gpu_loader.py)."""
import os, resource, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def rss(tag):
    cur = int(open("/proc/self/statm").read().split()[1]) * 4096
    print(f"{tag:30s} cur {cur / 2**30:6.2f} GB  peak {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20:6.2f} GB", flush=True)

rss("start")
import numpy as np, torch
rss("import torch")
torch.zeros(1, device="cuda")
rss("cuda init")
from paper_2410_13461_b200 import quant, tinylm
path = "/tmp/m_rss.pmpd"
if not os.path.exists(path):
    cfg = tinylm.ModelConfig(n_layers=int(sys.argv[1]) if len(sys.argv) > 1 else 8, n_heads=32, d_model=4096, d_ff=11008,
                             vocab_size=32000, max_context=1024)
    g = torch.Generator(device="cuda"); g.manual_seed(3)
    tensors = {}
    for name, shape in tinylm._weight_shapes(cfg):
        w = torch.randn(shape, generator=g, device="cuda").mul_(0.02)
        tensors[name] = quant.quantize_tensor(w, 4, 64)
        del w
    rss("quantized")
    norms = {n: np.ones(cfg.d_model, dtype=np.float32) for n in tinylm._norm_names(cfg)}
    tinylm.ModelVariants(cfg, quant.PrecisionSet((4, 3, 2)), tensors, norms).save(path)
    rss("saved")
    print("written; rerun to load"); sys.exit(0)
m = tinylm.ModelVariants.load(path)
torch.cuda.synchronize()
rss("loaded")
m.save(path + ".2")
rss("re-saved")
