"""Streaming PMPD v1 loader (reference quant.py:237-318, tinylm.py:233-257).

A 7B-shape model file (32 layers, d 4096, ff 11008, vocab 32000: 4.1 GB of planes and scales) is
written tensor by tensor and loaded in a fresh process straight into HBM: the loader's peak host
RSS stays under 2 GB, every tensor is bit-identical, and re-saving reproduces the file byte for
byte.  The small-file cases check the reader against the in-memory reader (same bytes, same
FormatError messages).
"""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2410_13461_b200 import quant, tinylm
from paper_2410_13461_b200.errors import FormatError

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tensor_sha(t):
    h = hashlib.sha256()
    for a in (t.mins, t.deltas, t.store.planes):
        h.update(a.cpu().numpy().tobytes())
    return h.hexdigest()


def _file_sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(64 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


CHILD = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import torch
from paper_2410_13461_b200 import tinylm
m = tinylm.ModelVariants.load(sys.argv[2])
torch.cuda.synchronize()
# peak RSS of THIS process image: VmHWM belongs to the address space created by exec (ru_maxrss
# would carry the forking pytest process's peak across fork + exec)
rss = next(int(l.split()[1]) * 1024 for l in open("/proc/self/status") if l.startswith("VmHWM:"))
shas = {}
for name, t in m.tensors.items():
    h = hashlib.sha256()
    for a in (t.mins, t.deltas, t.store.planes):
        h.update(a.cpu().numpy().tobytes())
    shas[name] = h.hexdigest()
m.save(sys.argv[3])
print(json.dumps({"rss": rss, "shas": shas}))
"""


def test_streaming_loader_7b_shape(tmp_path):
    cfg = tinylm.ModelConfig(n_layers=32, n_heads=32, d_model=4096, d_ff=11008, vocab_size=32000, max_context=1024)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    tensors = {}
    for name, shape in tinylm._weight_shapes(cfg):
        w = torch.randn(shape, generator=g, device="cuda").mul_(0.02)
        tensors[name] = quant.quantize_tensor(w, 4, 64)
        del w
    norms = {n: np.ones(cfg.d_model, dtype=np.float32) for n in tinylm._norm_names(cfg)}
    m = tinylm.ModelVariants(cfg, quant.PrecisionSet((4, 3, 2)), tensors, norms)
    f1, f2 = tmp_path / "m7b.pmpd", tmp_path / "m7b_resaved.pmpd"
    m.save(f1)
    want = {n: _tensor_sha(t) for n, t in tensors.items()}
    del m, tensors
    torch.cuda.empty_cache()
    assert os.path.getsize(f1) > 4_000_000_000
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(f1), str(f2)], check=True, capture_output=True,
                         text=True, timeout=900)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["shas"] == want
    assert res["rss"] < 2 << 30, res["rss"]
    assert _file_sha(f1) == _file_sha(f2)


def test_streaming_reader_matches_in_memory_reader(tmp_path):
    rng = np.random.default_rng(4)
    tensors = {"a": quant.quantize_tensor(rng.normal(size=(5, 12)), 3, 4),
               "b": quant.quantize_tensor(rng.normal(size=(70, 130)), 3, 4)}
    path = tmp_path / "two.pmpd"
    quant.write_model(path, tensors, {"note": "fixture"})
    blob = path.read_bytes()
    assert blob == quant.serialize_model(tensors, {"note": "fixture"})
    t2, meta = quant.read_model(path)
    t3, meta3 = quant.parse_model(blob)
    assert meta == meta3
    for n in tensors:
        assert _tensor_sha(t2[n]) == _tensor_sha(t3[n]) == _tensor_sha(tensors[n])
    # corrupted files: the same FormatError text as the in-memory reader
    for bad in (blob[:-3], blob + b"xx", b"PMPX" + blob[4:], blob[:20]):
        p = tmp_path / "bad.pmpd"
        p.write_bytes(bad)
        with pytest.raises(FormatError) as e1:
            quant.read_model(p)
        with pytest.raises(FormatError) as e2:
            quant.parse_model(bad)
        assert str(e1.value) == str(e2.value)


def test_seeded_model_precision16_is_lazy(tmp_path):
    """A file saved with its init seed serves precision 16 after loading (tinylm.py:252-256), the
    originals regenerated on first use only."""
    cfg = tinylm.ModelConfig(n_layers=1, n_heads=2, d_model=64, d_ff=64, max_context=32)
    m = tinylm.ModelVariants.from_random(cfg, quant.PrecisionSet((4, 2)), seed=9)
    m.save(tmp_path / "s.pmpd")
    m2 = tinylm.ModelVariants.load(tmp_path / "s.pmpd")
    assert isinstance(m2.full_weights, tinylm.SeededFullWeights) and m2.full_weights._dev is None
    w16 = m2.weights("layers.0.wq", 16)
    assert torch.equal(w16.cpu(), torch.from_numpy(m.full_weights["layers.0.wq"]))
    assert 16 in m2.allowed_precisions()
