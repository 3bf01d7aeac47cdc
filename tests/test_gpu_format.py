"""GPU parity of the weight format: device quantizer, packer, prefix reader and dequantizer
against the oracle and the reference golden vectors (bit-exact)."""
import numpy as np
import pytest
import torch

from oracle import quant as oq
from paper_2410_13461_b200 import _capi, quant
from paper_2410_13461_b200.errors import ConfigError, InputError

pytestmark = pytest.mark.gpu

LAYOUTS = [_capi.LAYOUT_REF, _capi.LAYOUT_KN, _capi.LAYOUT_NK]


def host(t):
    return t.detach().cpu().numpy()


def test_quantize_matches_reference_golden(gold_quant):
    for name in gold_quant["names"]:
        r, c, g, pm = (int(v) for v in gold_quant[f"{name}/meta"])
        qt = quant.quantize_tensor(gold_quant[f"{name}/w"], pm, g)
        assert np.array_equal(host(qt.mins).view(np.uint32), gold_quant[f"{name}/mins"].view(np.uint32)), name
        assert np.array_equal(host(qt.deltas).view(np.uint32), gold_quant[f"{name}/deltas"].view(np.uint32)), name
        assert np.array_equal(host(qt.store.planes), gold_quant[f"{name}/planes"]), name
        for p in range(1, pm + 1):
            assert np.array_equal(host(quant.unpack_prefix(qt.store, p)), gold_quant[f"{name}/prefix{p}"])
            d = host(quant.dequantize(qt, p))
            assert np.array_equal(d.view(np.uint32), gold_quant[f"{name}/deq{p}"].astype(np.float32).view(np.uint32))


@pytest.mark.parametrize("shape", [(64, 64), (128, 320), (257, 64), (100, 200), (512, 1024), (64, 11008 // 4)])
@pytest.mark.parametrize("dtype", [np.float32, np.float16])
def test_quantize_bit_exact_random(shape, dtype):
    rng = np.random.default_rng(sum(shape))
    w = (0.02 * rng.standard_normal(shape)).astype(dtype)
    ref = oq.quantize(w.astype(np.float64), 4, 64)
    qt = quant.quantize_tensor(w, 4, 64)
    assert np.array_equal(host(qt.store.planes), ref.planes)
    assert np.array_equal(host(qt.mins), ref.mins) and np.array_equal(host(qt.deltas), ref.deltas)


def test_quantize_errors():
    with pytest.raises(InputError):
        quant.quantize_tensor(np.array([[np.nan, 1.0]]), 4, 2)
    with pytest.raises(ConfigError):
        quant.quantize_tensor(np.ones((2, 2)), 9, 2)
    with pytest.raises(ConfigError):
        quant.dequantize(quant.quantize_tensor(np.ones((2, 2)), 4, 2), 5)


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("shape,g", [((64, 64), 64), ((128, 192), 64), ((200, 130), 64), ((257, 96), 64),
                                     ((96, 256), 128), ((1024, 512), 64)])
@pytest.mark.parametrize("pm", [4, 3, 2])
def test_pack_roundtrip_and_dequant_bit_exact(layout, shape, g, pm):
    rng = np.random.default_rng(shape[0] * 7 + shape[1] + pm)
    w = rng.standard_normal(shape)
    ref = oq.quantize(w, pm, g)
    qt = quant.quantize_tensor(w, pm, g)
    pk = qt.packed(layout)
    planes = torch.empty_like(qt.store.planes)
    mins = torch.empty_like(qt.mins)
    dels = torch.empty_like(qt.deltas)
    _capi.call("pmpd_unpack", pk.ref(), planes.data_ptr(), mins.data_ptr(), dels.data_ptr(),
               torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(host(planes), ref.planes)
    assert np.array_equal(host(mins), ref.mins) and np.array_equal(host(dels), ref.deltas)
    for p in range(1, pm + 1):
        got = host(quant.dequantize(qt, p, layout=layout))
        want = oq.dequantize(ref, p).astype(np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (layout, p)


def test_plane_prefix_memory_property():
    """Reading precision p touches exactly planes 0..p-1: corrupting planes >= p leaves dequant(p) unchanged."""
    w = np.random.default_rng(3).standard_normal((128, 256))
    qt = quant.quantize_tensor(w, 4, 64)
    pk = qt.packed(_capi.LAYOUT_KN)
    base = {p: host(quant.dequantize(qt, p, layout=_capi.LAYOUT_KN)) for p in (1, 2, 3)}
    pb = pk.desc.plane_bytes
    for p in (3, 2, 1):
        pk.buf[p * pb: 4 * pb] = 0xA5
        assert np.array_equal(host(quant.dequantize(qt, p, layout=_capi.LAYOUT_KN)), base[p])


def test_file_round_trip_byte_identical(gold_quant):
    blob = gold_quant["file/bytes"].tobytes()
    tensors, meta = quant.parse_model(blob)
    assert quant.serialize_model(tensors, {k: v for k, v in meta.items()
                                           if k not in ("p_max", "group_size", "tensors")}) == blob
