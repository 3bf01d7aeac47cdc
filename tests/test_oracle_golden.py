"""Pin the CPU oracle (oracle/) against golden vectors produced by the real reference."""
import struct

import numpy as np
import pytest

from oracle import learnsched as olearn
from oracle import model as om
from oracle import quant as oq
from oracle import schedule as osched
from oracle.errors import ConfigError, ContractViolation, FormatError, InputError
from oracle.rng import named_rng
from pmpd_testutil import rel_l2


def test_quantize_codes_scales_planes_bit_exact(gold_quant):
    for name in gold_quant["names"]:
        r, c, g, pm = (int(v) for v in gold_quant[f"{name}/meta"])
        qt = oq.quantize(gold_quant[f"{name}/w"], pm, g)
        assert np.array_equal(qt.mins.view(np.uint32), gold_quant[f"{name}/mins"].view(np.uint32)), name
        assert np.array_equal(qt.deltas.view(np.uint32), gold_quant[f"{name}/deltas"].view(np.uint32)), name
        assert np.array_equal(qt.planes, gold_quant[f"{name}/planes"]), name
        assert np.array_equal(qt.codes, gold_quant[f"{name}/codes"]), name
        for p in range(1, pm + 1):
            assert np.array_equal(oq.prefix_codes(qt.planes, r, c, pm, p), gold_quant[f"{name}/prefix{p}"])
            d = oq.dequantize(qt, p)
            assert np.array_equal(d.view(np.uint64), gold_quant[f"{name}/deq{p}"].view(np.uint64)), (name, p)
            assert np.array_equal(oq.error_bound(qt, p), gold_quant[f"{name}/bound{p}"])


def test_known_answers():
    qt = oq.quantize(np.array([[0.0, 1.0, 2.0, 3.0]]), 2, 4)
    assert qt.mins[0, 0] == 0.0 and qt.deltas[0, 0] == 1.0 and qt.codes.tolist() == [[0, 1, 2, 3]]
    assert oq.dequantize(qt, 2).tolist() == [[0.0, 1.0, 2.0, 3.0]]
    assert oq.dequantize(qt, 1).tolist() == [[1.0, 1.0, 3.0, 3.0]]  # bucket centres
    assert oq.quantize(np.array([[0.0, 0.5, 1.0]]), 1, 4).codes.tolist() == [[0, 1, 1]]
    planes = oq.pack_planes(np.array([[0b10, 0b01]], dtype=np.uint8), 2)
    assert oq.prefix_codes(planes, 1, 2, 2, 1).tolist() == [[1, 0]]
    assert oq.prefix_codes(planes, 1, 2, 2, 2).tolist() == [[2, 1]]
    qt = oq.quantize(np.random.default_rng(4).normal(size=(13, 21)), 3, 8)
    assert qt.planes.nbytes == 3 * ((13 * 21 + 7) // 8)


def test_random_nesting_property():
    rng = np.random.default_rng(2)
    for _ in range(60):
        pm = int(rng.integers(1, 9))
        codes = rng.integers(0, 1 << pm, (int(rng.integers(1, 20)), int(rng.integers(1, 20)))).astype(np.uint8)
        pl = oq.pack_planes(codes, pm)
        for p in range(1, pm + 1):
            assert np.array_equal(oq.prefix_codes(pl, *codes.shape, pm, p), codes >> (pm - p))


def test_quantize_errors():
    with pytest.raises(InputError):
        oq.quantize(np.array([[np.nan, 1.0]]), 4, 2)
    with pytest.raises(ConfigError):
        oq.quantize(np.ones((2, 2)), 9, 2)
    with pytest.raises(ConfigError):
        oq.quantize(np.ones((2, 2)), 4, 0)
    qt = oq.quantize(np.ones((2, 2)), 4, 2)
    with pytest.raises(ConfigError):
        oq.dequantize(qt, 5)
    with pytest.raises(ConfigError):
        oq.check_precisions((2, 3))


def test_file_format_bytes(gold_quant):
    a = oq.quantize(np.random.default_rng(7).normal(size=(5, 12)), 3, 4)
    b = oq.quantize(np.random.default_rng(8).normal(size=(8, 8)), 3, 4)
    blob = oq.serialize({"a": a, "b": b}, {"note": "fixture"})
    assert blob == gold_quant["file/bytes"].tobytes()
    back, meta = oq.parse(blob)
    assert meta["note"] == "fixture" and list(back) == ["a", "b"]
    assert np.array_equal(back["b"].planes, b.planes)
    bad = bytearray(blob)
    bad[0] ^= 0xFF
    with pytest.raises(FormatError, match="bad magic"):
        oq.parse(bytes(bad))
    with pytest.raises(FormatError, match="tensor 'b'"):
        oq.parse(blob[:-10])
    with pytest.raises(FormatError, match="trailing"):
        oq.parse(blob + b"\x00")
    bad = bytearray(blob)
    bad[4:8] = struct.pack("<I", 99)
    with pytest.raises(FormatError, match="version"):
        oq.parse(bytes(bad))


def test_layer_reference_outputs(gold_layer):
    for tag in ("nk256", "nk512x1024"):
        N, K, seed = (int(v) for v in gold_layer[f"{tag}/shape"])
        W = (0.02 * named_rng(seed, "W").standard_normal((N, K))).astype(np.float16)
        x = named_rng(seed, "x").standard_normal((1, K)).astype(np.float16)
        qt = oq.quantize(W.astype(np.float32), 4, 64)
        assert np.array_equal(qt.planes, gold_layer[f"{tag}/planes"])
        for p in (4, 3, 2):
            y = x.astype(np.float64) @ oq.dequantize(qt, p).T
            assert rel_l2(y, gold_layer[f"{tag}/y{p}"]) < 1e-13


def _small_model():
    cfg = om.Config(n_layers=2, n_heads=2, d_model=64, d_ff=128, max_context=128)
    return om.Model.from_random(cfg, (4, 3, 2), seed=7)


def test_model_weights_and_forward(gold_model):
    import hashlib

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    m = _small_model()
    for name, t in m.tensors.items():
        assert sha(t.planes) + sha(t.mins) + sha(t.deltas) == str(gold_model[f"small/sha/{name}"]), name
    toks = [int(t) for t in gold_model["small/tokens"]]
    for p in (2, 3, 4, 16):
        assert rel_l2(om.forward_full(m, p, toks), gold_model[f"small/full{p}"]) < 1e-12


def test_incremental_decode_matches_reference(gold_model):
    m = _small_model()
    prompt = [int(t) for t in gold_model["small/prompt"]]
    lg, cache = om.prefill(m, 4, prompt)
    assert rel_l2(lg, gold_model["small/prefill4"]) < 1e-12
    sched = osched.Schedule((4, 3, 2), 4, {4: 0, 3: 4, 2: 9}, 24)
    tok = int(np.argmax(lg))
    for i, ref in enumerate(gold_model["small/decode_logits"]):
        lg, cache = om.decode_step(m, sched.precision_at(i), tok, cache)
        assert rel_l2(lg, ref) < 1e-12
        tok = int(np.argmax(lg))


def test_toy_model_criterion6(gold_model):
    cfg = om.Config(n_layers=4, n_heads=4, d_model=128, d_ff=256, max_context=256)
    m = om.Model.from_random(cfg, (4, 3, 2), seed=11)
    toks = [int(t) for t in gold_model["toy/tokens"]]
    for p in (2, 3, 4, 16):
        assert rel_l2(om.forward_full(m, p, toks), gold_model[f"toy/full{p}"]) < 1e-12


def test_generation_traces(gold_model):
    m = _small_model()
    prompt = [int(t) for t in gold_model["small/prompt"]]
    runs = {
        "fixed4": (om.StaticSched.fixed(4), None, 10, prompt),
        "two_phase": (om.StaticSched(osched.Schedule.two_phase(3, 2, 3, 16, 4)), None, 8, prompt),
        "prog432": (om.StaticSched(osched.Schedule((4, 3, 2), 4, {4: 0, 3: 4, 2: 9}, 24)), -1, 24, prompt),
        "fp16": (om.StaticSched.fixed(16), None, 6, prompt),
        "prog432_64": (om.StaticSched(osched.Schedule((4, 3, 2), 4, {4: 0, 3: 8, 2: 24}, 64)), -1, 64, prompt),
    }
    net = olearn.Net.init(64, 64, 8, 5, 16, 3, 2, seed=0)
    runs["learned"] = (olearn.LearnedSched(net, 4), None, 12, list(b"A lantern in the window"))
    for k, (sch, eos, mx, pr) in runs.items():
        toks, precs, sched, term, _ = om.generate(m, pr, sch, eos_id=eos, max_new=mx)
        assert toks == gold_model[f"small/trace/{k}/tokens"].tolist(), k
        assert precs == gold_model[f"small/trace/{k}/precisions"].tolist(), k
        assert sorted(sched.switch_points.items()) == [tuple(r) for r in gold_model[f"small/trace/{k}/st"].tolist()]
        assert term == str(gold_model[f"small/trace/{k}/term"])


def test_generate_contracts():
    m = _small_model()
    with pytest.raises(ContractViolation):
        om.generate(m, [1, 2], om.StaticSched(osched.Schedule.two_phase(6, 2, 3, 16)), max_new=8)
    with pytest.raises(ContractViolation):
        om.generate(m, [1, 2], om.StaticSched(osched.Schedule((4, 3), 4, {4: 5, 3: 1}, 16)), max_new=8)
    with pytest.raises(InputError):
        om.generate(m, [1, 2], om.StaticSched(osched.Schedule.two_phase(3, 2, 2, 8)), max_new=9)
    with pytest.raises(InputError):
        om.prefill(m, 4, [])
    with pytest.raises(InputError):
        om.prefill(m, 4, [999])


def test_schedules(gold_sched):
    cases = {
        "a": ((3, 2), 3, {3: 0, 2: 3}, 5, 5),
        "b": ((3, 2), 3, {3: 0, 2: 0}, 4, 4),
        "c": ((3, 2), 3, {3: 0, 2: 4}, 4, 4),
        "cfg2": ((3, 2), 4, {3: 0, 2: 64}, 256, 256),
        "cfg3": ((4, 3, 2), 4, {4: 0, 3: 32, 2: 128}, 512, 512),
    }
    for k, (ps, pf, st, ol, n) in cases.items():
        s = osched.Schedule(ps, pf, st, ol)
        assert [s.precision_at(i) for i in range(n)] == gold_sched[f"{k}/pat"].tolist()
        assert osched.avg_bitwidth(s, n) == float(gold_sched[f"{k}/avg"])
    assert list(osched.grid_points(5, 512)) == gold_sched["grid5_512"].tolist()
    assert list(osched.grid_points(4, 9)) == gold_sched["grid4_9"].tolist()
    bad = osched.Schedule((4, 3), 4, {4: 3, 3: 1}, 8)
    assert bad.validate() == gold_sched["bad/violations"].tolist()
    w, sp = osched.weighted_latency({4: 12.0, 3: 9.0, 2: 7.0, 16: 97.0},
                                    osched.Schedule((4, 3, 2), 4, {4: 0, 3: 32, 2: 128}, 512), 512)
    assert [w, sp] == gold_sched["weighted"].tolist()


def test_learned_scheduler(gold_learn):
    net = olearn.Net.init(16, 16, 8, 5, 16, 3, 2, seed=3)
    for name in ("q", "w1", "b1", "w2", "b2"):
        assert np.array_equal(getattr(net, name), gold_learn[f"net/{name}"])
    for t in (1, 7, 40):
        K, V = gold_learn[f"T{t}/K"], gold_learn[f"T{t}/V"]
        assert np.allclose(olearn.pool(net, K, V), gold_learn[f"T{t}/pooled"], rtol=1e-13, atol=1e-15)
        assert np.allclose(olearn.class_logits(net, K, V), gold_learn[f"T{t}/logits"], rtol=1e-13, atol=1e-15)
        s = olearn.predict(net, K, V, 4)
        assert sorted(s.switch_points.items()) == [tuple(r) for r in gold_learn[f"T{t}/st"].tolist()]
    for lab in ("weights", "W", "x", "scheduler-init"):
        assert np.array_equal(named_rng(5, lab).standard_normal(4), gold_learn[f"rng/{lab}"])
