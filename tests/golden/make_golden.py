"""Generate golden vectors from the REAL reference implementation.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    python tests/golden/make_golden.py

It imports ``pmpd`` from ``/root/reference/pkg/src`` (read-only) and writes
small ``.npz`` fixtures next to this script.  The fixtures pin both the CPU
oracle (``oracle/``) and, through it, the B200 product: quantization codes,
f32 scales and bit planes, dequantized values, forward logits of the
reference test models, greedy generation traces under static / fixed /
learned schedulers, scheduler pooling outputs and the PMPD v1 file bytes.
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    sys.path.insert(0, str(REF))
    from pmpd import learnsched, quant, schedule, tinylm, util  # noqa: E402

    # ---------------------------------------------------------------- quant
    q = {}
    kat = [
        ("grid", np.array([[0.0, 1.0, 2.0, 3.0]]), 2, 4),
        ("const", np.full((1, 3), 5.0), 3, 4),
        ("ties", np.array([[0.0, 0.5, 1.0]]), 1, 4),
    ]
    rng = np.random.default_rng(20241017)
    for i, (r, c, g, pm) in enumerate([(4, 10, 4, 4), (13, 21, 8, 3), (7, 64, 64, 4), (64, 129, 64, 4),
                                       (33, 200, 64, 4), (16, 256, 128, 4), (5, 70, 7, 5), (9, 40, 40, 8)]):
        kat.append((f"rand{i}", rng.normal(0, 1, (r, c)), pm, g))
    names = []
    for name, w, pm, g in kat:
        qt = quant.quantize_tensor(w, pm, g)
        names.append(name)
        q[f"{name}/w"] = w
        q[f"{name}/meta"] = np.array([qt.rows, qt.cols, g, pm])
        q[f"{name}/mins"] = qt.mins
        q[f"{name}/deltas"] = qt.deltas
        q[f"{name}/planes"] = qt.store.planes
        q[f"{name}/codes"] = qt.codes
        for p in range(1, pm + 1):
            q[f"{name}/deq{p}"] = quant.dequantize(qt, p)
            q[f"{name}/prefix{p}"] = quant.unpack_prefix(qt.store, p)
            q[f"{name}/bound{p}"] = quant.max_reconstruction_error_bound(qt, p)
    q["names"] = np.array(names)
    # PMPD v1 file bytes for two tensors
    t_a = quant.quantize_tensor(np.random.default_rng(7).normal(size=(5, 12)), 3, 4)
    t_b = quant.quantize_tensor(np.random.default_rng(8).normal(size=(8, 8)), 3, 4)
    blob = quant.serialize_model({"a": t_a, "b": t_b}, {"note": "fixture"})
    q["file/bytes"] = np.frombuffer(blob, dtype=np.uint8)
    np.savez_compressed(OUT / "quant.npz", **q)

    # ----------------------------------------------- config-1 style layer (reduced size)
    lay = {}
    for tag, (N, K, seed) in {"nk256": (256, 256, 1234), "nk512x1024": (512, 1024, 99)}.items():
        W = (0.02 * util.named_rng(seed, "W").standard_normal((N, K))).astype(np.float16)
        x = util.named_rng(seed, "x").standard_normal((1, K)).astype(np.float16)
        qt = quant.quantize_tensor(W.astype(np.float32), 4, 64)
        lay[f"{tag}/shape"] = np.array([N, K, seed])
        lay[f"{tag}/planes_sha"] = np.array(sha(qt.store.planes))
        lay[f"{tag}/mins"] = qt.mins
        lay[f"{tag}/deltas"] = qt.deltas
        lay[f"{tag}/planes"] = qt.store.planes
        for p in (4, 3, 2):
            lay[f"{tag}/y{p}"] = x.astype(np.float64) @ quant.dequantize(qt, p).T
    np.savez_compressed(OUT / "layer.npz", **lay)

    # ---------------------------------------------------------------- model
    mdl = {}
    prompt = list(b"The river finds its way")
    small_cfg = tinylm.ModelConfig(n_layers=2, n_heads=2, d_model=64, d_ff=128, max_context=128)
    small = tinylm.ModelVariants.from_random(small_cfg, quant.PrecisionSet((4, 3, 2)), seed=7,
                                             dequant_budget=1 << 30)
    mdl["small/prompt"] = np.array(prompt)
    for name, t in small.tensors.items():
        mdl[f"small/sha/{name}"] = np.array(sha(t.store.planes) + sha(t.mins) + sha(t.deltas))
    toks = prompt + [10, 200, 33]
    mdl["small/tokens"] = np.array(toks)
    for p in (2, 3, 4, 16):
        mdl[f"small/full{p}"] = tinylm.forward_full(small, p, toks)
    # greedy traces
    traces = {
        "fixed4": (tinylm.generate(small, prompt, schedule.FixedScheduler(4), max_new=10), None),
        "two_phase": (tinylm.generate(small, prompt, schedule.StaticScheduler(
            schedule.PrecisionSchedule.two_phase(3, 2, 3, 16, p_prefill=4)), max_new=8), None),
        "prog432": (tinylm.generate(small, prompt, schedule.StaticScheduler(
            schedule.PrecisionSchedule(quant.PrecisionSet((4, 3, 2)), 4, {4: 0, 3: 4, 2: 9}, 24)),
            eos_id=-1, max_new=24), None),
        "fp16": (tinylm.generate(small, prompt, schedule.FixedScheduler(16), max_new=6), None),
        # north-star criterion: greedy ids identical over the first 64 tokens (4->3->2 switching)
        "prog432_64": (tinylm.generate(small, prompt, schedule.StaticScheduler(
            schedule.PrecisionSchedule(quant.PrecisionSet((4, 3, 2)), 4, {4: 0, 3: 8, 2: 24}, 64)),
            eos_id=-1, max_new=64), None),
    }
    net = learnsched.SchedulerNet.init(64, 64, 8, schedule.SwitchGrid(5, 16), 3, 2, seed=0)
    traces["learned"] = (tinylm.generate(small, list(b"A lantern in the window"),
                                         learnsched.LearnedScheduler(net, p_prefill=4), max_new=12), None)
    for k, (tr, _) in traces.items():
        mdl[f"small/trace/{k}/tokens"] = np.array(tr.output_tokens)
        mdl[f"small/trace/{k}/precisions"] = np.array(tr.precisions)
        mdl[f"small/trace/{k}/st"] = np.array(sorted(tr.schedule.switch_points.items()))
        mdl[f"small/trace/{k}/term"] = np.array(tr.termination)
    # prefill logits and per-step decode logits for the progressive schedule
    lg, cache = tinylm.prefill(small, 4, prompt)
    mdl["small/prefill4"] = lg
    step = []
    tok = int(np.argmax(lg))
    sched = schedule.PrecisionSchedule(quant.PrecisionSet((4, 3, 2)), 4, {4: 0, 3: 4, 2: 9}, 24)
    for i in range(12):
        lg, cache = tinylm.decode_step(small, sched.precision_at(i), tok, cache)
        step.append(lg)
        tok = int(np.argmax(lg))
    mdl["small/decode_logits"] = np.array(step)
    # acceptance criterion 6 model
    toy_cfg = tinylm.ModelConfig(n_layers=4, n_heads=4, d_model=128, d_ff=256, max_context=256)
    toy = tinylm.ModelVariants.from_random(toy_cfg, quant.PrecisionSet((4, 3, 2)), seed=11,
                                           dequant_budget=1 << 30)
    ttoks = list(b"Old maps mark the mountain") + [256, 17, 99]
    mdl["toy/tokens"] = np.array(ttoks)
    for p in (2, 3, 4, 16):
        mdl[f"toy/full{p}"] = tinylm.forward_full(toy, p, ttoks)
    np.savez_compressed(OUT / "model.npz", **mdl)

    # ------------------------------------------------------------ schedules
    sc = {}
    cases = {
        "a": ((3, 2), 3, {3: 0, 2: 3}, 5, 5),
        "b": ((3, 2), 3, {3: 0, 2: 0}, 4, 4),
        "c": ((3, 2), 3, {3: 0, 2: 4}, 4, 4),
        "cfg2": ((3, 2), 4, {3: 0, 2: 64}, 256, 256),
        "cfg3": ((4, 3, 2), 4, {4: 0, 3: 32, 2: 128}, 512, 512),
    }
    for k, (ps, pf, st, ol, n) in cases.items():
        s = schedule.PrecisionSchedule(ps, pf, st, ol)
        sc[f"{k}/pat"] = np.array([s.precision_at(i) for i in range(n)])
        sc[f"{k}/avg"] = np.array(schedule.avg_bitwidth(s, n))
    sc["grid5_512"] = np.array(schedule.SwitchGrid(5, 512).points)
    sc["grid4_9"] = np.array(schedule.SwitchGrid(4, 9).points)
    bad = schedule.PrecisionSchedule(quant.PrecisionSet((4, 3)), 4, {4: 3, 3: 1}, 8)
    sc["bad/violations"] = np.array(bad.validate())
    from pmpd.perf import weighted_gpu_latency
    w, sp = weighted_gpu_latency({4: 12.0, 3: 9.0, 2: 7.0, 16: 97.0},
                                 schedule.PrecisionSchedule((4, 3, 2), 4, {4: 0, 3: 32, 2: 128}, 512), 512)
    sc["weighted"] = np.array([w, sp])
    np.savez_compressed(OUT / "schedule.npz", **sc)

    # -------------------------------------------------------- learned scheduler
    ls = {}
    net = learnsched.SchedulerNet.init(16, 16, 8, schedule.SwitchGrid(5, 16), 3, 2, seed=3)
    r = np.random.default_rng(77)
    for t in (1, 7, 40):
        K, V = r.normal(size=(t, 16)), r.normal(size=(t, 16))
        ls[f"T{t}/K"], ls[f"T{t}/V"] = K, V
        ls[f"T{t}/pooled"] = learnsched.pool_kv(net, K, V)
        ls[f"T{t}/logits"] = learnsched.class_logits(net, K, V)

        class C:
            def layer_kv(self, layer, K=K, V=V):
                return K, V
        s = learnsched.predict_schedule(net, C(), 4)
        ls[f"T{t}/st"] = np.array(sorted(s.switch_points.items()))
    for name, a in net.params().items():
        ls[f"net/{name}"] = a
    rngs = {lab: util.named_rng(5, lab).standard_normal(4) for lab in ("weights", "W", "x", "scheduler-init")}
    for lab, v in rngs.items():
        ls[f"rng/{lab}"] = v
    np.savez_compressed(OUT / "learnsched.npz", **ls)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
