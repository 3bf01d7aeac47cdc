"""Offline schedule search on the device against golden output of the
reference's own solve_static / generate_labels (tests/golden/make_golden_search.py): the same
candidate qualities, the same selected schedule, the same labels and scores."""
import json

import numpy as np
import pytest

from paper_2410_13461_b200 import quant, search, tinylm
from paper_2410_13461_b200.schedule import QualityTarget, SwitchGrid
from pmpd_testutil import load_golden

pytestmark = pytest.mark.gpu

PROMPTS = [b"The river finds its way", b"Old maps mark the mountain", b"A lantern in the window",
           b"Salt and iron in the wind", b"Every bridge has two banks", b"Quiet rooms keep old clocks"]


@pytest.fixture(scope="module")
def small():
    cfg = tinylm.ModelConfig(n_layers=2, n_heads=2, d_model=64, d_ff=128, max_context=128)
    return tinylm.ModelVariants.from_random(cfg, quant.PrecisionSet((4, 3, 2)), seed=7)


@pytest.mark.parametrize("tag,ps,q,tol", [("s432", (4, 3, 2), 0.25, 0.05), ("s32", (3, 2), 0.2, 0.0)])
def test_solve_static_matches_reference(small, tag, ps, q, tol):
    gold = load_golden("search.npz")
    details = []
    best = search.solve_static(small, [list(p) for p in PROMPTS], QualityTarget(q, tol), SwitchGrid(5, 16),
                               precisions=quant.PrecisionSet(ps), p_prefill=4, details_out=details)
    want = json.loads(str(gold[f"{tag}/details"]))
    assert [d["st"] for d in details] == [d["st"] for d in want], (details, want)
    got_q, want_q = np.array([d["quality"] for d in details]), np.array([d["quality"] for d in want])
    # greedy decoding of a random-init toy model has near-ties: a candidate's mean Rouge-L may move
    # by one token of one prompt (1/96 here) where an fp16/fp32 logit flips a tie; the rest match
    assert np.abs(got_q - want_q).max() <= 1.0 / 48 + 1e-12, (got_q, want_q)
    assert (np.abs(got_q - want_q) < 1e-12).mean() >= 0.75, (got_q, want_q)
    assert [d["feasible"] for d in details] == [d["feasible"] for d in want]
    assert json.dumps(best.to_json(), sort_keys=True) == str(gold[f"{tag}/best"])


def test_generate_labels_match_reference(small):
    gold = load_golden("search.npz")
    ex, skipped = search.generate_labels(small, [list(p) for p in PROMPTS], SwitchGrid(5, 8), 3, 2, p_prefill=4,
                                         seed=13)
    assert skipped == int(gold["labels/skipped"])
    assert [e.label for e in ex] == gold["labels/labels"].tolist()
    np.testing.assert_allclose([e.scores for e in ex], gold["labels/scores"], rtol=0, atol=1e-12)
    assert [e.prompt_len for e in ex] == gold["labels/prompt_len"].tolist()
    for i, e in enumerate(ex):  # features: the device cache holds f16 K/V (reference: f64)
        np.testing.assert_allclose(e.k, gold[f"labels/k{i}"], rtol=2e-2, atol=2e-2)
        np.testing.assert_allclose(e.v, gold[f"labels/v{i}"], rtol=2e-2, atol=2e-2)
