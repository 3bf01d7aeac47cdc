"""Host logic of the device offline search (no GPU): Rouge-L, switch-map enumeration, the
selection rule and the label rule, against the reference's known answers
(pkg/tests/test_metrics.py, test_schedule.py, test_learnsched.py:205-209)."""
from paper_2410_13461_b200 import search
from paper_2410_13461_b200.quant import PrecisionSet
from paper_2410_13461_b200.schedule import QualityTarget, SwitchGrid


def test_rouge_l_known_answers():
    assert search.lcs_len("ABCBDAB", "BDCABA") == 4
    r = search.rouge_l([1, 2, 3, 4], [1, 3, 4, 5, 6])
    assert (r.precision, r.recall) == (0.75, 0.6)
    assert abs(r.f1 - 2 * 0.75 * 0.6 / 1.35) < 1e-15
    assert search.rouge_l([], [1]).f1 == 0.0


def test_switch_maps_and_selection():
    maps = list(search.enumerate_switch_maps((4, 3, 2), (0, 8, 16)))
    assert len(maps) == 6 and all(m[4] == 0 and m[3] <= m[2] for m in maps)
    grid = SwitchGrid(3, 16)
    # quality falls with earlier low-precision switches: the cheapest feasible one is picked
    q = lambda s: 1.0 - 0.05 * (16 - s.switch_points[2]) / 8  # noqa: E731
    best = search.solve_static(None, None, QualityTarget(1.0, 0.06), grid, precisions=PrecisionSet((4, 3, 2)),
                               p_prefill=4, quality_fn=q)
    assert best.feasible and best.switch_points == {4: 0, 3: 0, 2: 8}
    none = search.solve_static(None, None, QualityTarget(2.0, 0.0), grid, precisions=PrecisionSet((4, 3, 2)),
                               p_prefill=4, quality_fn=q)
    assert not none.feasible and none.switch_points == {4: 0, 3: 16, 2: 16}


def test_label_rule_minimality():
    assert search.label_from_scores([0.9, 0.5, 0.6, 0.9]) == 0
    assert search.label_from_scores([0.1, 0.2, 0.3, 0.9]) == 3
    assert search.label_from_scores([0.1, 0.9, 0.95, 0.9]) == 1
