"""NEXT-3 search logic (paper_2602_08190_b200/tune.py) on planted metric surfaces, and the C-ABI knobs (CPU)."""
import itertools
import math

import pytest

from paper_2602_08190_b200 import cdm, tune

P2 = lambda a, b: [1 << k for k in range(a, b + 1)]  # noqa: E731


def table3_spaces(warp=32):
    """PAPER.md Table 3: F.P. L 2^0..2^4, S warp..2^10, C = ceil(4/dtype.size) (int32: 1);
    G.P. L = numCUs (1 point), S warp..2^10, C 2^0..2^10; N.P. L = numCUs, S = warp, C 2^0..2^10."""
    S = [s for s in P2(0, 10) if s >= warp]
    return {"FP": {"S": S, "C": [math.ceil(4 / 4)], "L": P2(0, 4)},
            "GP": {"L": [148], "S": S, "C": P2(0, 10)},
            "NP": {"L": [148], "S": [warp], "C": P2(0, 10)}}


def test_brute_force_counts_match_table3():
    sp = table3_spaces()
    counts = {k: tune.brute_force(v, lambda c: 0.0)["evaluations"] for k, v in sp.items()}
    assert counts == {"FP": 5 * 6 * 1, "GP": 1 * 6 * 11, "NP": 1 * 1 * 11}  # "NVIDIA = 5x6x1, 1x6x11, 1x1x11"


def _unimodal(space, peak):
    """separable concave surface in log2 coordinates with its maximum at `peak`"""
    def f(cfg):
        return -sum((math.log2(cfg[d]) - math.log2(peak[d])) ** 2 for d in space)
    return f


@pytest.mark.parametrize("pattern", ["FP", "GP", "NP"])
def test_pruned_finds_the_brute_force_optimum_on_unimodal_surfaces(pattern):
    space = table3_spaces()[pattern]
    for peak_vals in itertools.product(*[v[:: max(1, len(v) // 3)] for v in space.values()]):
        peak = dict(zip(space.keys(), peak_vals))
        f = _unimodal(space, peak)
        bf, pr = tune.brute_force(space, f), tune.pruned(space, f)
        assert pr["best"] == bf["best"] == peak
        # cost: per free dimension, the points up to the peak plus the first decline
        bound = sum(min(len(v), v.index(peak[d]) + 2) for d, v in space.items() if len(v) > 1)
        assert pr["evaluations"] <= bound < bf["evaluations"] or bf["evaluations"] <= 11
        assert bf["best_metric"] >= max(m for _, m in pr["trace"])


def test_pruned_order_and_fixed_dimensions_cost_nothing():
    space = {"S": [32, 64, 128, 256], "C": [1], "L": [1, 2, 4, 8, 16]}
    calls = []
    f = lambda c: (calls.append(dict(c)), -abs(c["S"] - 128) - abs(c["L"] - 4))[1]  # noqa: E731
    r = tune.pruned(space, f, order=["S", "C", "L"])
    assert r["best"] == {"S": 128, "C": 1, "L": 4}
    assert r["evaluations"] == len(calls) == 4 + 3  # S: 32,64,128,256(decline); L: 2,4,8(decline); memoised
    assert all(c["C"] == 1 for c in calls)


def test_pruned_stops_at_first_decline_even_if_not_global():
    space = {"C": [1, 2, 4, 8, 16]}
    vals = {1: 1.0, 2: 3.0, 4: 2.0, 8: 9.0, 16: 0.0}  # bimodal: the pruned search keeps the first peak
    r = tune.pruned(space, lambda c: vals[c["C"]])
    assert r["best"] == {"C": 2} and r["evaluations"] == 3
    assert tune.brute_force(space, lambda c: vals[c["C"]])["best"] == {"C": 8}


def test_cabi_tuning_knobs():
    assert cdm.tune_get("lz4_lanes") in (1, 2, 4, 8, 16, 32)
    assert cdm.tune_get("scan_mode") in (0, 1, 2)
    old = cdm.tune_get("fp_ctas_per_sm")
    cdm.tune_set("fp_ctas_per_sm", 3)
    assert cdm.tune_get("fp_ctas_per_sm") == 3
    cdm.tune_set("fp_ctas_per_sm", old)
    lanes = cdm.tune_get("lz4_lanes")
    cdm.tune_set("lz4_lanes", 4)
    assert cdm.tune_get("lz4_lanes") == 4
    cdm.tune_set("lz4_lanes", lanes)
    mode = cdm.tune_get("scan_mode")
    cdm.tune_set("scan_mode", 1)
    assert cdm.tune_get("scan_mode") == 1
    cdm.tune_set("scan_mode", mode)
    gp = cdm.tune_get("gp_ctas_per_sm")
    cdm.tune_set("gp_ctas_per_sm", 2)
    assert cdm.tune_get("gp_ctas_per_sm") == 2
    cdm.tune_set("gp_ctas_per_sm", gp)
    assert cdm.tune_get("lz4_split") in (0, 1) and cdm.tune_get("lz4_split_g") in (0, 1, 2, 4, 8)
    assert cdm.tune_get("lz4_spec") == 1
    for knob, v in (("lz4_split", 0), ("lz4_split_g", 4), ("lz4_spec", 2), ("lz4_spec", 0)):
        old = cdm.tune_get(knob)
        cdm.tune_set(knob, v)
        assert cdm.tune_get(knob) == v
        cdm.tune_set(knob, old)
    for knob, v in (("fp_ctas_per_sm", 17), ("lz4_lanes", 5), ("scan_mode", 3), ("gp_ctas_per_sm", 9), ("lz4_split", 2),
                     ("lz4_split_g", 16), ("lz4_spec", 3), ("nope", 1)):
        with pytest.raises(cdm.CdmError):
            cdm.tune_set(knob, v)
