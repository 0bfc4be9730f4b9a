"""Johnson's rule oracle (Sec. 3.3) pinned by the paper's two-block example and brute force."""
import numpy as np

from oracle import johnson_order, flow_shop_makespan, brute_force_best


def test_paper_example(golden):
    j = golden("spec_examples.json")["johnson"]
    jobs = [tuple(x) for x in j["jobs"]]
    assert johnson_order(jobs) == j["order"]  # "initiating the pipeline with data B followed by data A"
    assert flow_shop_makespan(jobs, [1, 0]) == j["makespan_best"]
    assert flow_shop_makespan(jobs, [0, 1]) == j["makespan_other"]


def test_single_job_and_zero_decode():
    assert flow_shop_makespan([(3.0, 2.0)], [0]) == 5.0
    jobs = [(1.0, 0.0), (2.0, 0.0), (4.0, 0.0)]
    assert flow_shop_makespan(jobs, johnson_order(jobs)) == 7.0


def test_brute_force_optimality():
    rng = np.random.default_rng(11)
    for trial in range(200):
        n = int(rng.integers(1, 9))
        jobs = [(float(rng.integers(0, 20)), float(rng.integers(0, 20))) for _ in range(n)]
        assert flow_shop_makespan(jobs, johnson_order(jobs)) == brute_force_best(jobs)


def test_ties_by_id():
    jobs = [(2.0, 2.0)] * 5
    assert johnson_order(jobs) == [0, 1, 2, 3, 4]
