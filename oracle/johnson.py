"""Johnson's rule and the two-machine flow-shop simulator -- TEST INFRASTRUCTURE (oracle).

PAPER.md:283-287 (Sec. 3.3 Pipelining Layer): order CPU->GPU transfers so that "the maximum
concurrency between the data movement and decompression phases" is reached, using Johnson's
algorithm [johnson1954optimal].  Machine 1 = the H2D link, machine 2 = the decode engine.
Rule (textbook Johnson 1954): jobs with t <= d first, ascending t; then the rest, descending d;
ties by job id (reading R21).  Pinned by the Fig. `pipeline` example (B before A) and by brute
force over all permutations for n <= 8 (tests/test_johnson.py).
"""
from __future__ import annotations

import itertools


def johnson_order(jobs: list[tuple[float, float]]) -> list[int]:
    first = sorted((i for i, (t, d) in enumerate(jobs) if t <= d), key=lambda i: (jobs[i][0], i))
    second = sorted((i for i, (t, d) in enumerate(jobs) if t > d), key=lambda i: (-jobs[i][1], i))
    return first + second


def flow_shop_makespan(jobs: list[tuple[float, float]], order: list[int]) -> float:
    """Two-machine flow shop: one copy engine, one decode engine; decode j starts after copy j and decode j-1."""
    t_copy = 0.0
    t_dec = 0.0
    for i in order:
        t, d = jobs[i]
        t_copy += t
        t_dec = max(t_dec, t_copy) + d
    return t_dec


def brute_force_best(jobs: list[tuple[float, float]]) -> float:
    return min(flow_shop_makespan(jobs, list(p)) for p in itertools.permutations(range(len(jobs))))
