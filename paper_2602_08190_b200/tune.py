"""NEXT-3: offline launch-configuration search (Table 3).

Host logic only (no decode arithmetic).  A search space is an ordered dict {dimension: [candidate values,
ascending]}; `evaluate(config) -> metric` (higher is better) is supplied by the caller (tools/tune.py times a
device batch).  Two strategies, as in Table 3:
  brute_force  every point of the cross product ("B.F. Search");
  pruned       coordinate search exploiting the "hidden monotonicity in the performance distribution"
               (P:681): dimensions in the given order; along each, sweep the candidates ascending from the
               first while the metric improves, stop after the first decline, fix the best value, move on;
               a single-candidate dimension costs no evaluation of its own.
Repeated configurations are evaluated once (memoised), so `evaluations` counts distinct launches.
"""
from __future__ import annotations

import itertools
from typing import Callable


def _key(cfg: dict) -> tuple:
    return tuple(sorted(cfg.items()))


def brute_force(space: dict[str, list], evaluate: Callable[[dict], float]) -> dict:
    trace = []
    for vals in itertools.product(*space.values()):
        cfg = dict(zip(space.keys(), vals))
        trace.append((cfg, float(evaluate(cfg))))
    best_cfg, best = max(trace, key=lambda t: t[1])
    return {"strategy": "brute_force", "best": best_cfg, "best_metric": best, "evaluations": len(trace),
            "trace": trace}


def pruned(space: dict[str, list], evaluate: Callable[[dict], float], order: list[str] | None = None) -> dict:
    order = list(order or space.keys())
    cur = {k: v[0] for k, v in space.items()}
    seen: dict[tuple, float] = {}
    trace = []

    def ev(cfg):
        k = _key(cfg)
        if k not in seen:
            seen[k] = float(evaluate(dict(cfg)))
            trace.append((dict(cfg), seen[k]))
        return seen[k]

    for dim in order:
        cands = space[dim]
        if len(cands) == 1:
            continue
        best_v, best_m = cands[0], ev({**cur, dim: cands[0]})
        for v in cands[1:]:
            m = ev({**cur, dim: v})
            if m > best_m:
                best_v, best_m = v, m
            else:
                break  # first decline: the distribution is taken as unimodal along this dimension
        cur[dim] = best_v
    best_cfg = dict(cur)
    return {"strategy": "pruned", "best": best_cfg, "best_metric": seen.get(_key(best_cfg), ev(best_cfg)),
            "evaluations": len(trace), "trace": trace}
