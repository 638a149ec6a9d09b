"""Independent checkers for the prefetch selectors and capacity formulas.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Restates the reference's
``pkg/src/pipemax/oracle.py``:
* ``exhaustive_prefetch_select`` follows :47-79 -- enumerate every subset,
  rank by (saturated >= theta*budget first, |modeled-gap|, size, ids);
* ``budget_check`` follows :95-111 -- exact rationals for (nM - W)/T.
"""
from fractions import Fraction
from itertools import combinations

ENUMERATION_CAP = 20


def exhaustive_prefetch_select(pool, budget, gap, alpha, beta, theta=0.9):
    if len(pool) > ENUMERATION_CAP:
        raise ValueError("pool too large for enumeration")
    ids = sorted(pool)

    def rank(subset, total):
        modeled = alpha * len(subset) + beta * total
        return (0 if total >= theta * budget else 1, abs(modeled - gap), len(subset), tuple(subset))

    best = rank((), 0)
    best_ids = ()
    for size in range(1, len(ids) + 1):
        for combo in combinations(ids, size):
            total = sum(pool[r] for r in combo)
            if total > budget:
                continue
            key = rank(combo, total)
            if key < best:
                best, best_ids = key, combo
    return frozenset(best_ids), best[1]


def budget_check(n, mem_per_gpu, model_bytes, kv_bytes_per_token):
    per_gpu_kv = Fraction(mem_per_gpu) - Fraction(model_bytes, n)
    per_gpu_tok = Fraction(kv_bytes_per_token, n)
    system = per_gpu_kv / per_gpu_tok
    return int(system), int(system / n)
