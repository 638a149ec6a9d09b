"""The real-shape parity workloads (tests/real_shapes.py) exercise the
offload paths: the control plane alone (CPU) must evict, prefetch and run
micro-batches of >= 64 rows before the GPU test relies on it."""
import pytest

from paper_2605_02189_b200.control import DecodeControl
from real_shapes import CASES, build_case


@pytest.mark.parametrize("name", list(CASES))
def test_real_shape_plan_exercises_offload(name):
    spec, st, cfg, params, reqs, prompts = build_case(name)
    c = DecodeControl(st, cfg, params, reqs)
    ev = pf = 0
    rows = []
    while (w := c.step()) is not None:
        ev += len(w.evicted)
        pf += len(w.prefetch)
        rows.append(len(w.rows))
    assert c.metrics.completed_requests == len(reqs)
    assert ev > 50 and pf > 50 and max(rows) >= 64
    assert all(200 <= len(p) < 700 for p in prompts.values())
