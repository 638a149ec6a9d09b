"""Known-answer and property tests of the kept control-plane API, restating
the reference's own suites (TST = reference ``pkg/tests``):
test_scheduler.py:28-283 and test_model_core.py:52-188.  They pin the same
numbers against OUR modules."""
import numpy as np
import pytest

from oracle.plan_oracle import budget_check, exhaustive_prefetch_select
from paper_2605_02189_b200.model_core import (
    CalibrationWarning, ClusterConfig, DegenerateSamples, EstimatorParams, NoKvHeadroom,
    Request, blocks_for_tokens, calibrate_estimator, capacity_blocks, estimate_decode_time,
    kv_footprint, per_batch_token_budget, system_token_capacity)
from paper_2605_02189_b200.scheduler import (
    EmptySystem, SchedulerState, batch_indices, commit_plan, detect_steady, initial_partition,
    prefetch_budget, residual_set, schedule_step, select_prefetch_steady, select_prefetch_warmup)


def roomy(n=2, h2d=80.0, kv=1):
    return ClusterConfig(n=n, mem_per_gpu=10**7, model_bytes=10**6, kv_bytes_per_token=kv,
                         h2d_bandwidth=h2d, d2h_bandwidth=1e9, cpu_kv_capacity=10**12,
                         block_size=1)


def paper_cfg(n=8, mem=32e9, model=140e9, kv=145000, **kw):
    args = dict(h2d_bandwidth=1e9, d2h_bandwidth=1e9, cpu_kv_capacity=int(1e12))
    args.update(kw)
    return ClusterConfig(n=n, mem_per_gpu=mem, model_bytes=model, kv_bytes_per_token=kv, **args)


def make_state(n, batches, lengths, pool, cfg, **kw):
    res = set().union(*batches) if batches else set()
    st = SchedulerState(n=n, batches=batches, lengths=dict(lengths), gpu_resident=res,
                        cpu_pool=set(pool), **kw)
    st.configure_blocks(cfg.block_size)
    return st


# TST test_scheduler.py:28-36
@pytest.mark.parametrize("t,n,want", [(0, 4, (0, 1, 3)), (5, 4, (1, 2, 0)), (7, 1, (0, 0, 0))])
def test_batch_indices(t, n, want):
    assert batch_indices(t, n) == want


# TST test_scheduler.py:40-69
def test_initial_partition_known_answer():
    reqs = [Request(0, 10, 1), Request(1, 9, 1), Request(2, 2, 1), Request(3, 1, 1)]
    b = initial_partition(reqs, 2)
    assert b == [{0, 3}, {1, 2}]


def test_initial_partition_sizes_and_cover():
    reqs = [Request(0, 1000, 1)] + [Request(i, 1, 1) for i in range(1, 8)]
    for n in (2, 3, 4):
        b = initial_partition(reqs, n)
        sizes = [len(x) for x in b]
        assert max(sizes) - min(sizes) <= 1
        assert set().union(*b) == set(range(8))
    assert initial_partition([], 3) == [set(), set(), set()]
    assert sorted(len(x) for x in initial_partition([Request(5, 7, 1)], 4)) == [0, 0, 0, 1]


# TST test_scheduler.py:72-83
def test_prefetch_budget():
    assert prefetch_budget(20e9, 0.05, 100000) == 10000
    assert prefetch_budget(20e9, 0.0, 100000) == 0
    assert prefetch_budget(0.0, 0.05, 100000) == 0
    assert prefetch_budget(float("inf"), 0.05, 100000) == 1 << 62


def test_residual_set():
    assert residual_set({"a", "b", "c"}, {"b", "c", "d"}) == {"b", "c"}
    assert residual_set({"a"}, set()) == set()


# TST test_scheduler.py:99-111
def test_warmup_selector():
    assert select_prefetch_warmup({0: 300, 1: 100, 2: 50, 3: 200}, 400) == {1, 2, 3}
    assert select_prefetch_warmup({0: 300, 1: 100}, 50) == set()
    assert select_prefetch_warmup({}, 400) == set()
    assert select_prefetch_warmup({4: 100, 1: 100, 2: 100}, 200) == {1, 2}


# TST test_scheduler.py:117-150
P1 = EstimatorParams(alpha=1.0, beta=0.01, delta=0.0)


def test_steady_selector_known_answer():
    pool = {0: 100, 1: 200, 2: 300, 3: 50}
    assert select_prefetch_steady(pool, 400, 5.0, P1, saturation_theta=0.9) == {0, 2}
    assert select_prefetch_steady({}, 400, 5.0, P1) == set()
    assert select_prefetch_steady({0: 10}, 0, 5.0, P1) == set()
    got = select_prefetch_steady(pool, 400, -1.0, P1, saturation_theta=0.9)
    assert sum(pool[r] for r in got) >= 360
    best, err = exhaustive_prefetch_select(pool, 400, 5.0, 1.0, 0.01, 0.9)
    assert best == frozenset({0, 2}) and err == pytest.approx(1.0)


def test_steady_selector_vs_exhaustive_oracle():
    params = EstimatorParams(alpha=1e-3, beta=1e-5, delta=0.0)
    rng = np.random.default_rng(9)
    hits = 0
    for _ in range(120):
        pool = {int(i): int(rng.integers(10, 500)) for i in range(int(rng.integers(1, 13)))}
        budget = int(rng.integers(50, 1200))
        gap = float(rng.uniform(0.0, 0.02))
        got = select_prefetch_steady(pool, budget, gap, params)
        total = sum(pool[r] for r in got)
        assert total <= budget
        _, best_err = exhaustive_prefetch_select(pool, budget, gap, params.alpha, params.beta)
        if abs(params.alpha * len(got) + params.beta * total - gap) <= 2 * best_err + params.alpha + 1e-12:
            hits += 1
    assert hits >= 108


# TST test_scheduler.py:153-170
def test_detect_steady():
    assert detect_steady([100, 150, 200, 210, 205, 208], 3, 0.05) is True
    assert detect_steady([100, 200], 3, 0.05) is False
    assert detect_steady([100, 200, 100], 3, 0.05) is False
    assert detect_steady([0, 0, 0], 3, 0.05) is False
    tail = [500, 510, 505]
    assert detect_steady([1, 2, 3] + tail, 3, 0.05) == detect_steady(tail, 3, 0.05)


# TST test_scheduler.py:181-283
def test_schedule_step_single_stage_and_empty():
    cfg = roomy(n=1)
    p = EstimatorParams(1e-3, 1e-5, 1e-3)
    plan = schedule_step(make_state(1, [{0, 1}], {0: 10, 1: 20}, set(), cfg), p, cfg)
    assert plan.prefetch_set == frozenset() and plan.evictions == ()
    assert plan.updated_next_batch == frozenset({0, 1})
    with pytest.raises(EmptySystem):
        schedule_step(make_state(2, [set(), set()], {}, set(), roomy()), p, roomy())


def test_schedule_step_warmup_feedback():
    cfg = roomy(n=2, h2d=100.0)
    p = EstimatorParams(0.01, 0.001, 0.0)
    lengths = {0: 100, 1: 100, **{i: 1 for i in range(100, 160)}}
    st = make_state(2, [{0}, {1}], lengths, set(range(100, 160)), cfg)
    sizes = []
    for _ in range(3):
        plan = schedule_step(st, p, cfg)
        assert not plan.steady
        sizes.append(len(plan.prefetch_set))
        commit_plan(st, plan, cfg)
    assert sizes == sorted(sizes) and sizes[-1] > sizes[0]


def test_schedule_step_steady_example():
    cfg = roomy(n=2, h2d=80.0)
    lengths = {10: 400, 0: 100, 1: 200, 2: 300, 3: 50}
    st = make_state(2, [{10}, set()], lengths, {0, 1, 2, 3}, cfg, steady=True)
    plan = schedule_step(st, P1, cfg)
    assert plan.predicted_exec_seconds == pytest.approx(5.0)
    assert plan.prefetch_budget_tokens == 400
    assert plan.prefetch_set == frozenset({0, 2}) == plan.updated_next_batch


def test_schedule_step_feasible_disjoint_and_safe():
    cfg = ClusterConfig(n=3, mem_per_gpu=4000, model_bytes=3000, kv_bytes_per_token=1,
                        h2d_bandwidth=50.0, d2h_bandwidth=1e9, cpu_kv_capacity=10**9,
                        block_size=4)
    p = EstimatorParams(0.05, 0.01, 0.01)
    rng = np.random.default_rng(21)
    lengths = {i: int(rng.integers(5, 40)) for i in range(40)}
    st = make_state(3, [{0, 1}, {2, 3}, {4, 5}], lengths, set(range(6, 40)), cfg)
    for _ in range(60):
        plan = schedule_step(st, p, cfg)
        assert sum(st.lengths[r] for r in plan.prefetch_set) <= plan.prefetch_budget_tokens
        for v in plan.evictions:
            assert v not in plan.exec_batch and v not in plan.residual
        commit_plan(st, plan, cfg)
        seen = set()
        for b in st.batches:
            assert not (b & seen)
            seen |= b
        assert seen <= st.gpu_resident and not (st.cpu_pool & st.gpu_resident)
        for rid in sorted(plan.exec_batch):
            st.bump_generated(rid)
    with pytest.raises(ValueError):
        commit_plan(st, plan, cfg)


# TST test_model_core.py:52-188
def test_estimator_and_budgets():
    assert estimate_decode_time(EstimatorParams(1e-4, 1e-6, 5e-3), 32, 10000) == pytest.approx(0.0182)
    cfg = paper_cfg()
    assert per_batch_token_budget(cfg) == 100000
    assert system_token_capacity(cfg) == 800000
    assert capacity_blocks(cfg) == 800000 // 16
    assert budget_check(8, int(32e9), int(140e9), 145000) == (800000, 100000)
    with pytest.raises(NoKvHeadroom):
        per_batch_token_budget(paper_cfg(n=4, mem=10**9, model=4 * 10**9, kv=1000))
    assert kv_footprint(524288, 253680) == 133001379840
    assert [blocks_for_tokens(x, 16) for x in (0, 1, 16, 17)] == [0, 1, 1, 2]
    with pytest.raises(ValueError):
        paper_cfg(n=2, mem=10**9, model=3 * 10**9)


def test_calibration():
    true = (2e-4, 5e-7, 4e-3)
    bs = np.repeat([1, 2, 4, 8, 16, 32, 64, 128, 192, 256], 20)
    ls = np.tile(np.linspace(0, 200000, 20).astype(int), 10)
    y = true[0] * bs + true[1] * ls + true[2]
    fit = calibrate_estimator(list(zip(bs, ls, y)))
    assert (fit.alpha, fit.beta, fit.delta) == pytest.approx(true, rel=1e-9)
    with pytest.raises(DegenerateSamples):
        calibrate_estimator([(8, 800, 0.01), (8, 800, 0.011), (8, 800, 0.009)])
    rows = [(b, l, 0.01 - 1e-4 * b + 1e-6 * l) for b in (1, 5, 9) for l in (100, 5000, 20000)]
    with pytest.warns(CalibrationWarning):
        assert calibrate_estimator(rows).alpha == 0.0
