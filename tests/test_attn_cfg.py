"""Host logic of the attention launch-configuration choice (ops.choose_attn_cfg):
the cost model over the work list's own snake assignment picks 8 warps x 3
stages for the C3 stage shape and 12 x 2 for C2 / C4 (the measured winners),
and PM_ATTN_CFG overrides it.  Worker counts are those of a 148-SM B200
(12 x 2: 1776 warps, 8 x 3: 1184), stubbed so this runs without a GPU."""
import pytest

from paper_2605_02189_b200 import _C, ops

WARPS = {1: 148 * 12, 2: 148 * 8}


class _Lib:
    """Only the worker-count query the cost model makes (no libpmb200.so needed)."""

    def pm_attn_workers_cfg(self, hd, cfg):
        return WARPS[cfg]


@pytest.fixture
def b200_workers(monkeypatch):
    monkeypatch.setattr(_C, "lib", lambda: _Lib())
    monkeypatch.delenv("PM_ATTN_CFG", raising=False)


@pytest.mark.parametrize("name,m_cap,max_blocks,want", [
    ("C2 qwen3-8b, 128 rows, 512+512", 128, 65, 1),
    ("C3 qwen3-32b stage, 64 rows, ~1050", 64, 67, 2),
    ("C4 llama3-70b stage, 32 rows, ~1050", 32, 67, 1),
])
def test_cost_model_picks_measured_winner(b200_workers, name, m_cap, max_blocks, want):
    assert ops.choose_attn_cfg(m_cap, 8, 128, max_blocks, 12) == want, name


def test_engine_passes_rows_per_step():
    """The engine sizes the choice by a micro-batch's rows (requests / micro-
    batches), not by the workspace capacity (all requests)."""
    from paper_2605_02189_b200.engine import attn_rows_hint
    assert attn_rows_hint(512, 8) == 64 and attn_rows_hint(256, 2) == 128 and attn_rows_hint(256, 8) == 32
    assert attn_rows_hint(10, 3) == 4


def test_env_override(b200_workers, monkeypatch):
    monkeypatch.setenv("PM_ATTN_CFG", "0")
    assert ops.choose_attn_cfg(64, 8, 128, 67, 12) == 0
