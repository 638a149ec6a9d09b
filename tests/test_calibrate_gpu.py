"""On-box estimator calibration (calibrate.py; REF model_core.py:148-182,
cli.py:311-327): measured decode iterations of the engine's own executors
grow with batch and prefix length, the affine fit reproduces them, and the
sample file is in the reference CLI's ``b,L,seconds`` format."""
import csv

import pytest

from paper_2605_02189_b200.calibrate import calibrate_on_device, write_samples_csv
from test_engine_gpu import build  # noqa: E402

pytestmark = pytest.mark.gpu


def test_calibrate_on_device(tmp_path):
    spec, eng, reqs, prompts = build(graphs=True)
    grid = [(16, 16 * 8), (16, 16 * 50), (24, 24 * 8), (24, 24 * 50), (8, 8 * 30)]   # per-row prefix < max_len
    params, samples, err = calibrate_on_device(eng, grid=grid, reps=5)
    assert len(samples) == len(grid)
    assert all(t > 0 for _, _, t in samples)
    t = {(b, L): s for b, L, s in samples}
    # more KV is not faster (at this tiny shape a step is ~0.1 ms of launch-bound
    # kernels, so repeated runs scatter by ~10 %)
    assert t[(24, 24 * 50)] >= t[(24, 24 * 8)] * 0.85
    assert params.delta > 0 and err < 0.5
    path = tmp_path / "samples.csv"
    write_samples_csv(str(path), samples)
    rows = [r for r in csv.reader(open(path))]
    assert rows[0] == ["b", "L", "seconds"]
    assert [(float(r[0]), float(r[1])) for r in rows[1:]] == [(float(b), float(L)) for b, L, _ in samples]
