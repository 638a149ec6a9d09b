"""The reference's OWN scheduler and model-core test files
(/root/reference/pkg/tests/test_scheduler.py, test_model_core.py) run
unchanged against this package imported as ``pipemax`` (tests/
pipemax_alias.py).  Skipped where the reference checkout is absent (the GPU
box); the committed golden streams cover the same ground there."""
import os
import subprocess
import sys

import pytest

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")), reason="no reference checkout")


def test_reference_scheduler_and_model_core_suites_pass_unchanged(tmp_path):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([HERE, ROOT]), PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "pipemax_alias", "-p", "no:cacheprovider",
           "--rootdir", str(tmp_path), "-c", os.devnull,
           os.path.join(REF, "tests", "test_scheduler.py"), os.path.join(REF, "tests", "test_model_core.py")]
    r = subprocess.run(cmd, env=env, cwd=tmp_path, capture_output=True, text=True, timeout=600)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
    print(tail.strip().splitlines()[-1])
