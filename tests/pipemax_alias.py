"""pytest plugin: import THIS package under the reference's name ``pipemax``
so the reference's own test files run unchanged against it
(tests/test_reference_suites.py).  ``pipemax.scheduler`` and
``pipemax.model_core`` are ours; ``pipemax.oracle`` -- the checker those
tests compare against -- is the reference's own oracle module, loaded from
the checkout (test infrastructure, never on the product path)."""
import importlib.util
import os
import sys

REF_SRC = os.environ.get("PIPEMAX_REF_SRC", "/root/reference/pkg/src/pipemax")

import paper_2605_02189_b200 as _pkg  # noqa: E402
from paper_2605_02189_b200 import model_core as _mc  # noqa: E402
from paper_2605_02189_b200 import scheduler as _sched  # noqa: E402

sys.modules["pipemax"] = _pkg
sys.modules["pipemax.scheduler"] = _sched
sys.modules["pipemax.model_core"] = _mc
_spec = importlib.util.spec_from_file_location("pipemax.oracle", os.path.join(REF_SRC, "oracle.py"))
_oracle = importlib.util.module_from_spec(_spec)
sys.modules["pipemax.oracle"] = _oracle
_spec.loader.exec_module(_oracle)
_pkg.oracle = _oracle
