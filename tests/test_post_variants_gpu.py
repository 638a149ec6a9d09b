"""The vectorised stream-K fixup kernels (4 rows per thread, the default) are
bit-identical to the thread-per-row kernels they replaced (PM_POST_SCALAR=1):
same partial-sum order, same epilogue arithmetic.  The switch is read once per
process, so each variant runs in its own interpreter on the same seeded
inputs and the outputs are compared here."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
from paper_2605_02189_b200 import ops
DEV = "cuda"
out = {{}}
def ws_for(lin, m_cap=256):
    return ops.GemmWorkspace(m_cap, ops.GemmWorkspace.floats_needed([lin], m_cap), lin.n_units, lin.n_units, DEV)
g = torch.Generator(device=DEV).manual_seed(11)
for name, n_out, k, m, epi in [("store", 6144, 4096, 77, ops.EPI_STORE_BF16), ("resid", 4096, 12288, 128, ops.EPI_RESID_ADD),
                               ("silu", 2 * 3072, 4096, 100, ops.EPI_SILU_MUL), ("pad", 640, 8192, 33, ops.EPI_STORE_BF16),
                               ("logits", 30000, 1024, 50, ops.EPI_LOGITS_ARGMAX)]:
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    x = torch.zeros(256, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    lin = ops.Linear(w)
    ws = ws_for(lin)
    assert lin.plan(m)[2] > 1, name   # the partition splits units: the fixup kernel runs
    width = n_out // 2 if epi == ops.EPI_SILU_MUL else n_out
    dt = torch.float32 if epi in (ops.EPI_RESID_ADD, ops.EPI_LOGITS_ARGMAX) else torch.bfloat16
    y = torch.randn(256, width, generator=g, device=DEV).to(dt)
    lin(ops.activation_maps(x), m, epi, y, width, ws)
    if epi == ops.EPI_LOGITS_ARGMAX:
        ids = torch.full((256,), -1, dtype=torch.int32, device=DEV)
        ops.argmax_reduce(ws, lin.n_units, m, ids)
        out[name + "_ids"] = ids.cpu()
    out[name] = y.cpu()
# O projection fused with residual + next RMSNorm
w = (torch.randn(4096, 4096, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
x = torch.zeros(256, 4096, device=DEV, dtype=torch.bfloat16)
x[:90] = torch.randn(90, 4096, generator=g, device=DEV).to(torch.bfloat16)
lin = ops.Linear(w)
ws = ws_for(lin)
resid = torch.randn(256, 4096, generator=g, device=DEV)
nw = (1 + 0.1 * torch.randn(4096, generator=g, device=DEV)).to(torch.bfloat16)
xn = torch.zeros(256, 4096, device=DEV, dtype=torch.bfloat16)
lin.resid_rmsnorm(ops.activation_maps(x), 90, resid, ws, nw, xn, 1e-6)
torch.cuda.synchronize()
out["norm_resid"], out["norm_xn"] = resid.cpu(), xn.cpu()
torch.save(out, sys.argv[1])
"""


def _run(tmp_path, scalar):
    path = str(tmp_path / f"post_{scalar}.pt")
    env = dict(os.environ, PM_POST_SCALAR=str(scalar), PM_FIX_POLL="0")   # scalar kernels do not poll
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), path], env=env, check=True, timeout=600)
    return torch.load(path)


def test_vectorised_fixups_bit_identical_to_scalar(tmp_path):
    vec, sca = _run(tmp_path, 0), _run(tmp_path, 1)
    assert vec.keys() == sca.keys()
    for key in vec:
        assert torch.equal(vec[key], sca[key]), key
