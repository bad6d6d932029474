"""Swapping with PyTorch's own caching allocator (no liblms pool installed).

``lms_swap_out`` holds the source block until its D2H lands only when
liblms's pool owns it (include/lms.h).  A tensor from PyTorch's caching
allocator must not be handed back to the compute stream while the D2H channel
still reads it: the binding records the tensor on the D2H stream.  The
session pool is installed in every other GPU test, so this runs in a fresh
interpreter with LMS_TEST_NO_POOL=1.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, %(root)r)
from paper_1807_02037_b200 import runtime as rt
from paper_1807_02037_b200.executor import ExecConfig, execute
from paper_1807_02037_b200 import RewriteConfig, rewrite
from paper_1807_02037_b200.workloads import ffchain, ffchain_inputs
import numpy as np
assert rt.installed_context() is None
ctx = rt.Context(device=0, timing=True)
n = 64 << 20
for codec in ("ce", "sm", "zvc"):
    t = torch.randn(n, device="cuda")
    want = t.cpu()
    old = t.data_ptr()
    torch.cuda._sleep(200_000_000)          # the D2H waits behind ~0.1 s of compute
    h = ctx.swap_out(t, codec)
    del t
    y = torch.empty(n, device="cuda")      # same size, same stream: the freed block if allowed
    assert y.data_ptr() != old, "caching allocator reused a block the D2H still reads"
    y.fill_(7.0)
    out = ctx.swap_in(h)
    ctx.wait(h)
    ctx.release(h)
    assert torch.equal(out.cpu(), want), codec
# the drop-in executor on its own context (no allocator installed)
g = ffchain(3, 256)
inputs = ffchain_inputs(g, 256, seed=0)
base, _ = execute(g, inputs, ExecConfig())
g2, _ = rewrite(g, RewriteConfig(lb=1, ub=3))
got, rep = execute(g2, inputs, ExecConfig(codec="zvc"))
for k in base:
    assert np.array_equal(got[k], base[k]), k
print("nopool ok")
"""


def test_swap_without_pool_is_safe():
    env = dict(os.environ, LMS_TEST_NO_POOL="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "nopool ok" in r.stdout
