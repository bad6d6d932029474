import torch, sys
sys.path.insert(0, '.')
from paper_1807_02037_b200 import runtime as rt
ctx = rt.Context(device=0, device_reserve=4 << 30, timing=True)
rt.install_allocator(ctx)
base = torch.randn(6, 40, 66, device="cuda")
views = {"contig": base, "slice_rows": base[:, 3:37, :], "transpose": base.transpose(1, 2),
         "step": base[::2, ::3, ::5], "expand": base[:, :1, :].expand(6, 40, 66),
         "big_rows": torch.randn(257, 1030, device="cuda")[:, 7:1007]}
for name, v in views.items():
    got = ctx.pack(v)
    torch.cuda.synchronize()
    want = v.contiguous()
    bad = (got != want).nonzero()
    print(name, tuple(v.shape), v.stride(), "mismatches", bad.shape[0], bad[:3].tolist(),
          got.flatten()[:4].tolist(), want.flatten()[:4].tolist())
from paper_1807_02037_b200.workloads import ffchain, ffchain_inputs
from paper_1807_02037_b200 import rewrite, RewriteConfig
from paper_1807_02037_b200.executor import execute, ExecConfig
import numpy as np
g = ffchain(8, 1024); inputs = ffchain_inputs(g, 1024)
base, rep0 = execute(g, inputs, ExecConfig(), ctx=ctx)
g2, rr = rewrite(g, RewriteConfig(lb=1, ub=3))
for codec in ("ce", "sm", "zvc"):
    got, rep = execute(g2, inputs, ExecConfig(codec=codec), ctx=ctx)
    print(codec, [np.array_equal(got[k], base[k]) for k in base], rep0.peak_device_bytes, rep.peak_device_bytes,
          rep.transfer_time_total, rep.transfer_wait_total, rep.makespan, rep0.makespan)
st = ctx.stats()
try:
    ctx.set_limit(st["device_in_use"] + (64 << 20))
    a = torch.empty(32 << 20, dtype=torch.uint8, device="cuda")
    torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
except Exception as e:
    print("OOM raised:", type(e).__name__, str(e)[:200])
