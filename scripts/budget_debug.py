import sys, time, faulthandler
faulthandler.dump_traceback_later(60, repeat=True)
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1807_02037_b200 import runtime as rt, RewriteConfig, rewrite
from paper_1807_02037_b200.executor import execute, ExecConfig
from paper_1807_02037_b200.workloads import ffchain, ffchain_inputs
ctx = rt.Context(device=0, device_reserve=24 << 30, timing=True)
rt.install_allocator(ctx)
L, N = 8, 4096
tb = N * N * 4
g = ffchain(L, N); inputs = ffchain_inputs(g, N, seed=1)
for i in range(2):
    t0 = time.time(); base, rep0 = execute(g, inputs, ExecConfig(), ctx=ctx)
    print("noswap", i, round(time.time() - t0, 2), "peak tensors", rep0.peak_device_bytes / tb, flush=True)
torch.cuda.synchronize(); ctx.synchronize()
st = ctx.stats(); print({k: st[k] / tb for k in ("device_in_use", "device_mapped", "device_cached")}, flush=True)
limit = st["device_in_use"] + (L + 1) * tb + int(0.75 * rep0.peak_device_bytes)
ctx.set_limit(limit); print("limit tensors", limit / tb, ctx.stats()["device_limit"] / tb, flush=True)
try:
    _, r = execute(g, inputs, ExecConfig(), ctx=ctx)
    print("no-swap under limit: NO OOM, peak", r.peak_device_bytes / tb, ctx.stats()["device_peak"] / tb, flush=True)
except RuntimeError as e:
    print("no-swap OOM as expected", str(e)[:150], flush=True)
g2, _ = rewrite(g, RewriteConfig(lb=1, ub=3))
t0 = time.time()
got, rep = execute(g2, inputs, ExecConfig(codec="ce"), ctx=ctx)
print("swap under limit", round(time.time() - t0, 2), "peak", rep.peak_device_bytes / tb, all(np.array_equal(got[k], base[k]) for k in base), flush=True)
st = ctx.stats(); print({k: st[k] for k in ("n_map", "n_unmap", "n_oom", "n_deferred_frees", "pool_driver_ms")}, flush=True)
