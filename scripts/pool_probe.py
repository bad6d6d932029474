"""Allocator behaviour probe: ResNet-50 no-swap steps near a budget, pool counters per step."""
import sys, time, json
sys.path.insert(0, '.')
import torch, torchvision
from paper_1807_02037_b200 import runtime as rt
budget = int(float(sys.argv[1]) * (1 << 30)) if len(sys.argv) > 1 else 16 << 30
ctx = rt.Context(device=0, device_reserve=budget, timing=True)
rt.install_allocator(ctx)
torch.backends.cudnn.benchmark = False
torch.backends.cudnn.allow_tf32 = False
m = torchvision.models.resnet50().cuda()
opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
for B in [int(a) for a in sys.argv[2:]] or [64, 128, 160]:
    x = torch.randn(B, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (B,), device="cuda")
    try:
        for i in range(6):
            s0 = ctx.stats(); t0 = time.perf_counter()
            opt.zero_grad(set_to_none=True)
            torch.nn.functional.cross_entropy(m(x), y).backward(); opt.step()
            torch.cuda.synchronize(); dt = time.perf_counter() - t0; s1 = ctx.stats()
            print(json.dumps({"B": B, "step": i, "ms": round(dt * 1e3, 1), "maps": s1["n_map"] - s0["n_map"],
                              "unmaps": s1["n_unmap"] - s0["n_unmap"], "syncs": s1["n_device_syncs"] - s0["n_device_syncs"],
                              "driver_ms": round(s1["pool_driver_ms"] - s0["pool_driver_ms"], 1),
                              "live_peak_GiB": round(s1["device_peak"] / 2**30, 2),
                              "mapped_GiB": round(s1["device_mapped"] / 2**30, 2)}), flush=True)
    except RuntimeError as e:
        print("B", B, "OOM", str(e)[:200], flush=True)
    x = y = None
