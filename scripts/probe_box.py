"""One-off probe of the GPU box: topology, host RAM, host-link bandwidth, ResNet-50 fp32 step."""
import json, os, subprocess, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["nproc"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
out["free"] = sh("free -g")
out["cgroup_mem"] = sh("cat /sys/fs/cgroup/memory.max 2>/dev/null; cat /sys/fs/cgroup/memory/memory.limit_in_bytes 2>/dev/null")
out["topo"] = sh("nvidia-smi topo -m")
out["smi"] = sh("nvidia-smi --query-gpu=name,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,pcie.link.gen.current,memory.total --format=csv")
out["numa"] = sh("lscpu | head -30")
out["ulimit_l"] = sh("ulimit -l")
print(json.dumps(out, indent=1))

dev = torch.device("cuda:0")
res = {}
for mib in (64, 256, 1024):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        res[f"{name}_{mib}MiB_GBs"] = 5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res[f"duplex_{mib}MiB_GBs_each"] = 5 * n / dt / 1e9
    del h, d, h2, d2
print(json.dumps(res, indent=1))

t0 = time.perf_counter()
big = torch.empty(16 << 30, dtype=torch.uint8, pin_memory=True)
print("pin 16GiB s", time.perf_counter() - t0)
del big

import torchvision
torch.backends.cudnn.benchmark = True
for tf32 in (False, True):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    m = torchvision.models.resnet50().to(dev)
    opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
    for B in (64, 256):
        x = torch.randn(B, 3, 224, 224, device=dev); y = torch.randint(0, 1000, (B,), device=dev)
        torch.cuda.reset_peak_memory_stats()
        for i in range(8):
            if i == 3:
                torch.cuda.synchronize(); t0 = time.perf_counter()
            opt.zero_grad(set_to_none=True)
            loss = torch.nn.functional.cross_entropy(m(x), y)
            loss.backward(); opt.step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(json.dumps({"tf32": tf32, "B": B, "img_s": B / dt, "peak_GiB": torch.cuda.max_memory_allocated() / 2**30}))
    del m, opt
