"""Host-link probe: pinned copy-engine bandwidth with 1, 2 and 4 concurrent streams per
direction (does splitting a transfer across copy engines beat one stream?)."""

import json
import torch

MIB = 1 << 20
n = 1024 * MIB
dev = torch.device("cuda", 0)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device=dev)
res = {}
for k in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    for name in ("d2h", "h2d"):
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i, s in enumerate(ss):
                s.wait_event(e0)
                with torch.cuda.stream(s):
                    if name == "d2h":
                        h[i * part:(i + 1) * part].copy_(d[i * part:(i + 1) * part], non_blocking=True)
                    else:
                        d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
            for s in ss:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
        res[f"{name}_{k}streams_gbs"] = round(n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
print(json.dumps(res))
