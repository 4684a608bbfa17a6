"""Host<->device copy bandwidth with pinned host memory (the e2e bound of bench.py): one
direction at a time and both at once, 805 MB D2H / 268 MB H2D as in the configs[3] step."""
import json
import torch

n_d2h, n_h2d = 805306368 // 8, 268435456 // 8
dev_out = torch.empty(n_d2h, dtype=torch.float64, device="cuda")
dev_in = torch.empty(n_h2d, dtype=torch.float64, device="cuda")
host_out = torch.empty(n_d2h, dtype=torch.float64).pin_memory()
host_in = torch.empty(n_h2d, dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in (("d2h", lambda: host_out.copy_(dev_out, non_blocking=True)),
                 ("h2d", lambda: dev_in.copy_(host_in, non_blocking=True))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    nbytes = (n_d2h if name == "d2h" else n_h2d) * 8
    res[name] = {"ms": round(ms, 3), "GBps": round(nbytes / ms / 1e6, 1)}
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        host_out.copy_(dev_out, non_blocking=True)
    with torch.cuda.stream(s2):
        dev_in.copy_(host_in, non_blocking=True)
torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
res["both_ms_per_step"] = round(e0.elapsed_time(e1) / 5, 3)
print(json.dumps(res))
