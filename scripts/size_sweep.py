"""μ-mode product throughput vs tensor size at n = 256 (L2-resident small
tensors vs HBM-streamed large ones): does DRAM latency limit the kernel?"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import mode_product  # noqa: E402

def timed(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3

M = torch.randn(256 * 256, dtype=torch.float64, device="cuda")
for R in (16, 32, 64, 128, 256, 512):
    dims = (256, 256, R)
    N = 256 * 256 * R
    x = torch.randn(N, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    out = {"dims": dims, "MB_in": N * 8 / 1e6}
    for mu in (0, 1):
        t = timed(lambda: mode_product(dims, mu, [x], [M], [y]))
        out[f"mode{mu+1}_tf"] = round(2 * N * 256 / t / 1e12, 2)
    print(json.dumps(out), flush=True)
