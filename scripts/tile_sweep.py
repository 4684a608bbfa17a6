"""Time μ-mode products and one configs[3] step for the tile variant selected
by the PHIKS_TILE environment variable (read once per process)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS, mode_product
from paper_2210_07667_b200 import workloads as W


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


out = {"variant": os.environ.get("PHIKS_TILE", "0")}
dims = (256, 256, 256)
N = int(np.prod(dims))
x = torch.randn(N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for mu in range(3):
    M = torch.randn(256 * 256, dtype=torch.float64, device="cuda")
    t = timed(lambda: mode_product(dims, mu, [x], [M], [y]))
    out[f"mode{mu}_tf"] = round(2 * N * 256 / t / 1e12, 2)
wl = W.config(3)
ops, vs, os_ = [], [], []
for pb in wl.problems:
    ops.append(PhiKS(pb.A)); vs.append(torch.from_numpy(W.as_flat(pb.vs[0]).copy()).cuda())
    os_.append([torch.empty_like(vs[-1]) for _ in pb.ells])
def step():
    for op, pb, v, o in zip(ops, wl.problems, vs, os_):
        op.apply(pb.tau, pb.ells, [v], outs=o)
t = timed(step, 5)
fl = sum(op.stats()["mu_mode_flops"] for op in ops)
out["step_ms"] = round(t * 1e3, 3)
out["step_tf"] = round(fl / t / 1e12, 2)
print(json.dumps(out), flush=True)
