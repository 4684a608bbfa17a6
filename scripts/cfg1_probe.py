import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2210_07667_b200 import PhiKS
from paper_2210_07667_b200 import workloads as W
wl = W.config(1)
pb = wl.problems[0]
for graphs in (1, 0):
    op = PhiKS(pb.A)
    op.set_option("graphs", graphs)
    v = [torch.from_numpy(np.ascontiguousarray(W.as_flat(x))).cuda() for x in pb.vs]
    outs = [torch.empty(op.N, dtype=torch.float64, device="cuda") for _ in range(pb.n_scales)]
    ts = []
    for i in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply(pb.tau, pb.ells, v, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
        e1.record()
        torch.cuda.synchronize()
        ts.append((round((time.perf_counter() - t0) * 1e3, 3), round(e0.elapsed_time(e1), 3)))
    print("graphs", graphs, ts)
