"""One configs[4] apply after a warm-up (for an ncu launch list of the 8-GPU BASELINE config on one GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_07667_b200 import PhiKS
from paper_2210_07667_b200 import workloads as W
wl = W.config(4)
pb = wl.problems[0]
op = PhiKS(pb.A)
v = [torch.from_numpy(np.ascontiguousarray(W.as_flat(x))).cuda() for x in pb.vs]
outs = [torch.empty(op.N, dtype=torch.float64, device="cuda") for _ in range(pb.n_scales)]
for _ in range(2):
    op.apply(pb.tau, pb.ells, v, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
torch.cuda.synchronize()
