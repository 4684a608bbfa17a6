import json, os, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2210_07667_b200 import PhiKS
from paper_2210_07667_b200 import workloads as W
from oracle import phiks_oracle as O
for cfg in (1, 0):
    pb = W.config(cfg).problems[0]
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in pb.vs]
    for path in ("auto", "i8", "dmma"):
        op = PhiKS(pb.A); op.set_gemm_path(path)
        nout = len(pb.ells) * pb.n_scales if pb.mode == "same" else pb.n_scales
        outs = [torch.empty(op.N, dtype=torch.float64, device="cuda") for _ in range(nout)]
        for _ in range(3): op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
        e1.record(); torch.cuda.synchronize()
        print(cfg, path, round(e0.elapsed_time(e1) / 20, 3), "ms", op.stats()["i8_mode_launches"], flush=True)
