"""Per-config A/B of the GEMM paths (auto / dmma / i8) for the small BASELINE configs: φ-action ms, best of 3 windows of 10."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2210_07667_b200 import PhiKS
from paper_2210_07667_b200 import workloads as W
for idx in (1, 0, 2):
    wl = W.config(idx)
    pb = wl.problems[0]
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in pb.vs]
    for path in ("auto", "dmma", "i8"):
        op = PhiKS(pb.A)
        op.set_gemm_path(path)
        nout = len(pb.ells) * pb.n_scales if pb.mode == "same" else pb.n_scales
        outs = [torch.empty(op.N, dtype=torch.float64, device="cuda") for _ in range(nout)]
        for _ in range(3):
            op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
        torch.cuda.synchronize()
        best = 1e9
        for w in range(3):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(10):
                op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 10)
        st = op.stats()
        print(json.dumps({"config": idx, "path": path, "ms": round(best, 3), "i8_launches": st["i8_mode_launches"], "chained": st["i8_chained_ops"]}), flush=True)
