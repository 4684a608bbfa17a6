"""GEMM path A/B (DMMA vs int8) over shapes near the auto threshold (n ≥ 128, N ≥ 2^20): φ-action ms, best of 3 windows of 10."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2210_07667_b200 import PhiKS
from paper_2210_07667_b200 import workloads as W
cases = [((512, 512), "lincomb", 1), ((256, 256), "same", 0), ((384, 384), "same", 0), ((256, 256, 16), "same", 0),
         ((128, 128, 32), "same", 0), ((512, 256), "lincomb", 1), ((128, 128, 64), "lincomb", 1)]
if os.environ.get("CASES") == "short":
    cases = [((512, 512), "lincomb", 1), ((256, 256, 16), "same", 0)]
for dims, mode, lin in cases:
    A = [W.fd_dxx_dirichlet(n) + 10.0 * W.fd_dx_dirichlet(n) for n in dims]
    ells = (0, 1, 2, 3) if mode == "lincomb" else (0, 1, 2)
    vs = [W.uniform_tensor(dims, -1, 1, seed=3 + k) for k in range(len(ells) if mode == "lincomb" else 1)]
    dv = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in vs]
    res = {}
    for path in ("auto", "dmma", "i8"):
        op = PhiKS(A); op.set_gemm_path(path)
        outs = [torch.empty(op.N, dtype=torch.float64, device="cuda") for _ in range(len(ells) if mode == "same" else 1)]
        for _ in range(3): op.apply(1e-4, ells, dv, mode=mode, outs=outs)
        torch.cuda.synchronize()
        best = 1e9
        for w in range(3):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(10): op.apply(1e-4, ells, dv, mode=mode, outs=outs)
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 10)
        res[path] = round(best, 3)
    print(json.dumps({"dims": dims, "mode": mode, "N": int(np.prod(dims)), **res, "s_q": (op.stats()["s"], op.stats()["q"])}), flush=True)
