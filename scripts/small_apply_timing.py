"""Per-apply latency of small problems (launch-bound): configs[0] (2-D 32²) and
the small configs[2], device memory, 200 applies; GRAPHS=0/1 sets the handles' PHIKS_OPT_GRAPHS."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

res = {"graphs": int(os.environ.get("GRAPHS", "1"))}
for name, pb in (("cfg0", W.config(0).problems[0]), ("cfg2_small", W.config(2, small=True).problems[0])):
    op = PhiKS(pb.A)
    op.set_option("graphs", res["graphs"])
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in pb.vs]
    nout = len(pb.ells) * pb.n_scales if pb.mode == "same" else pb.n_scales
    outs = [torch.empty(op.N, dtype=torch.float64, device="cuda") for _ in range(nout)]
    for _ in range(5):
        op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
    torch.cuda.synchronize()
    res[name + "_us_per_apply"] = round((time.perf_counter() - t0) / 200 * 1e6, 1)
    res[name + "_launches"] = op.stats()["kernel_launches"]
print(json.dumps(res))
