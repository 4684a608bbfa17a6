"""BASELINE configs[4] at FULL size (512×512×256, 67 M unknowns, lincomb ℓ = 0..4, ETD-RK4-
shaped) through the C ABI on cuda:0, against the CPU oracle on the same seeded inputs
(relative 2-norm ≤ 1e-12), with the oracle's wall time.  Writes one JSON object
(profiles/r02_cfg4_fullsize_parity.json).  Run on the GPU box:
    python scripts/fullsize_cfg4_parity.py > profiles/r02_cfg4_fullsize_parity.json
tests/test_gpu_fullsize.py::test_config4_full_oracle_parity runs the same check when
PHIKS_SLOW_TESTS=1."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import torch
    from oracle import phiks_oracle as O
    from paper_2210_07667_b200 import PhiKS
    from paper_2210_07667_b200 import workloads as W

    pb = W.config(4).problems[0]
    op = PhiKS(pb.A)
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in pb.vs]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    st = op.stats()
    got = out[0].cpu().numpy()
    del out, vs, op
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=pb.n_scales)
    t_oracle = time.perf_counter() - t0
    exp = W.as_flat(ref.out[0])
    err = float(np.linalg.norm(got - exp) / np.linalg.norm(exp))
    return {"config": "BASELINE configs[4]: d=3, (512,512,256), ADR eps=1, alpha=(10,10,-10), Dirichlet, "
                      "tau=1e-4, lincomb l=0..4, 5 vectors U[-1,1] seed 4",
            "rel_2norm_err": err, "tol": 1e-12, "pass": err <= 1e-12,
            "library_plan": {"s": st["s"], "q": st["q"], "tucker_ops": st["tucker_ops"],
                             "i8_chained_ops": st["i8_chained_ops"]},
            "oracle_plan": {"s": ref.plan.s, "q": ref.plan.q, "tucker_ops": ref.tucker_ops},
            "gpu_first_apply_s": t_gpu, "oracle_wall_s": t_oracle, "host_cores": os.cpu_count()}


if __name__ == "__main__":
    print(json.dumps(run()))
