"""Context numbers for DESIGN.md: one φ-action on the paper's own ADR workload
shape (§4.2, Eq. (ADR) l.1455-1476: ε = 0.5, α = 10, Dirichlet,
n = 64..121 per direction, τ = 0.1/100 as in the ETD2RK runs of Table
'tab:ord2' l.1836-1849) on one B200.  The paper's per-call time on an
i7-10750H with MATLAB (l.1058-1061) is context only: its tolerance was tuned
to the integrator's accuracy, ours is 2^-53."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

tau = 0.1 / 100
for n in (64, 81, 100, 121):
    A = 0.5 * W.fd_dxx_dirichlet(n) + 10.0 * W.fd_dx_dirichlet(n)
    op = PhiKS([A, A, A])
    rng = np.random.default_rng(n)
    vs = [torch.from_numpy(rng.uniform(-1, 1, n ** 3)).cuda() for _ in range(3)]
    res = {"n": n}
    for mode, ells, vin in (("lincomb", (0, 1, 2), vs), ("same", (1, 2), vs[:1])):
        for _ in range(3):
            op.apply(tau, ells, vin, mode=mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            op.apply(tau, ells, vin, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        st = op.stats()
        res[mode] = {"ms_per_call": round(e0.elapsed_time(e1) / 10, 3), "s": st["s"], "q": st["q"],
                     "tucker_ops": st["tucker_ops"]}
    print(json.dumps(res), flush=True)
