"""Randomised parity sweep against the oracle (one-off robustness check, not
part of the suite): random d, dims (ragged, odd, TMA and cp.async shapes),
real/complex factors, both modes, several scales, library-chosen plans."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

seed = int(os.environ.get("SEED", "1"))
count = int(os.environ.get("COUNT", "60"))
rng = np.random.default_rng(seed)
worst, fails = 0.0, []
t0 = time.time()
for c in range(count):
    d = int(rng.integers(1, 5))
    hi = {1: 300, 2: 200, 3: 70, 4: 20}[d]
    dims = tuple(int(x) for x in rng.integers(1, hi, size=d))
    cplx = bool(rng.integers(0, 4) == 0)
    fac = W.random_factors(dims, seed=1000 + c, scale=float(rng.uniform(0.1, 40.0)), complex_=cplx)
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(0, 6))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    nv = 1 if mode == "same" else len(ells)
    vs = [W.random_tensor(dims, seed=5000 + 7 * c + k, complex_=cplx) for k in range(nv)]
    tau = float(rng.uniform(0.05, 2.0))
    ns = int(rng.integers(1, 4))
    try:
        op = PhiKS(fac)
        dt = torch.complex128 if cplx else torch.float64
        outs = op.apply(tau, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to("cuda", dt) for v in vs],
                        mode=mode, n_scales=ns)
        torch.cuda.synchronize()
        ref = O.phiks(fac, tau, mode, ells, vs, n_scales=ns)
        st = op.stats()
        e = 0.0
        for j in range(ns):
            if mode == "same":
                for i, ell in enumerate(ells):
                    r = W.as_flat(ref.out[(ell, j)])
                    g = outs[j * len(ells) + i].cpu().numpy()
                    e = max(e, float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)))
            else:
                r = W.as_flat(ref.out[j])
                g = outs[j].cpu().numpy()
                e = max(e, float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)))
        same_plan = (st["s"], st["q"]) == (ref.plan.s, ref.plan.q)
        worst = max(worst, e)
        if e > 1e-12 or not same_plan:
            fails.append({"case": c, "dims": dims, "cplx": cplx, "mode": mode, "ells": ells, "err": e,
                          "plan": (st["s"], st["q"]), "oracle_plan": (ref.plan.s, ref.plan.q)})
    except Exception as ex:  # noqa: BLE001
        fails.append({"case": c, "dims": dims, "cplx": cplx, "mode": mode, "ells": ells, "exception": repr(ex)})
print(json.dumps({"seed": seed, "count": count, "worst_rel_err": worst, "fails": fails,
                  "seconds": round(time.time() - t0, 1)}))
