"""Randomised parity sweep of the chained int8 modes against the oracle
(one-off robustness check, not part of the suite): shapes that take the chained route
(n_1 ∈ {128, 256}, the other n_μ multiples of 16 up to 256, d = 2..4), real random factors
of random scale, both modes, 1-3 scales, the int8 path forced; CHAIN=0/1/2 is the handle's
PHIKS_OPT_CHAIN (default 2: chained regardless of the Metzler guard)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

seed = int(os.environ.get("SEED", "1"))
count = int(os.environ.get("COUNT", "40"))
path = os.environ.get("GEMM_PATH", "i8")  # i8 or dmma
chain = int(os.environ.get("CHAIN", "2"))
per_case = []
rng = np.random.default_rng(seed)
worst, fails, chained = 0.0, [], 0
t0 = time.time()
for c in range(count):
    d = int(rng.integers(2, 5))
    while True:
        dims = [int(rng.choice([128, 256]))] + [16 * int(x) for x in rng.integers(1, 17, size=d - 1)]
        if np.prod(dims) <= 1 << 20:
            break
    dims = tuple(dims)
    fac = W.random_factors(dims, seed=5000 + c, scale=float(rng.uniform(0.1, 30.0)))
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(0, 5))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    vs = [W.random_tensor(dims, seed=6000 + 7 * c + k) * float(np.exp(rng.uniform(-30, 30)))
          for k in range(1 if mode == "same" else len(ells))]
    tau = float(rng.uniform(0.05, 2.0))
    ns = int(rng.integers(1, 4))
    op = PhiKS(fac)
    op.set_gemm_path(path)
    op.set_option("chain", chain)
    outs = op.apply(tau, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in vs],
                    mode=mode, n_scales=ns)
    torch.cuda.synchronize()
    st = op.stats()
    chained += st["i8_chained_ops"]
    ref = O.phiks(fac, tau, mode, ells, vs, n_scales=ns)
    exps = ([W.as_flat(ref.out[(ell, j)]) for j in range(ns) for ell in ells] if mode == "same"
            else [W.as_flat(ref.out[j]) for j in range(ns)])
    cw = 0.0
    for k, (g, e) in enumerate(zip(outs, exps)):
        err = float(np.linalg.norm(g.cpu().numpy() - e) / max(np.linalg.norm(e), 1e-300))
        worst = max(worst, err)
        cw = max(cw, err)
        if not err <= 1e-12:
            fails.append({"case": c, "dims": dims, "mode": mode, "out": k, "err": err})
    per_case.append(cw)
    op.close()
print(json.dumps({"seed": seed, "count": count, "path": path, "chain": chain,
                  "worst_rel_err": worst, "fails": fails, "per_case_worst": per_case,
                  "chained_tucker_ops": int(chained), "seconds": time.time() - t0}))
