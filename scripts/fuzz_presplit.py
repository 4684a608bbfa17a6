"""Randomised sweep of the chained int8 path with the pre-split combination (one-off robustness
check, not part of the suite): FD-shaped Metzler factors (diffusion + advection), shapes on which
the modes chain, both modes, random orders and scales; each case against the oracle and against the
same handle with PHIKS_OPT_PRESPLIT = 0 (bit for bit)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

seed = int(os.environ.get("SEED", "7"))
count = int(os.environ.get("COUNT", "16"))
rng = np.random.default_rng(seed)
worst, fails, hits = 0.0, [], 0
t0 = time.time()


def factor(n, k):
    if rng.integers(0, 2) == 0:
        return float(rng.uniform(0.1, 1.0)) * W.fd_dxx_neumann(n)
    return float(rng.uniform(0.1, 1.0)) * W.fd_dxx_dirichlet(n) + float(rng.uniform(-20, 20)) * W.fd_dx_dirichlet(n)


for c in range(count):
    d = int(rng.integers(2, 4))
    if d == 2:
        dims = (int(rng.choice([128, 256, 384, 512])), int(rng.choice([128, 256])))
    else:
        dims = (int(rng.choice([128, 256, 384])), int(rng.choice([128, 256])), int(rng.choice([16, 32, 48])))
    fac = [factor(n, k) for k, n in enumerate(dims)]
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(1, 5))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    nv = 1 if mode == "same" else len(ells)
    vs = [W.uniform_tensor(dims, -1.0, 1.0, seed=7000 + 11 * c + k) for k in range(nv)]
    tau = float(10 ** rng.uniform(-4, -1.5))
    ns = int(rng.integers(1, 5))
    case = {"case": c, "dims": dims, "mode": mode, "ells": ells, "tau": tau, "n_scales": ns}
    try:
        res = []
        for pre in (1, 0):
            op = PhiKS(fac)
            op.set_gemm_path("i8")
            op.set_option("presplit", pre)
            outs = op.apply(tau, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in vs],
                            mode=mode, n_scales=ns)
            torch.cuda.synchronize()
            st = op.stats()
            res.append([o.cpu().numpy() for o in outs])
            if pre:
                case["plan"] = (st["s"], st["q"])
                case["presplit_inputs"] = st["presplit_inputs"]
                case["chained_ops"] = st["i8_chained_ops"]
                hits += st["presplit_inputs"] > 0
        ref = O.phiks(fac, tau, mode, ells, vs, n_scales=ns)
        refs = ([W.as_flat(ref.out[(ell, j)]) for j in range(ns) for ell in ells] if mode == "same"
                else [W.as_flat(ref.out[j]) for j in range(ns)])
        e = max(float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)) for g, r in zip(res[0], refs))
        bitwise = all(np.array_equal(a, b) for a, b in zip(*res))
        worst = max(worst, e)
        case.update({"err": e, "bitwise": bitwise})
        if e > 1e-12 or not bitwise:
            fails.append(case)
    except Exception as ex:  # noqa: BLE001
        case["exception"] = repr(ex)
        fails.append(case)
    print(json.dumps(case), flush=True)
print(json.dumps({"seed": seed, "count": count, "cases_with_presplit": hits, "worst_rel_err": worst, "fails": fails,
                  "seconds": round(time.time() - t0, 1)}))
