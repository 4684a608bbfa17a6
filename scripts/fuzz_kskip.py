"""Randomised sweep of the zero-block skipping (PHIKS_OPT_KSKIP; one-off robustness
check, not part of the suite): banded factors of random bandwidth (FD stencils and random banded
matrices, Metzler or not, so both the chained and the unchained int8 paths run), mode sizes with one
to four k-blocks, both request modes, random τ, orders and scales; each case bit for bit against the
same handle with the option off, with the k-block counters showing how much was skipped, and against
the oracle on the smaller cases."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

seed = int(os.environ.get("SEED", "11"))
count = int(os.environ.get("COUNT", "24"))
rng = np.random.default_rng(seed)
t0 = time.time()
res_all, fails, worst = [], [], 0.0


METZLER = bool(int(os.environ.get("METZLER", "0")))  # 1: Metzler factors only, so the int8 modes chain


def factor(n):
    kind = int(rng.integers(0, 2 if METZLER else 3))
    if kind == 0:  # diffusion (Metzler)
        return float(rng.uniform(0.05, 1.0)) * W.fd_dxx_neumann(n)
    if kind == 1:  # advection-diffusion (Metzler at cell Péclet < 2 only)
        eps = float(rng.uniform(0.05, 1.0))
        amax = 1.9 * eps * (n + 1) if METZLER else 200.0  # cell Péclet |α|h/ε < 2: off-diagonals ≥ 0
        return eps * W.fd_dxx_dirichlet(n) + float(rng.uniform(-amax, amax)) * W.fd_dx_dirichlet(n)
    b = int(rng.integers(1, 40))  # random banded, mixed signs, scaled to ‖A‖ ~ n²
    A = rng.standard_normal((n, n)) * float(n) ** 2 / (2 * b + 1)
    i, j = np.indices((n, n))
    A[np.abs(i - j) > b] = 0.0
    return A


for c in range(count):
    d = int(rng.integers(2, 4))
    sizes = [128, 192, 256, 320, 384, 448, 512]
    if d == 2:
        dims = (int(rng.choice(sizes)), int(rng.choice([128, 256, 384])))
    else:
        dims = (int(rng.choice([128, 256, 384])), int(rng.choice([128, 256, 512])), int(rng.choice([16, 32, 64, 128, 256])))
    fac = [factor(n) for n in dims]
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(1, 5))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    nv = 1 if mode == "same" else len(ells)
    vs = [W.uniform_tensor(dims, -1.0, 1.0, seed=9000 + 13 * c + k) * float(10 ** rng.uniform(-3, 3))
          for k in range(nv)]
    tau = float(10 ** rng.uniform(-6, -3))
    ns = int(rng.integers(1, 4))
    case = {"case": c, "dims": dims, "mode": mode, "ells": ells, "tau": tau, "n_scales": ns}
    try:
        outs2 = []
        for ks in (1, 0):
            op = PhiKS(fac)
            op.set_gemm_path("i8")
            op.set_option("kskip", ks)
            op.set_profiling(True)
            outs = op.apply(tau, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in vs],
                            mode=mode, n_scales=ns)
            torch.cuda.synchronize()
            st = op.stats()
            outs2.append([o.cpu().numpy() for o in outs])
            if ks:
                case.update(plan=(st["s"], st["q"]), chained_ops=st["i8_chained_ops"],
                            kblocks=st["i8_kblocks"], kblocks_run=st["i8_kblocks_run"])
            op.close()
        case["bitwise"] = all(np.array_equal(a, b) for a, b in zip(*outs2))
        if int(np.prod(dims)) <= (1 << 21):
            ref = O.phiks(fac, tau, mode, ells, vs, n_scales=ns)
            refs = ([W.as_flat(ref.out[(ell, j)]) for j in range(ns) for ell in ells] if mode == "same"
                    else [W.as_flat(ref.out[j]) for j in range(ns)])
            e = max(float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)) for g, r in zip(outs2[0], refs))
            case["err_vs_oracle"] = e
            worst = max(worst, e)
            if e > 1e-12:
                fails.append(c)
        if not case["bitwise"]:
            fails.append(c)
    except Exception as ex:  # noqa: BLE001
        case["error"] = repr(ex)
        fails.append(c)
    res_all.append(case)
    print(json.dumps(case), flush=True)
print(json.dumps({"summary": {"count": count, "seed": seed, "fails": fails, "worst_err_vs_oracle": worst,
                              "bitwise_all": all(c.get("bitwise") for c in res_all),
                              "skipped_fraction": 1 - sum(c.get("kblocks_run", 0) for c in res_all) /
                              max(1, sum(c.get("kblocks", 0) for c in res_all)),
                              "seconds": time.time() - t0}}))
