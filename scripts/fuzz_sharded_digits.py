"""Randomised sweep of the sharded int8 digit stages (round 2): P ∈ {2, 4, 8}
emulated ranks, d = 3..4 with n_1 ∈ {128, 256} and n_{d-1} a multiple of 32·P (so the stage-0
epilogue writes mode d's digit planes into the owners), FD (Metzler) factors under the default
guard or dense random factors with chaining forced, both modes, 1-3 scales; each case against the
oracle and against one GPU (one-off robustness check, not part of the suite)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, ShardedPhiKS, apply_ranks_serial  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402
from paper_2210_07667_b200.sharding import split_slabs  # noqa: E402

seed = int(os.environ.get("SEED", "1"))
count = int(os.environ.get("COUNT", "24"))
rng = np.random.default_rng(seed)
worst_oracle, worst_single, fails, digit_cases = 0.0, 0.0, [], 0
t0 = time.time()
for c in range(count):
    d = int(rng.integers(3, 5))
    P = int(rng.choice([2, 4, 8])) if d == 3 else 2  # d = 4 with P > 2 cannot stay below 2^19 elements
    for _ in range(1000):  # bounded: draw until the tensor is small enough for the oracle
        dims = [int(rng.choice([128, 256]))]
        dims += [16 * int(x) for x in rng.integers(1, 5, size=d - 3)]
        dims += [32 * P * int(rng.integers(1, 3)), 16 * int(rng.integers(1, 5))]  # n_d % 16: int8 stage 1
        if np.prod(dims) <= (1 << 21 if d == 4 else 1 << 19):
            break
    else:
        raise RuntimeError("no admissible dims")
    dims = tuple(dims)
    fd = bool(rng.integers(0, 2))
    if fd:
        fac = [(0.2 + rng.uniform(0, 1)) * (W.fd_dxx_neumann(n) if k % 2 == 0 else
                                           W.fd_dxx_dirichlet(n) + rng.uniform(0, 5) * W.fd_dx_dirichlet(n))
               for k, n in enumerate(dims)]
        tau = float(rng.uniform(1e-4, 5e-3))
    else:
        fac = W.random_factors(dims, seed=7000 + c, scale=float(rng.uniform(0.5, 10.0)))
        tau = float(rng.uniform(0.05, 1.0))
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(1, 5))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    ns = int(rng.integers(1, 4))
    vs = [W.random_tensor(dims, seed=8000 + 7 * c + k) for k in range(1 if mode == "same" else len(ells))]
    chain = 1 if fd else 2
    ranks = [ShardedPhiKS(fac, r, P, connect=None) for r in range(P)]
    ShardedPhiKS.connect_local(ranks)
    for r in ranks:
        r.set_gemm_path("i8")
        r.set_option("chain", chain)
    flat = [W.as_flat(v) for v in vs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, P)[r])).cuda() for x in flat] for r in range(P)]
    outs = apply_ranks_serial(ranks, tau, ells, vecs, mode=mode, n_scales=ns)
    torch.cuda.synchronize()
    gathered = [torch.cat([outs[r][i] for r in range(P)]).cpu().numpy() for i in range(len(outs[0]))]
    digit_cases += int(all(r.stats()["shard_digit_ops"] > 0 for r in ranks))
    for r in ranks:
        r.close()
    op = PhiKS(fac)
    op.set_gemm_path("i8")
    op.set_option("chain", chain)
    single = [o.cpu().numpy() for o in op.apply(tau, ells, [torch.from_numpy(x.copy()).cuda() for x in flat],
                                                  mode=mode, n_scales=ns)]
    op.close()
    ref = O.phiks(fac, tau, mode, ells, vs, n_scales=ns)
    exps = ([W.as_flat(ref.out[(ell, j)]) for j in range(ns) for ell in ells] if mode == "same"
            else [W.as_flat(ref.out[j]) for j in range(ns)])
    for k, (g, s1, e) in enumerate(zip(gathered, single, exps)):
        eo = float(np.linalg.norm(g - e) / max(np.linalg.norm(e), 1e-300))
        es = float(np.linalg.norm(g - s1) / max(np.linalg.norm(s1), 1e-300))
        worst_oracle, worst_single = max(worst_oracle, eo), max(worst_single, es)
        if not (eo <= 1e-12 and es <= 1e-13):  # noqa: E501
            fails.append({"case": c, "dims": dims, "P": P, "mode": mode, "out": k, "vs_oracle": eo, "vs_single": es})
    print(json.dumps({"case": c, "dims": dims, "P": P, "mode": mode, "fd": fd, "t": round(time.time() - t0, 1)}),
          file=sys.stderr, flush=True)
print(json.dumps({"seed": seed, "count": count, "digit_stage_cases": digit_cases, "worst_vs_oracle": worst_oracle,
                  "worst_vs_single_gpu": worst_single, "fails": fails, "seconds": time.time() - t0}))
