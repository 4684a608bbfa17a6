"""Randomised check of the slab-sharded path (ranks emulated on one GPU)
against the single-GPU path: random d = 2..4, P ∈ {2, 4, 8}, both modes,
several scales (one-off robustness sweep, not part of the suite)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS, ShardedPhiKS, apply_ranks_serial  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402
from paper_2210_07667_b200.sharding import split_slabs  # noqa: E402

seed = int(os.environ.get("SEED", "1"))
count = int(os.environ.get("COUNT", "40"))
rng = np.random.default_rng(seed)
worst, fails = 0.0, []
for c in range(count):
    P = int(rng.choice([2, 4, 8]))
    d = int(rng.integers(2, 5))
    dims = [int(x) for x in rng.integers(2, 40 if d <= 3 else 12, size=d)]
    if os.environ.get("RAGGED"):
        dims[-1] = P + int(rng.integers(0, 60 if d <= 3 else 12))
        dims[-2] = P + int(rng.integers(0, 60 if d <= 3 else 12))
    else:
        dims[-1] = P * int(rng.integers(1, 40 if d <= 3 else 6))
        dims[-2] = P * int(rng.integers(1, 40 if d <= 3 else 6))
    dims = tuple(dims)
    fac = W.random_factors(dims, seed=2000 + c, scale=float(rng.uniform(0.2, 20.0)))
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(0, 6))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    nv = 1 if mode == "same" else len(ells)
    vs = [W.as_flat(W.random_tensor(dims, seed=7000 + 5 * c + k)) for k in range(nv)]
    tau = float(rng.uniform(0.05, 2.0))
    ns = int(rng.integers(1, 3))
    try:
        single = PhiKS(fac).apply(tau, ells, [torch.from_numpy(v.copy()).cuda() for v in vs], mode=mode, n_scales=ns)
        ranks = [ShardedPhiKS(fac, r, P, connect=None) for r in range(P)]
        ShardedPhiKS.connect_local(ranks)
        vecs = [[torch.from_numpy(np.ascontiguousarray(split_slabs(v, P, dims)[r])).cuda() for v in vs]
                for r in range(P)]
        outs = apply_ranks_serial(ranks, tau, ells, vecs, mode=mode, n_scales=ns)
        torch.cuda.synchronize()
        e = 0.0
        for i in range(len(single)):
            g = torch.cat([outs[r][i] for r in range(P)]).cpu().numpy()
            s = single[i].cpu().numpy()
            e = max(e, float(np.linalg.norm(g - s) / max(np.linalg.norm(s), 1e-300)))
        worst = max(worst, e)
        if e > 1e-13:
            fails.append({"case": c, "P": P, "dims": dims, "mode": mode, "ells": ells, "err": e})
        for r in ranks:
            r.close()
    except Exception as ex:  # noqa: BLE001
        fails.append({"case": c, "P": P, "dims": dims, "mode": mode, "ells": ells, "exception": repr(ex)})
print(json.dumps({"seed": seed, "count": count, "worst_rel_diff_vs_single_gpu": worst, "fails": fails}))
