"""Randomised check of block-diagonal handles (phiks_create_blocks) against
one handle per block: random nb = 1..4, d = 1..4, both modes, several scales
(one-off robustness sweep, not part of the suite)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

seed = int(os.environ.get("SEED", "1"))
count = int(os.environ.get("COUNT", "40"))
rng = np.random.default_rng(seed)
worst, fails = 0.0, []
for c in range(count):
    nb = int(rng.integers(1, 5))
    d = int(rng.integers(1, 5))
    dims = tuple(int(x) for x in rng.integers(1, {1: 200, 2: 90, 3: 30, 4: 12}[d], size=d))
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(0, 6))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    nv = 1 if mode == "same" else len(ells)
    blocks = [W.random_factors(dims, seed=3000 + 10 * c + b, scale=float(rng.uniform(0.2, 30.0))) for b in range(nb)]
    vs = [[W.as_flat(W.random_tensor(dims, seed=9000 + 50 * c + 7 * b + k)) for k in range(nv)] for b in range(nb)]
    tau = float(rng.uniform(0.05, 2.0))
    ns = int(rng.integers(1, 3))
    try:
        op = PhiKS(blocks)
        outs = op.apply(tau, ells, [torch.from_numpy(v.copy()).cuda() for vb in vs for v in vb], mode=mode,
                        n_scales=ns)
        per = len(outs) // nb
        e = 0.0
        for b in range(nb):
            sep = PhiKS(blocks[b]).apply(tau, ells, [torch.from_numpy(v.copy()).cuda() for v in vs[b]], mode=mode,
                                         n_scales=ns)
            for k in range(per):
                g = outs[b * per + k].cpu().numpy()
                s = sep[k].cpu().numpy()
                e = max(e, float(np.linalg.norm(g - s) / max(np.linalg.norm(s), 1e-300)))
        worst = max(worst, e)
        if e > 1e-14:
            fails.append({"case": c, "nb": nb, "dims": dims, "mode": mode, "ells": ells, "err": e})
    except Exception as ex:  # noqa: BLE001
        fails.append({"case": c, "nb": nb, "dims": dims, "mode": mode, "ells": ells, "exception": repr(ex)})
print(json.dumps({"seed": seed, "count": count, "worst_rel_diff_vs_separate_handles": worst, "fails": fails}))
