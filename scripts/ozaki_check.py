"""Correctness and timing of the int8 tensor-core μ-mode product
(phiks_mode_product_i8) against the fp64 DMMA kernel and numpy.

    python scripts/ozaki_check.py [--quick]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import mode_product, mode_product_i8  # noqa: E402


def np_mode(x, dims, mu, M):
    X = x.reshape(dims[::-1])  # C order: last axis = mode 0
    ax = len(dims) - 1 - mu
    Y = np.moveaxis(np.tensordot(M, X, axes=([1], [ax])), 0, ax)
    return Y.reshape(-1)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    quick = "--quick" in sys.argv
    dev = "cuda"
    rng = np.random.default_rng(0)
    res = {"checks": [], "timing": []}
    shapes = [((40, 33, 17), 0), ((40, 33, 17), 1), ((40, 33, 17), 2), ((256, 9), 0), ((7, 250), 1),
              ((130, 64, 5), 1), ((256, 70), 0), ((3, 128, 129), 2), ((33, 200, 41), 1), ((1, 1000, 96), 2)]
    for dims, mu in shapes:
        N = int(np.prod(dims))
        n = dims[mu]
        for S in (6, 7):
            xs = [rng.standard_normal(N) * np.exp(rng.uniform(-3, 3, N)) for _ in range(2)]
            Ms = [rng.standard_normal((n, n)) for _ in range(2)]
            xin = [torch.from_numpy(x).to(dev) for x in xs]
            Min = [torch.from_numpy(np.asfortranarray(M).reshape(-1, order="F").copy()).to(dev) for M in Ms]
            ins = [xin[0], xin[1], xin[0]]
            mats = [Min[0], Min[1], Min[1]]
            outs = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(3)]
            mode_product_i8(dims, mu, ins, mats, outs, slices=S)
            torch.cuda.synchronize()
            for b, (xi, Mi) in enumerate([(0, 0), (1, 1), (0, 1)]):
                ref = np_mode(xs[xi], dims, mu, Ms[Mi])
                e = rel(outs[b].cpu().numpy(), ref)
                res["checks"].append({"dims": dims, "mu": mu, "S": S, "term": b, "rel": e})
                print(f"dims={dims} mu={mu} S={S} term={b} rel={e:.3e}", flush=True)
    if not quick:
        dims = (256, 256, 256)
        N = 256 ** 3
        x = torch.rand(N, dtype=torch.float64, device=dev)
        M = torch.randn(256 * 256, dtype=torch.float64, device=dev)
        for mu in range(3):
            for nb in (1, 8):
                ins = [x] * nb if mu == 0 else [torch.rand(N, dtype=torch.float64, device=dev) for _ in range(nb)]
                outs = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(nb)]
                mats = [M] * nb
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                row = {"mu": mu, "terms": nb}
                for S in (0, 6, 7):
                    ws = None
                    for it in range(4):
                        if it == 1:
                            ev[0].record()
                        if S == 0:
                            mode_product(dims, mu, ins, mats, outs)
                        else:
                            ws = mode_product_i8(dims, mu, ins, mats, outs, slices=S, workspace=ws)
                    ev[1].record()
                    torch.cuda.synchronize()
                    ms = ev[0].elapsed_time(ev[1]) / 3
                    row["dmma_ms" if S == 0 else f"i8_S{S}_ms"] = ms
                    if S == 0:
                        ref = outs[0].clone()
                    else:
                        row[f"i8_S{S}_rel_vs_dmma"] = rel(outs[0].cpu().numpy(), ref.cpu().numpy())
                res["timing"].append(row)
                print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/ozaki_check.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
