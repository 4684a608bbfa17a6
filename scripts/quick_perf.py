"""Quick GPU timing probe: FP64 peaks (DMMA/DFMA microbenchmark), per-mode
μ-mode product throughput at 256^3, and one full configs[3] φ-action."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS, fp64_peak_launch, mode_product  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402


def timed(fn, reps=5):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


res = {}
sink = torch.empty(148 * 8 * 256, dtype=torch.float64, device="cuda")
for kind, name in ((0, "dmma"), (1, "dfma")):
    for blocks in (148, 296, 592):
        fl = [0.0]

        def f():
            fl[0] = fp64_peak_launch(kind, blocks, 20000, sink)
        t = timed(f, 3)
        res[f"peak_{name}_{blocks}"] = fl[0] / t / 1e12
print(json.dumps(res), flush=True)

for dims in ((256, 256, 256), (512, 512, 256), (128, 128, 128), (512, 512)):
    N = int(np.prod(dims))
    x = torch.randn(N, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for mu, n in enumerate(dims):
        M = torch.randn(n * n, dtype=torch.float64, device="cuda")
        t = timed(lambda: mode_product(dims, mu, [x], [M], [y]))
        print(f"mode_product dims={dims} mu={mu}: {t*1e3:.3f} ms  {2*N*n/t/1e12:.2f} TF/s  "
              f"{2*N*8/t/1e9:.0f} GB/s", flush=True)

wl = W.config(3)
for pb in wl.problems:
    op = PhiKS(pb.A)
    v = torch.from_numpy(W.as_flat(pb.vs[0]).copy()).cuda()
    outs = [torch.empty_like(v) for _ in pb.ells]
    op.apply(pb.tau, pb.ells, [v], outs=outs)
    torch.cuda.synchronize()
    t0 = time.time()
    t = timed(lambda: op.apply(pb.tau, pb.ells, [v], outs=outs), 3)
    st = op.stats()
    print(pb.name, f"{t*1e3:.2f} ms", st, f"mu-mode {st['mu_mode_flops']/t/1e12:.2f} TF/s", flush=True)
