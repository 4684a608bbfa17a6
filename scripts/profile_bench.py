"""ncu target in the bench configuration: configs[3] species 0 (256^3,
phi_0..phi_2 same-vector), one warm apply then one profiled apply.  Each
apply launches 9 TMA mode-product kernels (quadrature batch, squaring batch,
exp action; 3 modes each):

  ncu --set full -k regex:mode_product_tma -s 9 -c 9 python scripts/profile_bench.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

pb = W.config(3).problems[0]
op = PhiKS(pb.A)
v = torch.from_numpy(np.ascontiguousarray(W.as_flat(pb.vs[0]))).cuda()
outs = [torch.empty_like(v) for _ in pb.ells]
for _ in range(2):
    op.apply(pb.tau, pb.ells, [v], mode=pb.mode, n_scales=pb.n_scales, outs=outs)
torch.cuda.synchronize()
st = op.stats()
print("ok", st["s"], st["q"], st["tucker_ops"], st["kernel_launches"])
