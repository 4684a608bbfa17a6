"""ncu target in the bench configuration: configs[3], both species in one
block-diagonal handle (256^3, phi_0..phi_2 same-vector), one warm apply then
one profiled apply.  On the default (int8) path an apply launches 10 int8
GEMMs (oz_gemm_kernel: merged quadrature+exp-action batch of both species and
the merged squaring batch, 3 modes each, inputs split in chunks of 8):

  ncu --set full -k regex:oz_gemm -s 10 -c 10 python scripts/profile_bench.py

with GEMM_PATH=dmma (the handle's phiks_set_gemm_path), 6 DMMA launches of the 64x128
instantiation:

  GEMM_PATH=dmma ncu --set full --kernel-name-base demangled \
      -k "regex:tma_kernel<.int.64, .int.128" -s 6 -c 6 python scripts/profile_bench.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

wl = W.config(3)
pb = wl.problems[0]
op = PhiKS([p.A for p in wl.problems])
op.set_gemm_path(os.environ.get("GEMM_PATH", "auto"))
vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(p.vs[0]))).cuda() for p in wl.problems]
outs = [torch.empty_like(vs[0]) for _ in range(len(wl.problems) * len(pb.ells))]
for _ in range(2):
    op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)
torch.cuda.synchronize()
st = op.stats()
print("ok", st["block_plans"], st["tucker_ops"], st["kernel_launches"])
