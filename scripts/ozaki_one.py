"""One int8 μ-mode product of a 256³ tensor (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import mode_product_i8  # noqa: E402

S = int(os.environ.get("OZ_S", "8"))
mu = int(os.environ.get("OZ_MU", "1"))
nb = int(os.environ.get("OZ_TERMS", "1"))
dims = (256, 256, 256)
N = 256 ** 3
ins = [torch.rand(N, dtype=torch.float64, device="cuda") for _ in range(nb)]
outs = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(nb)]
M = torch.randn(256 * 256, dtype=torch.float64, device="cuda")
ws = None
for _ in range(3):
    ws = mode_product_i8(dims, mu, ins, [M] * nb, outs, slices=S, workspace=ws)
torch.cuda.synchronize()
