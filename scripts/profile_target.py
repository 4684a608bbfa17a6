"""ncu target: a few 256^3 μ-mode products (mode 2 = strided, mode 0 = KMAJ)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import mode_product
dims = (256, 256, 256)
N = 256 ** 3
x = torch.randn(N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
M = torch.randn(256 * 256, dtype=torch.float64, device="cuda")
for mu in (2, 2, 0, 0):
    mode_product(dims, mu, [x], [M], [y])
torch.cuda.synchronize()
print("ok")
