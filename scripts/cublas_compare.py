"""cuBLAS DGEMM (torch.matmul, fp64) on the μ-mode-product shapes of a 256^3
tensor, next to this library's mode-product kernel: the library baseline for
the same contraction (not used by the library)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import mode_product  # noqa: E402

def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3

n = 256
N = n ** 3
x = torch.randn(N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
M = torch.randn(n, n, dtype=torch.float64, device="cuda")
fl = 2.0 * N * n
res = {}
# mode 1 (k contiguous): Y(r, j) = X(r, k) M(j, k)  -> (65536 x 256) @ (256 x 256)
X1 = x.view(n * n, n)
Y1 = y.view(n * n, n)
res["cublas_mode1_tf"] = fl / timed(lambda: torch.matmul(X1, M.t(), out=Y1)) / 1e12
# mode 3 (outermost): Y(l, j) = Σ_k M(j,k) X(l, k) with l contiguous -> M @ X3 where X3 = (256 x 65536)
X3 = x.view(n, n * n)
Y3 = y.view(n, n * n)
res["cublas_mode3_tf"] = fl / timed(lambda: torch.matmul(M, X3, out=Y3)) / 1e12
# mode 2 (middle): batched over the outer index: (256 batches) M @ X(l-contiguous 256 x 256)
X2 = x.view(n, n, n)
Y2 = y.view(n, n, n)
res["cublas_mode2_batched_tf"] = fl / timed(lambda: torch.matmul(M, X2, out=Y2)) / 1e12
Mf = M.t().contiguous().reshape(-1)  # column-major for the library
for mu in range(3):
    res[f"phiks_mode{mu+1}_tf"] = fl / timed(lambda: mode_product((n, n, n), mu, [x], [Mf], [y])) / 1e12
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
