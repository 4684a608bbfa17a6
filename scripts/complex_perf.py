"""Complex handle on the int8 path against FP64 DMMA: (1+i)/100·Δ factors on
256×256×64, φ_0..φ_2; prints per-apply time per path and the relative difference."""
import numpy as np, torch, sys, os, json
sys.path.insert(0, os.getcwd())
from paper_2210_07667_b200 import PhiKS
from paper_2210_07667_b200 import workloads as W
dims = (256, 256, 64)
fac = [(1 + 1j) / 100 * W.fd_dxx_dirichlet(n) for n in dims]
v = torch.from_numpy(np.ascontiguousarray(W.as_flat(W.random_tensor(dims, seed=3, complex_=True)).astype(np.complex128))).cuda()
res = {}
for path in ("dmma", "i8", "auto"):
    op = PhiKS(fac)
    op.set_gemm_path(path)
    for _ in range(2): op.apply(1.0, (0, 1, 2), [v])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): outs = op.apply(1.0, (0, 1, 2), [v])
    e1.record(); torch.cuda.synchronize()
    st = op.stats()
    res[path] = {"ms": e0.elapsed_time(e1) / 5, "i8_launches": st["i8_mode_launches"], "tucker": st["tucker_ops"], "launches": st["kernel_launches"]}
    res[path + "_out"] = [o.cpu().numpy() for o in outs]
    op.close()
err = max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(res["i8_out"], res["dmma_out"]))
print(json.dumps({k: v for k, v in res.items() if not k.endswith("_out")}), "i8_vs_dmma_rel", err)
