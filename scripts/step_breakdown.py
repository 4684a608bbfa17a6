"""Per-step breakdown of the bench workload from the library's per-launch CUDA events
(set_profiling): int8 GEMMs, digit splits + chain tables, DMMA launches (exponential stage),
against the step time measured without profiling — what the kernels leave as gaps."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

wl = W.config(3)
pb = wl.problems[0]
op = PhiKS([p.A for p in wl.problems])
vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(p.vs[0]))).cuda() for p in wl.problems]
outs = [torch.empty_like(vs[0]) for _ in range(len(wl.problems) * len(pb.ells))]


def step():
    op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=outs)


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    step()
e1.record()
torch.cuda.synchronize()
t_plain = e0.elapsed_time(e1) / 10
op.set_profiling(True)
step()
torch.cuda.synchronize()
st = op.stats()
print(json.dumps({"step_ms_unprofiled": round(t_plain, 3), "i8_ms (splits+chain+gemm)": round(st["i8_ms"], 3),
                  "i8_gemm_ms": round(st["i8_gemm_ms"], 3), "i8_gemm_launches": st["i8_gemm_launches"],
                  "mode_product_ms (DMMA)": round(st["mode_product_ms"], 3), "expm_ms": round(st["expm_ms"], 3),
                  "kernel_launches": st["kernel_launches"]}))
