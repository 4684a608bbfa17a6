"""configs[3] slab-sharded at P = 8 emulated on one GPU: k-block counters per rank (profiling) for
PHIKS_OPT_KSKIP on and off, and one apply to profile under ncu (KSKIP env)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_07667_b200 import ShardedPhiKS, apply_ranks_serial
from paper_2210_07667_b200 import workloads as W
from paper_2210_07667_b200.sharding import split_slabs
wl = W.config(3)
pb0 = wl.problems[0]
P = 8
ranks = [ShardedPhiKS([pb.A for pb in wl.problems], r, P, connect=None) for r in range(P)]
ShardedPhiKS.connect_local(ranks)
ks = int(os.environ.get("KSKIP", "1"))
for r in ranks:
    r.set_option("kskip", ks)
xs = [W.as_flat(v) for pb in wl.problems for v in pb.vs]
ins = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, P)[r])).cuda() for x in xs] for r in range(P)]
for _ in range(2):
    apply_ranks_serial(ranks, pb0.tau, pb0.ells, ins, mode=pb0.mode, n_scales=pb0.n_scales)
torch.cuda.synchronize()
for r in ranks:
    r.op.set_profiling(True)
apply_ranks_serial(ranks, pb0.tau, pb0.ells, ins, mode=pb0.mode, n_scales=pb0.n_scales)
torch.cuda.synchronize()
st = [r.op.stats() for r in ranks]
print(json.dumps({"kskip": ks, "kblocks": [s["i8_kblocks"] for s in st], "run": [s["i8_kblocks_run"] for s in st],
                  "i8_gemm_ms": [round(s["i8_gemm_ms"], 3) for s in st]}))
