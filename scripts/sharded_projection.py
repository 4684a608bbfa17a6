"""Projection (NOT a measurement) of the slab-sharded configs[3] step at P
GPUs from one GPU: phiks_apply_ranks_serial runs the P ranks' launches back to
back on one GPU (same kernels, same peer-store epilogues, writing into the
other ranks' regions in local HBM instead of over NVLink), so its time / P
is the per-rank kernel time; the projection adds nothing for barriers or
NVLink latency.  Used only for DESIGN.md's scaling discussion.

A real apply runs stage A (the exponential stage and its all-gather) on the
handle's pre stream, overlapped with the previous apply (on one GPU that hides
it: DESIGN.md §0(f)), while the emulation replays it on the one stream.  So for
P > 1 the script also times the replay without stage A (phiks_apply_ranks_serial_ex
which = 2, reading the exponentials of the earlier full applies) and reports the
efficiency with stage A overlapped beside the all-inclusive one."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS, ShardedPhiKS, apply_ranks_serial  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402
from paper_2210_07667_b200.sharding import split_slabs  # noqa: E402

CFG = int(os.environ.get("CONFIG", "3"))  # 3: 256^3 Brusselator (bench); 4: 512x512x256 ADR lincomb (the 8-GPU config)
wl = W.config(CFG)
pb0 = wl.problems[0]
blocks = [pb.A for pb in wl.problems]
mode = pb0.mode
res = []
for P in [int(x) for x in os.environ.get("PS", "1,2,4,8").split(",")]:
    xs = [W.as_flat(v) for pb in wl.problems for v in pb.vs]
    if P == 1:
        ranks = [PhiKS(blocks)]
    else:
        ranks = [ShardedPhiKS(blocks, r, P, connect=None) for r in range(P)]
        ShardedPhiKS.connect_local(ranks)
    if os.environ.get("KSKIP") is not None:  # A/B of PHIKS_OPT_KSKIP
        for r in ranks:
            r.set_option("kskip", int(os.environ["KSKIP"]))
    ins = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, P)[r])).cuda() for x in xs] for r in range(P)]
    nout = len(wl.problems) * len(pb0.ells) if mode == "same" else pb0.n_scales
    outs = [[torch.empty(xs[0].size // P, dtype=torch.float64, device="cuda")
             for _ in range(nout)] for _ in range(P)]

    def step(which=0):
        if P == 1:
            ranks[0].apply(pb0.tau, pb0.ells, ins[0], mode=mode, n_scales=pb0.n_scales, outs=outs[0])
        else:
            apply_ranks_serial(ranks, pb0.tau, pb0.ells, ins, mode=mode, n_scales=pb0.n_scales, outs=outs,
                               which=which)

    def windows(which=0):
        reps = []
        for _ in range(int(os.environ.get("REPS", "3"))):  # best of REPS windows of 5 steps (power-cap noise)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                step(which)
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1) / 5)
        return reps
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    reps = windows()
    t = min(reps)
    res.append({"config": CFG, "P": P, "serial_ms": round(t, 3), "per_rank_ms": round(t / P, 3),
                "windows_ms": [round(x, 3) for x in reps]})
    if P > 1:
        ref = [o.clone() for o in outs[0]]
        reps2 = windows(2)  # stage A overlapped (its launches left out of the replay)
        assert all(torch.equal(a, b) for a, b in zip(ref, outs[0])), "which = 2 changed the outputs"
        res[-1].update({"serial_ms_stage_a_overlapped": round(min(reps2), 3),
                        "windows_ms_stage_a_overlapped": [round(x, 3) for x in reps2]})
    print(json.dumps(res[-1]), flush=True)
    del ranks, ins, outs
    torch.cuda.empty_cache()
t1 = res[0]["per_rank_ms"] * res[0]["P"]
for r in res:
    r["projected_efficiency"] = round(t1 / (r["P"] * r["per_rank_ms"]), 3)
    if "serial_ms_stage_a_overlapped" in r:
        r["projected_efficiency_stage_a_overlapped"] = round(t1 / r["serial_ms_stage_a_overlapped"], 3)
print(json.dumps(res))
