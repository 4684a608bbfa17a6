"""φ-action time and μ-mode GFLOP/s of every BASELINE.json config on one
B200 (device-resident inputs, CUDA events, after warm-up): the per-config
table of DESIGN.md.  configs[4] is the 8-GPU config of BASELINE; here it
runs whole on one GPU."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

reps = int(os.environ.get("REPS", "5"))
for idx in [int(x) for x in os.environ.get("CONFIGS", "0,1,2,3,4").split(",")]:
    wl = W.config(idx)
    ops, vins, outs = [], [], []
    for pb in wl.problems:
        op = PhiKS(pb.A)
        if os.environ.get("PRESPLIT") is not None:  # A/B of PHIKS_OPT_PRESPLIT
            op.set_option("presplit", int(os.environ["PRESPLIT"]))
        if os.environ.get("KSKIP") is not None:  # A/B of PHIKS_OPT_KSKIP
            op.set_option("kskip", int(os.environ["KSKIP"]))
        ops.append(op)
        vins.append([torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in pb.vs])
        nout = len(pb.ells) * pb.n_scales if pb.mode == "same" else pb.n_scales
        outs.append([torch.empty(op.N, dtype=torch.float64, device="cuda") for _ in range(nout)])

    def step():
        for op, pb, v, o in zip(ops, wl.problems, vins, outs):
            op.apply(pb.tau, pb.ells, v, mode=pb.mode, n_scales=pb.n_scales, outs=o)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    # timed without per-launch events (CUDA-graph replays), then a profiled pass for the shares
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    for op in ops:
        op.set_profiling(True)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(reps):
        step()
    e3.record()
    torch.cuda.synchronize()
    tp = e2.elapsed_time(e3) / reps / 1e3
    st = [op.stats() for op in ops]
    fl = sum(s["mu_mode_flops"] for s in st)
    mp_ms = sum(s["mode_product_ms"] for s in st)
    mp_fl = sum(s["mode_product_flops"] for s in st)
    print(json.dumps({"config": idx, "dims": wl.problems[0].dims, "mode": wl.problems[0].mode,
                      "plans": [(s["s"], s["q"], s["tucker_ops"]) for s in st],
                      "phi_action_ms": round(t * 1e3, 3), "mu_mode_gflops": round(fl / t / 1e9, 1),
                      "tucker_launch_tflops": round(mp_fl / (mp_ms / 1e3) / 1e12, 2) if mp_ms else None,
                      "profiled_ms": round(tp * 1e3, 3),
                      "tucker_share": round(mp_ms / reps / 1e3 / tp, 3) if mp_ms else None,
                      "expm_share": round(sum(s["expm_ms"] for s in st) / reps / 1e3 / tp, 3),
                      "expm_launches": sum(s["expm_launches"] for s in st) // reps,
                      "launches": sum(s["kernel_launches"] for s in st),
                      "presplit_inputs": sum(s["presplit_inputs"] for s in st)}), flush=True)
    del ops, vins, outs
    torch.cuda.empty_cache()
