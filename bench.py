#!/usr/bin/env python
"""PHIKS benchmark (driver contract: one JSON line on rank 0).

Workload: BASELINE.json configs[3] — d=3, n=256^3 (N≈16.8M, 134 MB per
vector), fp64, two independent Kronecker sums (Brusselator species, block-
diagonal K̂, §4.4), each A_μ = D_s·(Neumann FD Laplacian), D_u=2e-3,
D_v=1e-3, τ=5e-3; φ_0..φ_2 (same-vector mode) on one U[0,3] vector per species
(seed 3).  One step = the φ-action of both species (planning, small-matrix
exponentials, quadrature, squaring, exp action), inputs resident in HBM.

metric: fp64 μ-mode GFLOP/s (2·N·Σ_μ n_μ per executed Tucker operator) of the
whole φ-action, plus φ-action wall time (ms_per_step).

  python bench.py [--gpus N --steps K --warmup W]      # this framework (CUDA)
  python bench.py --impl reference ...                 # the CPU oracle (reference arm)
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 μ-mode GFLOP/s & φ-action time, 3D 256³"
UNIT = "GFLOP/s"
WORKLOAD = ("configs[3]: d=3, n=256^3, fp64, Brusselator-shaped block-diagonal K (2 species, "
            "A_mu = D_s*Neumann FD Laplacian, D_u=2e-3, D_v=1e-3), tau=5e-3, phi_0..phi_2 same-vector, "
            "v ~ U[0,3] seed 3")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML every 5 ms on a
    thread (nvidia-smi as the fallback, whose start-up can miss a short timed region)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = [0x8, 0x40, 0x20, 0x4]  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap

            def poll():
                while True:
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append([str(self.gpu), str(sm), str(mx), "", ""] +
                                         ["Active" if rs & b else "Not Active" for b in bits])
                    except Exception:
                        pass
                    if self.stop.wait(0.005):
                        return

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        self.stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.t is not None:
            self.t.join(timeout=1)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            js = json.load(f)
        return js.get("dram_bytes_per_gflop"), js.get("source")
    except Exception:
        return None, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def expm_entry(args, ex_n, ex_ms):
    return {"launches": ex_n, "event_ms_per_step": ex_ms / max(args.steps, 1),
            "note": "runs on the handle's side stream, overlapped with the other species' Tucker "
                    "launches; its event time includes that sharing"}


def dmma_roofline(args, t_local, mp_ms, mp_fl, mp_n, ex_n, ex_ms, peak_tf):
    bpg, tsrc = load_traffic()
    # dram bytes per launch: the committed ncu capture's bytes per algorithmic GFLOP
    # of this kernel, times the average GFLOP of the launches timed here
    traffic = bpg * (mp_fl / max(mp_n, 1) / 1e9) if (bpg and mp_n) else None
    ach = mp_fl / (mp_ms / 1e3) / 1e12 if mp_ms > 0 else None
    return {"bound": "tensor", "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": (ach / peak_tf) if ach else None, "traffic": traffic,
            "kernel": "mode_product_tma_kernel (FP64 DMMA.8x8x4, TMA + mbarrier ring): the Tucker-operator launches",
            "algorithmic_bytes_per_launch": 16.0 * (mp_fl / max(mp_n, 1)) / (2.0 * 256),
            "peak_source": "measured in this run: phiks_fp64_peak_launch DMMA microbenchmark (max of 3)",
            "per_launch_ms": mp_ms / max(mp_n, 1), "launches_timed": mp_n,
            "share_of_step": (mp_ms / 1e3) / t_local if t_local > 0 else None,
            "expm_stage": expm_entry(args, ex_n, ex_ms), "traffic_source": tsrc}


I8_PAIRS = 28  # digit products per fp64 product: pairs (s, t) of 7 digits with s + t < 7


def i8_roofline(args, t_local, mp_ms, mp_fl, mp_n, i8_ms, i8_fl, g_ms, g_n, ex_n, ex_ms, dmma_peak, clocks=None,
                kblocks=(0, 0)):
    """Roofline of the dominant kernel, the int8 digit-product GEMM (ozaki.cu): algorithmic int8
    ops = 28 digit pairs × 2·rows·n² per fp64 product; peak = the measured bf16 dense peak of
    MEASURED_PEAKS.json × 2 (the guide's nominal int8 : bf16 ratio).  The denominator follows the
    clock the kernel actually ran at: the burst figure (measured at max SM clock) when the median
    SM clock sampled over the timed region is ≥ 0.95 of max, else the sustained figure (measured
    at a power-capped 1342 MHz median).  With PHIKS_OPT_KSKIP the GEMM skips the digit blocks of E
    that are all zero: `achieved` counts only the MMAs that ran (the library's
    k-block counters), the dense count is reported beside it."""
    pk = measured_peaks()
    burst_bf16, sust_bf16 = pk.get("bf16_tflops"), pk.get("bf16_tflops_sustained")
    at_max = bool(clocks and clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
                  and clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    bf16 = (burst_bf16 if at_max else sust_bf16) or burst_bf16 or sust_bf16
    peak = 2.0 * bf16 if bf16 else 4500.0
    dense_ops = I8_PAIRS * i8_fl  # i8_flops counts 2·rows·n² per GEMM term
    kb_tot, kb_run = kblocks
    run_frac = kb_run / kb_tot if kb_tot else 1.0
    ops = dense_ops * run_frac  # the MMAs that ran (equal work per (unit, k-block))
    ach = ops / (g_ms / 1e3) / 1e12 if g_ms > 0 else None
    tr = load_i8_traffic()
    per_launch_gflop = i8_fl / max(g_n, 1) / 1e9
    traffic = tr["dram_bytes_per_fp64_gflop"] * per_launch_gflop if tr else None
    # algorithmic bytes of a GEMM launch: the fiber digits (7 B per element and distinct input, once)
    # + the fp64 outputs (8 B per element and term); elements per term = flops / (2·n), n = 256
    elems = i8_fl / max(g_n, 1) / (2.0 * 256)
    burst = 2.0 * pk["bf16_tflops"] if pk.get("bf16_tflops") else None
    # the tcgen05 kind::i8 issue rate measured by scripts/umma_probe.cu (profiles/r01_mma_probes.json):
    # 7930 MACs/SM/clk with the GEMM's own MMA sequence and stage synchronisation, operands in smem
    probe = 2.0 * 7930 * 148 * 1.965e9 / 1e12
    sust = 2.0 * sust_bf16 if sust_bf16 else None
    return {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TOP/s (int8)",
            "frac": (ach / peak) if ach else None, "traffic": traffic,
            "peak_basis": "burst (SM clock median >= 0.95 of max in the timed region)" if at_max
            else "sustained (SM clocks below 0.95 of max in the timed region)",
            "frac_vs_burst": (ach / burst) if (ach and burst) else None,
            "frac_vs_sustained": (ach / sust) if (ach and sust) else None,
            "frac_vs_mma_probe": (ach / probe) if ach else None,
            "other_peaks": {"burst_tops": burst, "sustained_tops": sust, "mma_probe_tops": probe,
                            "note": "burst = MEASURED_PEAKS bf16_tflops x 2 (max SM clock); sustained = "
                                    "bf16_tflops_sustained x 2 (1342 MHz power-capped median); the MMA-issue "
                                    "probe (scripts/umma_probe.cu) is the GEMM's own MMA sequence from smem"},
            "kernel": "oz_gemm_kernel<7, AMN, OUTD> (tcgen05.mma kind::i8, TMEM accumulators, TMA SWIZZLE_128B, chained modes: DESIGN.md §4d): "
                      "the Tucker-operator μ-mode products",
            "algorithmic_ops_per_launch": ops / max(g_n, 1),
            "dense_ops_per_launch": dense_ops / max(g_n, 1),
            "frac_dense_equivalent": (dense_ops / (g_ms / 1e3) / 1e12 / peak) if g_ms > 0 else None,
            "kblocks_run_fraction": run_frac,
            "kblocks_note": "(fibre tile x 64-row n-tile, 128-wide k-block) units whose E digits are not all zero "
                            "(PHIKS_OPT_KSKIP, DESIGN.md §4g); the skipped ones add exact integer zeros",
            "algorithmic_bytes_per_launch_max": elems * 15.0,
            "peak_source": (f"MEASURED_PEAKS.json {'bf16_tflops' if at_max else 'bf16_tflops_sustained'} × 2 "
                            "(int8 : bf16 dense = 2, B200_PROFILING.md)") if bf16
            else "nominal 4.5 POPS (MEASURED_PEAKS.json absent)",
            "per_launch_ms": g_ms / max(g_n, 1), "launches_timed": g_n,
            "share_of_step": (g_ms / 1e3) / t_local if t_local > 0 else None,
            "fp64_equivalent": {"tflops": i8_fl / (i8_ms / 1e3) / 1e12 if i8_ms > 0 else None,
                                "vs_measured_dmma_peak": (i8_fl / (i8_ms / 1e3) / 1e12 / dmma_peak)
                                if i8_ms > 0 else None, "dmma_peak_tflops": dmma_peak,
                                "note": "fp64 flops of the products over the int8 path's time (splits of the inputs, chain exponent bounds "
                                        "+ GEMM)"},
            "digit_splits": {"ms_per_step": (i8_ms - g_ms) / max(args.steps, 1)},
            "tucker_launches": {"ms_per_step": mp_ms / max(args.steps, 1), "launches": mp_n},
            "expm_stage": expm_entry(args, ex_n, ex_ms),
            "traffic_source": tr.get("source") if tr else None}


def load_i8_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_summary_i8.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
def run_oracle_sample(problems):
    """The oracle (as it stands) on a bounded sample; returns (flops, seconds)."""
    from oracle import phiks_oracle as O
    flops = 0.0
    t0 = time.perf_counter()
    for pb in problems:
        res = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=pb.n_scales)
        flops += res.tucker_ops * 2.0 * np.prod(pb.dims) * sum(pb.dims)
    return flops, time.perf_counter() - t0


def blas_threads():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return int(max(i.get("num_threads", 1) for i in info)) if info else os.cpu_count()
    except Exception:
        return os.cpu_count()


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2210_07667_b200 import workloads as W
    wl = W.config(3)
    sample = [wl.problems[0]]  # bounded sample: species 0 (u) φ-action at full 256^3
    for _ in range(args.warmup):
        run_oracle_sample(sample)
    tot_f, tot_t = 0.0, 0.0
    for _ in range(args.steps):
        f, t = run_oracle_sample(sample)
        tot_f += f
        tot_t += t
    value = tot_f / tot_t / 1e9
    ms = tot_t / args.steps * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": "species 0 only per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
                         "sample": "one species (u) φ_0..φ_2 action at full 256^3 per step (numpy/OpenBLAS fp64)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def b200_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2210_07667_b200 import PhiKS, ShardedPhiKS, fp64_peak_launch
    from paper_2210_07667_b200 import workloads as W
    from paper_2210_07667_b200.sharding import split_slabs

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    # ---- workload: configs[3], the block-diagonal K̂ = diag(K_u, K_v) of the two
    # species in ONE handle (phiks_create_blocks, §4.4: per-species plans,
    # shared launches); N > 1 slab-shards every tensor along mode 3 ----
    wl = W.config(3)
    pb0 = wl.problems[0]
    assert all((pb.tau, pb.ells, pb.mode, pb.n_scales) == (pb0.tau, pb0.ells, pb0.mode, pb0.n_scales)
               for pb in wl.problems)
    blocks = [pb.A for pb in wl.problems]
    op = ShardedPhiKS(blocks, rank, world) if world > 1 else PhiKS(blocks)
    ops = [op]
    vins, host_in = [], []
    for pb in wl.problems:
        x = W.as_flat(pb.vs[0])
        if world > 1:
            x = np.ascontiguousarray(split_slabs(x, world)[rank])
        vins.append(torch.from_numpy(x.copy()).to(dev))
        hi = torch.empty(x.size, dtype=torch.float64, pin_memory=True)
        hi.numpy()[:] = x
        host_in.append(hi)
    nloc = vins[0].numel()
    outs = [torch.empty_like(vins[0]) for _ in range(len(wl.problems) * len(pb0.ells))]
    host_out = [torch.empty(nloc, dtype=torch.float64, pin_memory=True) for _ in outs]

    def step():
        op.apply(pb0.tau, pb0.ells, vins, mode=pb0.mode, n_scales=pb0.n_scales, outs=outs, stream=stream)

    def step_host():
        # public API with pinned host buffers: H2D of the step's inputs and D2H of every
        # output inside the library's apply (PHIKS_MEM_HOST_ASYNC: copies on its own
        # streams; the exp-action outputs leave while the rest of the step runs)
        op.apply(pb0.tau, pb0.ells, [v.numpy() for v in host_in], mode=pb0.mode, n_scales=pb0.n_scales,
                 outs=[t.numpy() for t in host_out], host_async=True)

    # ---- measured FP64 tensor-core peak (DMMA microbenchmark) ----
    sink = torch.empty(148 * 4 * 256, dtype=torch.float64, device=dev)
    fp64_peak_launch(0, 148 * 4, 2000, sink)
    torch.cuda.synchronize()
    peaks = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fl = fp64_peak_launch(0, 148 * 4, 40000, sink)
        e1.record(stream)
        torch.cuda.synchronize()
        peaks.append(fl / (e0.elapsed_time(e1) / 1e3) / 1e12)
    peak_tf = max(peaks)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    flops_step = sum(o.stats()["mu_mode_flops"] for o in ops)
    plans = [{"species": b, "s": s, "q": q} for b, (s, q) in enumerate(op.stats()["block_plans"])]
    plans.append({"T_executed_total": op.stats()["tucker_ops"]})

    # ---- timed region (device-resident inputs) ----
    for op in ops:
        op.set_profiling(True)
    launches0 = sum(op.stats()["total_kernel_launches"] for op in ops)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_local = e0.elapsed_time(e1) / 1e3
    st = [op.stats() for op in ops]
    launches = sum(s["total_kernel_launches"] for s in st) - launches0
    mp_ms = sum(s["mode_product_ms"] for s in st)
    mp_fl = sum(s["mode_product_flops"] for s in st)
    mp_n = sum(s["mode_product_launches"] for s in st)
    ex_ms = sum(s["expm_ms"] for s in st)
    ex_n = sum(s["expm_launches"] for s in st)
    i8_ms = sum(s["i8_ms"] for s in st)
    i8_fl = sum(s["i8_flops"] for s in st)
    i8_gemm_ms = sum(s["i8_gemm_ms"] for s in st)
    i8_gemm_n = sum(s["i8_gemm_launches"] for s in st)
    kblocks = (sum(s["i8_kblocks"] for s in st), sum(s["i8_kblocks_run"] for s in st))
    for op in ops:
        op.set_profiling(False)
    t = t_local
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    value = flops_step * world * args.steps / t / 1e9

    # ---- N > 1: self-check of the gathered slabs of the last timed step against one GPU ----
    parity = None
    if world > 1:
        torch.cuda.synchronize()
        gathered = []
        for o in outs:
            parts = [torch.empty_like(o) for _ in range(world)]
            dist.all_gather(parts, o)
            gathered.append(torch.cat(parts) if rank == 0 else None)
        if rank == 0:
            ref_op = PhiKS(blocks)
            full_in = [torch.from_numpy(W.as_flat(pb.vs[0]).copy()).to(dev) for pb in wl.problems]
            ref = ref_op.apply(pb0.tau, pb0.ells, full_in, mode=pb0.mode, n_scales=pb0.n_scales, stream=stream)
            torch.cuda.synchronize()
            errs = [float(torch.linalg.norm(g - r) / torch.linalg.norm(r)) for g, r in zip(gathered, ref)]
            parity = {"vs": "the same apply on one GPU (rank 0, unsharded handle)", "max_rel_2norm_err": max(errs),
                      "tol": 1e-12, "pass": max(errs) <= 1e-12, "outputs": len(errs)}
            del ref_op, full_in, ref
        del gathered
        torch.cuda.empty_cache()
        dist.barrier()

    # ---- end-to-end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        step_host()
        for op in ops:
            op.wait()
        torch.cuda.synchronize()
        k = max(1, args.steps)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            step_host()
        for op in ops:
            op.wait()
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": flops_step * world * k / te / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": sum(8 * t.numel() for t in host_in),
               "d2h_bytes_per_step": sum(8 * t.numel() for t in host_out),
               "ms_per_step": te / k * 1e3, "timing": "host wall clock around k steps of C-ABI applies with pinned host buffers (PHIKS_MEM_HOST_ASYNC) and the final wait"}

    # ---- CPU baseline: the oracle, rank 0, N = 1 only ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        f, tc = run_oracle_sample(wl.problems)
        cpu = {"value": f / tc / 1e9, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
               "sample": "the full step (both species, 256^3) once, numpy/OpenBLAS fp64", "seconds": tc}

    if i8_gemm_n:
        roof = i8_roofline(args, t_local, mp_ms, mp_fl, mp_n, i8_ms, i8_fl, i8_gemm_ms, i8_gemm_n, ex_n, ex_ms,
                           peak_tf, clocks=clk.summary(), kblocks=kblocks)
    else:
        roof = dmma_roofline(args, t_local, mp_ms, mp_fl, mp_n, ex_n, ex_ms, peak_tf)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "compute": ("μ-mode products as exact int8 digit products on the tcgen05 tensor cores (7 balanced "
                        "base-256 digits per fp64 operand, int32 accumulation, fp64 splits and epilogue: "
                        "DESIGN.md §4c)") if i8_gemm_n else "fp64 DMMA tensor cores",
            "config": {"workload": WORKLOAD, "handle": "one block-diagonal handle (2 blocks = species)",
                       "parallelism": f"slab{world} (mode-3 slabs, transposition fused into peer stores)"
                       if world > 1 else "single",
                       "l2": "inputs larger than L2 (134 MB per vector > 126 MB L2)", "plans": plans,
                       "mu_mode_gflop_per_step": flops_step / 1e9,
                       "mu_mode_flops": "2*N*sum(n_mu) per executed Tucker operator (dense mu-mode products, the "
                                        "metric's count); the int8 GEMM skips the E digit blocks that are all zero "
                                        "(roofline.kblocks_run_fraction)"},
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches,
            "roofline": roof, "cpu_baseline": cpu, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
