"""profiles/ncu_summary_i8.json from an `ncu --set full -k regex:oz_gemm -s 6 -c 3` capture of
scripts/profile_bench.py (the three chained GEMM launches of the 19-term batch of one apply):

  python scripts/summarize_ncu_i8.py gpurun_out/final_gemm.ncu-rep profiles/ncu_summary_i8.json
"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
g = lambda r, k: r[hdr.index(k)]
names = {"oz_gemm_kernel<7, 0, 1": "mode 1 (K-major A from the split of v; epilogue writes mode-2 digits)",
         "oz_gemm_kernel<7, 1, 1": "mode 2 (MN-major A = mode-1 digit planes; epilogue writes mode-3 digits)",
         "oz_gemm_kernel<7, 1, 0": "mode 3 (MN-major A; fp64 outputs)"}
L, tot_b, tot_g = [], 0.0, 0.0
terms, elems = 19, 65536 * 256
for r in data:
    kn = g(r, "Kernel Name")
    key = next(k for k in names if k in kn)
    us = float(g(r, "gpu__time_duration.sum")) * 1e3
    rd = float(g(r, "dram__bytes_read.sum")) * 1e3
    wr = float(g(r, "dram__bytes_write.sum")) * 1e3
    gflop = 2 * elems * 256 * terms / 1e9
    tot_b += (rd + wr) * 1e6
    tot_g += gflop
    a_in = 7 * elems * (1 if key.endswith("0, 1") else terms)
    out_b = (7 if key.endswith("1") else 8) * elems * terms
    L.append({"what": "19-term batch, " + names[key], "kernel": key + ">", "terms": terms,
              "us_under_ncu": round(us, 1), "dram_read_MB": round(rd, 1), "dram_write_MB": round(wr, 1),
              "algorithmic_MB": round((a_in + out_b) / 1e6, 1), "fp64_equiv_gflop": round(gflop, 2),
              "tensor_pipe_active_pct": round(float(g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")), 2),
              "int8_ops_pct_of_hw_peak": round(float(g(r, "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed")), 2),
              "registers": g(r, "launch__registers_per_thread"), "grid": g(r, "launch__grid_size")})
old = json.load(open(out)) if len(sys.argv) < 4 else {}
res = {"source": "ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 6 -c 3 python scripts/profile_bench.py "
                 "(B200, round 2 kernel): the three chained GEMM launches of the 19-term batch of one apply of the "
                 "block-diagonal configs[3] handle on the default path",
       "kernel": "oz_gemm_kernel<7, AMN, OUTD, SE=false> (tcgen05.mma kind::i8, M=128 x N<=256 x K=32 concatenated-diagonal "
                 "MMAs, fully unrolled issue, TMEM accumulators, TMA SWIZZLE_128B, A K-major (mode 1) or MN-major (chained "
                 "modes), resident E digits, 8 epilogue warps writing fp64 or the next mode's digits)",
       "dram_bytes_per_fp64_gflop": tot_b / tot_g,
       "note": "algorithmic bytes = the A digits read once (7 B/element per distinct input) + the outputs (7 B digits per "
               "element and term on chained modes, 8 B fp64 on the last mode); the kernel is not DRAM-bound (< 1.5 TB/s).",
       "launches": L,
       "previous_unchained": old.get("previous_unchained", old)}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({"dram_bytes_per_fp64_gflop": res["dram_bytes_per_fp64_gflop"],
                  "launches": [(l["kernel"], l["us_under_ncu"], l["tensor_pipe_active_pct"]) for l in L]}))
