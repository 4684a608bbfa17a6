"""Summarise ncu output for profiles/: per-kernel launch list shares (from a
`--metrics gpu__time_duration.sum --csv` log) and the key counters of a
`--set full` capture of the mode-product kernel.

  python scripts/summarize_ncu.py --launches gpurun_out/launches.csv \
      --rep gpurun_out/prof_mp.ncu-rep --out profiles/r01
"""
import argparse
import collections
import csv
import io
import json
import subprocess


def parse_launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d["Metric Unit"]
                v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
                data.append((d["Kernel Name"], d.get("Grid Size", ""), v))
    agg = collections.OrderedDict()
    for name, grid, us in data:
        key = name.split("(")[0]
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(v[1] for k, v in agg.items() if "fp64_peak" not in k)
    out = []
    for k, (cnt, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if "fp64_peak" in k:
            continue
        out.append({"kernel": k, "launches": cnt, "total_us": round(us, 1), "share": round(us / total, 4)})
    return out, data


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
            "launch__block_size", "launch__registers_per_thread", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "Kernel Name"]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in want:
                d[h] = r[i] + (f" {units[i]}" if units[i] else "")
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    summary = {}
    if a.launches:
        agg, _ = parse_launches(a.launches)
        summary["launch_shares"] = agg
    if a.rep:
        summary["full_capture"] = ncu_raw(a.rep)
    with open(a.out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()
