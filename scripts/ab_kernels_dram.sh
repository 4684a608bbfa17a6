#!/bin/bash
# Per-kernel A/B of libphiks variants (build_exp/<name>/libphiks.so) with DRAM bytes: time and
# DRAM read / write GB per template instance over one configs[3] apply (scripts/profile_bench.py).
# usage (GPU box): scripts/ab_kernels_dram.sh name1 name2 ...  -> gpurun_out/abd_<name>.csv + a line each
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for name in "$@"; do
  PHIKS_LIB_PATH=$ROOT/build_exp/$name/libphiks.so timeout 300 ncu \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:oz_gemm --csv --log-file "$ROOT/gpurun_out/abd_$name.csv" \
    python "$ROOT/scripts/profile_bench.py" > /dev/null 2>&1
  python - "$ROOT/gpurun_out/abd_$name.csv" "$name" <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "KB": 1e-6, "MB": 1e-3, "GB": 1.0}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0].split("::")[-1]
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        a = agg.setdefault(k, collections.defaultdict(float))
        a[d["Metric Name"]] += v
print(sys.argv[2], " | ".join("%s %.0f us rd %.2f GB wr %.2f GB" % (k, a["gpu__time_duration.sum"],
      a["dram__bytes_read.sum"], a["dram__bytes_write.sum"]) for k, a in agg.items()))
PY
done
