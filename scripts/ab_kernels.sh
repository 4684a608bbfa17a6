#!/bin/bash
# Per-kernel A/B of libphiks variants (build_exp/<name>/libphiks.so): the ncu launch list
# (gpu__time_duration only) of the int8 GEMM launches of one configs[3] apply
# (scripts/profile_bench.py), grouped by template instance.  usage (GPU box):
#   scripts/ab_kernels.sh name1 name2 ...   -> gpurun_out/abk_<name>.csv + a summary line each
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for name in "$@"; do
  PHIKS_LIB_PATH=$ROOT/build_exp/$name/libphiks.so timeout 300 ncu --metrics gpu__time_duration.sum \
    --clock-control none -k regex:oz_ --csv --log-file "$ROOT/gpurun_out/abk_$name.csv" \
    python "$ROOT/scripts/profile_bench.py" > /dev/null 2>&1
  python - "$ROOT/gpurun_out/abk_$name.csv" "$name" <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
        k = d["Kernel Name"].split("(")[0].split("::")[-1]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
print(sys.argv[2], " | ".join("%s x%d %.0f us" % (k, n, t) for k, (n, t) in agg.items()))
PY
done
