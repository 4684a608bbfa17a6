#!/bin/bash
# ncu A/B of the combination kernels on one configs[4] apply (scripts/cfg4_once.py) for libphiks
# variants build_exp/<name>: usage scripts/mc_ab.sh name1 name2 ... -> gpurun_out/mc_<name>.csv
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for v in "$@"; do
  PHIKS_LIB_PATH=$ROOT/build_exp/$v/libphiks.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:multi_combine --csv --log-file "$ROOT/gpurun_out/mc_$v.csv" python "$ROOT/scripts/cfg4_once.py" > /dev/null 2>&1
done
