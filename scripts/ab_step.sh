#!/bin/bash
# A/B timing of libphiks variants (build_exp/<name>/libphiks.so) on the bench step:
# usage (on the GPU box): scripts/ab_step.sh name1 name2 ...  -> gpurun_out/ab_<name>.jsonl
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for rep in 1 2; do
  for name in "$@"; do
    PHIKS_LIB_PATH=$ROOT/build_exp/$name/libphiks.so timeout 300 python "$ROOT/bench.py" --steps 10 --warmup 3 \
      --no-e2e --no-cpu-baseline > "$ROOT/gpurun_out/ab_${name}_$rep.jsonl" 2> "$ROOT/gpurun_out/ab_${name}_$rep.err"
    python - "$ROOT/gpurun_out/ab_${name}_$rep.jsonl" "$name" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[2], "ms/step %.3f" % d["ms_per_step"], "gemm/launch %.3f ms" % r["per_launch_ms"],
          "TOP/s %.0f" % r["achieved"], "share %.3f" % r["share_of_step"], "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  done
done
