#!/bin/bash
# per-config phi-action timings of libphiks variants: scripts/ab_configs.sh "1,2" name1 name2 ...
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CFGS=$1; shift
for name in "$@"; do
  PHIKS_LIB_PATH=$ROOT/build_exp/$name/libphiks.so CONFIGS=$CFGS REPS=5 timeout 600 python "$ROOT/scripts/all_configs_perf.py" 2>/dev/null \
    | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$name', d['config'], d['phi_action_ms'], d['profiled_ms'])"
done
