#!/bin/bash
# timing experiments: PHIKS_DBG=2 drops the epilogue stores (timing only)
for v in 0 2; do
  echo "dbg=$v"; PHIKS_DBG=$v timeout 120 python scripts/tile_sweep.py 2>&1 | tail -1
done
