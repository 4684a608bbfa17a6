#!/bin/bash
# tile / pipeline variants of the TMA mode-product kernel (PHIKS_TILE, kernels.cu launch_mode_product)
for v in ${VARIANTS:-0 1 10 12}; do
  PHIKS_TILE=$v timeout 120 python scripts/tile_sweep.py 2>&1 | tail -1
done
