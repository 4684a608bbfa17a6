#!/bin/bash
# tile / pipeline variants of the TMA mode-product kernel (PHIKS_TILE, kernels.cu launch_mode_product)
for v in ${VARIANTS:-0 10 11 12 13 14 15 16}; do
  PHIKS_TILE=$v timeout 120 python scripts/tile_sweep.py 2>&1 | tail -1
done
