#!/bin/bash
# Time the cz-ladder tile passes with parts of the kernel disabled:
#   0 full | 1 skip all gate ops | 2 skip phases (HBM only)
#   4 skip diagonal ops (CZ/RZ/parity) | 8 skip 1-qubit dense ops
n=${1:-28}
for d in ${DBG:-0 1 2 4 8}; do
  echo "QSV_TILE_DEBUG=$d $(QSV_TILE_DEBUG=$d timeout 100 python profiles/diag_tiles.py $n 12 2>&1 | tail -1)"
done
