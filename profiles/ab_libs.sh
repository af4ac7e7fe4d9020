#!/bin/bash
# A/B timing of libqsv build variants (build/libqsv_*.so) on the benchmark circuits
n=${1:-30}
for lib in build/libqsv_*.so; do
  echo "== $lib"
  QSV_LIB=$lib TC_VARIANTS="[dict(real_frames=1)]" timeout 300 python profiles/time_circuit.py $n 20 2 2>&1 | tail -2
done
