#!/bin/bash
# per-target GB/s of single gates for each build/libqsv_*.so
for lib in build/libqsv_*.so; do
  echo "== $lib"
  QSV_LIB=$lib timeout 300 python profiles/per_target.py 28 ${GATES:-H CZ CNOT} 2>&1 | tail -3
done
