#!/bin/bash
# A/B of library variants on the batched engine (16 bootstrap refits + CV)
for lib in paper_1208_0945_b200/_lib/libbsccs_b200*.so; do
  echo "== $(basename $lib)"
  BSCCS_B200_LIB=$PWD/$lib timeout 600 python scripts/bench_batch.py "$@" 2>&1 | cut -c1-400
done
