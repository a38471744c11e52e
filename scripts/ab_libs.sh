#!/bin/bash
# A/B of built library variants on one box: ab/<name>.so, same bench command.
#   scripts/ab_libs.sh "<bench args>" lib1 lib2 ...
args="$1"; shift
for lib in "$@"; do
  for rep in 1 2; do
    echo "== $lib rep $rep: $args"
    BSCCS_B200_LIB=$PWD/ab/$lib timeout 600 python bench.py $args 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(f\"ms_per_step {d['ms_per_step']:.2f} value {d['value']:.0f} k_ccd_ms {d['roofline']['ms_per_launch']:.3f} frac {d['roofline']['frac']:.4f}\")"
  done
done
