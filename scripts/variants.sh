#!/bin/bash
# A/B of k_ccd shapes: each variant library drives the same probe
for lib in paper_1208_0945_b200/_lib/libbsccs_b200*.so; do
  echo "== $lib"
  BSCCS_B200_LIB=$PWD/$lib timeout 300 python scripts/probe_sweep.py ${1:-1M} 148 2>&1 | grep -E "full |nospec|xchg_only " 
done
