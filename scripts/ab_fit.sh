#!/bin/bash
# A/B of library variants on full fits: every _lib/libbsccs_b200*.so drives
# scripts/probe_fit.py on the given workloads, with the shared-memory subject
# tile on and off (BSCCS_SUBJ_SMEM)
for wl in ${@:-1M}; do
  for lib in paper_1208_0945_b200/_lib/libbsccs_b200*.so; do
    for ss in 1 0; do
      echo "== $(basename $lib) $wl subj_smem=$ss"
      BSCCS_SUBJ_SMEM=$ss BSCCS_B200_LIB=$PWD/$lib timeout 600 python scripts/probe_fit.py $wl 2>&1 | tail -1
    done
  done
done
