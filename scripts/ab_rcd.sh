#!/bin/bash
# A/B of resident-beta sweep variants (every _lib/libbsccs_b200*.so) on full
# fits of the given workloads (scripts/probe_fit.py), two rounds
for round in 1 2; do
  for wl in ${@:-1M 10M}; do
    for lib in paper_1208_0945_b200/_lib/libbsccs_b200*.so; do
      echo "== r$round $(basename $lib) $wl: $(BSCCS_B200_LIB=$PWD/$lib timeout 600 python scripts/probe_fit.py $wl 2>&1 | tail -1)"
    done
  done
done
