#!/bin/bash
# Round-2 evidence (one B200): launch list of a short default bench run, one
# `--set full` capture of the sweep kernel (k_rcd, and k_ccd for comparison)
# at 10M and 1M, globaltimer traces (RCD_TRACE=1 variant), the bench lines.
O=gpurun_out/${1:-p}
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_10M.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-config2 --no-many-fit > $O/launches.log 2>&1
for wl in 10M 1M; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rcd -s 1 -c 1 -o $O/k_rcd_$wl python scripts/probe_ccd.py $wl > $O/ncu_rcd_$wl.log 2>&1
  timeout 300 python scripts/trace_sweep.py $wl > $O/trace_$wl.txt 2>&1
done
ls -la $O
