#!/bin/bash
# ncu evidence kept under profiles/ (one B200): the launch list of a short
# bench run and one `--set full` capture of each dominant kernel; summarised
# here with scripts/ncu_summary.py.
set -x
mkdir -p gpurun_out/r
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r/launches_1M.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ccd -s 8 -c 1 -o gpurun_out/r/k_ccd_1M python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-many-fit > gpurun_out/r/ncu_ccd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ccd -s 8 -c 1 -o gpurun_out/r/k_ccd_1M_zipf python bench.py --zipf --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-many-fit > gpurun_out/r/ncu_ccd_zipf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bccd -c 1 -o gpurun_out/r/k_bccd_1M python scripts/probe_batch.py > gpurun_out/r/ncu_bccd.log 2>&1
ncu --set full --clock-control none -k regex:k_ccd -s 1 -c 1 -o gpurun_out/r/k_ccd_10M python scripts/probe_ccd.py 10M > gpurun_out/r/ncu_ccd10.log 2>&1
ls -la gpurun_out/r
