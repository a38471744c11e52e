#!/bin/bash
# Round-2 ncu evidence (one B200): launch list of a short default bench run,
# one `--set full` capture of k_ccd at 10M and 1M, globaltimer traces.
O=gpurun_out/${1:-p}
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_10M.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-config2 --no-many-fit > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ccd -s 1 -c 1 -o $O/k_ccd_10M python scripts/probe_ccd.py 10M > $O/ncu_ccd10.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ccd -s 1 -c 1 -o $O/k_ccd_1M python scripts/probe_ccd.py 1M > $O/ncu_ccd1.log 2>&1
timeout 300 python scripts/trace_sweep.py 10M > $O/trace_10M.txt 2>&1
timeout 300 python scripts/trace_sweep.py 1M > $O/trace_1M.txt 2>&1
ls -la $O
