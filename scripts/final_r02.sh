#!/bin/bash
# End-of-round evidence on one B200: the bench line (default workload:
# config 3) and the reference arm, a launch list, `--set full` captures of
# k_rcd at 10M and 1M, globaltimer traces (RCD_TRACE=1 variant library),
# compute-sanitizer over the smoke script.  Outputs under gpurun_out/$1.
O=gpurun_out/${1:-final}
mkdir -p $O
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_10M.json 2> $O/bench_10M.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_10M.json 2> $O/bench_reference_10M.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_10M.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-config2 --no-many-fit > $O/launches.log 2>&1
for wl in 10M 1M; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rcd -s 1 -c 1 -o $O/k_rcd_$wl python scripts/probe_ccd.py $wl > $O/ncu_rcd_$wl.log 2>&1
  timeout 300 python scripts/trace_sweep.py $wl > $O/trace_$wl.txt 2>&1
done
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|done|rror" | head -20 >> $O/sanitizer.txt
done
ls -la $O
