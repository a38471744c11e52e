O=gpurun_out/ev
# Evidence refresh at HEAD (one B200): the reference arm, a launch list of a
# short default bench run, compute-sanitizer over the smoke script.
mkdir -p $O
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_10M.json 2> $O/bench_reference_10M.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_10M.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-config2 --no-many-fit > $O/launches.log 2>&1
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|done|rror" | head -20 >> $O/sanitizer.txt
done
ls -la $O
