#!/bin/bash
# Bench lines and many-fit logs kept under profiles/ (one B200).
mkdir -p gpurun_out/r
python bench.py > gpurun_out/r/bench_1M.json 2> gpurun_out/r/bench_1M.err
python bench.py --zipf --no-many-fit > gpurun_out/r/bench_1M_zipf.json 2> gpurun_out/r/bench_1M_zipf.err
python bench.py --workload 10M --steps 3 --warmup 3 --no-cpu-baseline --no-many-fit > gpurun_out/r/bench_10M.json 2> gpurun_out/r/bench_10M.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r/bench_reference_1M.json 2> gpurun_out/r/bench_reference_1M.err
python scripts/bench_batch.py --cv --subset > gpurun_out/r/bench_batch_1M.log 2>&1
python scripts/bench_batch.py --replicates 200 > gpurun_out/r/bench_bootstrap200_1M.log 2>&1
python scripts/bench_batch.py --workload 10M --replicates 16 > gpurun_out/r/bench_batch_10M.log 2>&1
ls -la gpurun_out/r
