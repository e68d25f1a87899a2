#!/bin/bash
# Round profile capture (run under gpurun, one GPU):
#   1. plain bench (exit 0 required before ncu)
#   2. ncu launch list of the same bench command (per-launch device times)
#   3. ncu --set full of the top kernels on the run_build driver
set -u
TAG=${1:-r2}
python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-wt --no-api > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-wt --no-api > gpurun_out/ncu_launch.log 2>&1 || exit 2
python tools/run_build.py --config c2 --iters 2 > gpurun_out/plain.log 2>&1 || exit 3
ncu --set full --clock-control none --import-source on -k regex:"level_pass|digits_fast|hist_u8|hist8|tiles8" -s 3 -c 3 \
    -o gpurun_out/full_${TAG} python tools/run_build.py --config c2 --iters 2 > gpurun_out/ncu_full.log 2>&1 || exit 4
echo profile-ok
