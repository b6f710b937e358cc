#!/bin/bash
# one GPU round: parity tests, bench (C2), launch list and one ncu --set full capture of k_forward
set -u
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -3 gpurun_out/bench_${TAG}.err
cat gpurun_out/bench_${TAG}.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 3 -c 1 -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-flush > /dev/null 2>&1
fi
ls gpurun_out
