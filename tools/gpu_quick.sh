#!/bin/bash
# quick GPU iteration: parity tests, per-stage times (C2, C4) and a short C2 bench
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in ${CONFIGS:-C2 C4}; do timeout 200 python tools/stage_times.py $c 10 2>&1 | tail -1; done
if [ "${TRACE:-0}" = "1" ]; then DNLS_LIB=trace timeout 200 python tools/trace.py C2 > gpurun_out/trace_${TAG}.txt 2>&1; head -12 gpurun_out/trace_${TAG}.txt; fi
timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('BENCH', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
