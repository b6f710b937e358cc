#!/bin/bash
# index prefetch in the contribution loops; large-batch schedule from 512 problems
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { # tag, args
  local tag=$1; shift
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/r3j_$tag.json 2>gpurun_out/r3j_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3j_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3j_$tag.err
}
run c5
run c5b
run c4_512 --config C4 --batch 512
run c4_1024 --config C4 --batch 1024
