#!/bin/bash
# full C5 launch list (K=1: 4 factorisations) for the factorisation traffic; BL-vs-per-element crossover at C4 / C2
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r3h_launches.csv python tools/bl_once.py C5 1 > gpurun_out/r3h_ncu.log 2>&1; tail -1 gpurun_out/r3h_ncu.log
run() { # tag, args...
  local tag=$1; shift
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/r3h_$tag.json 2>gpurun_out/r3h_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3h_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), d['config']['path'])" || tail -3 gpurun_out/r3h_$tag.err
}
run c4 --config C4
run c4bl --config C4 --interleave 32
run c4_128bl --config C4 --batch 128 --interleave 32
run c2 --config C2
run c2bl --config C2 --interleave 32
run c2_512 --config C2 --batch 512
run c2_512bl --config C2 --batch 512 --interleave 32
