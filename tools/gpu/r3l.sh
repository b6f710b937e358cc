#!/bin/bash
# latency floor of the large-batch factorisation schedule: C4 graph (= C5 graph) at small batches
mkdir -p gpurun_out
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > gpurun_out/r3l_$tag.json 2>gpurun_out/r3l_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3l_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3l_$tag.err
}
for Bb in 32 128 512 1024 2048 4096; do ARGS="--config C4 --batch $Bb --interleave 32" run b$Bb DNLS_BL_UPD=1 DNLS_BL_SUBANY=1; done
ARGS="--config C4 --batch 32 --interleave 32" run b32_nosub DNLS_BL_UPD=1 DNLS_BL_SUB=-1
