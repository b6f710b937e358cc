#!/bin/bash
# path crossover on the C2 (256 poses) and C4 (1024 poses) graphs
mkdir -p gpurun_out/r3q
O=gpurun_out/r3q
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2))" || tail -3 $O/$tag.err
}
for Bb in 256 512; do
ARGS="--config C2 --batch $Bb --interleave 1" run c2_${Bb}_pe DNLS_X=0
ARGS="--config C2 --batch $Bb --interleave 32" run c2_${Bb}_bl DNLS_BL_UPD=1 DNLS_BL_SUBANY=1 DNLS_BL_PERSIST=4
done
ARGS="--config C4 --batch 128 --interleave 32" run c4_128_bl DNLS_BL_UPD=1 DNLS_BL_SUBANY=1 DNLS_BL_PERSIST=4
ARGS="--config C4 --batch 128 --interleave 1" run c4_128_pe DNLS_X=0
