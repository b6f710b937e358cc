#!/bin/bash
# solve tail split sweep at C5; C4 (B=256) with the large-batch BL schedule forced
mkdir -p gpurun_out
run() { # tag, env..., -- args
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > gpurun_out/r3i_$tag.json 2>gpurun_out/r3i_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3i_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3i_$tag.err
}
run default DNLS_X=0
for S in 11 20 26 30 40 49; do run ss$S DNLS_BL_SSPLIT=$S; done
ARGS="--config C4 --interleave 32" run c4large DNLS_BL_UPD=1 DNLS_BL_SUBANY=1 DNLS_BL_PERSIST=0
ARGS="--config C4 --interleave 32" run c4large_p DNLS_BL_UPD=1 DNLS_BL_SUBANY=1
ARGS="--config C4 --batch 512 --interleave 32" run c4_512large DNLS_BL_UPD=1 DNLS_BL_SUBANY=1
ARGS="--config C4 --batch 512 --interleave 32" run c4_512 DNLS_X=0
