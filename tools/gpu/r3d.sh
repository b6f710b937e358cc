#!/bin/bash
# C5: persistent-tail start level / group width sweep with the subtree + chunked schedule; subtree kernel at 3 CTAs/SM
mkdir -p gpurun_out
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3d_$tag.json 2>gpurun_out/r3d_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3d_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3d_$tag.err
}
run default DNLS_X=0
run sub3 DNLS_LIB=sub3
for S in 26 30 38 42 49; do run split$S DNLS_BL_SPLIT=$S; done
run gw8 DNLS_BL_PERSIST=8
run gw8s30 DNLS_BL_PERSIST=8 DNLS_BL_SPLIT=30
