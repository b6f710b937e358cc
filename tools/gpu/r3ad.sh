#!/bin/bash
# column-task backward solve threshold (levels with >= BSCT columns use bl_bsolve_ct)
mkdir -p gpurun_out/r3ad
O=gpurun_out/r3ad
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],3), round(r['kernel_ms'],3))" || tail -3 $O/$tag.err
}
for T in 16 1 4 8 32; do run bsct$T DNLS_BL_BSCT=$T; done
