#!/bin/bash
# bl_lsolve: the unit's first column of a level (x_k, L_kk, inverse pivots) loaded before the level's items
mkdir -p gpurun_out/r3ab
O=gpurun_out/r3ab
DNLS_LIB=lspre timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],3), round(r['kernel_ms'],3))" || tail -3 $O/$tag.err
}
run base DNLS_X=0
run lspre DNLS_LIB=lspre
run base2 DNLS_X=0
run lspre2 DNLS_LIB=lspre
