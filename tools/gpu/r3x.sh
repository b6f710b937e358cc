#!/bin/bash
# multi-pass bottom subtrees (DNLS_BL_SUBW = cap of each pass)
mkdir -p gpurun_out/r3x
O=gpurun_out/r3x
DNLS_BL_SUBW=40,20 timeout 900 python -m pytest tests/test_gpu_bl.py -x -q -k "chunked or subtree" 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 $O/$tag.err
}
for W in 400 400,100 400,200 400,60 400,100,40 240,80 400,400; do run w$W DNLS_BL_SUBW=$W; done
