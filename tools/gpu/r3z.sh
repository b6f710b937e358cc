#!/bin/bash
# factor records (k, block, diagonal block) + status loaded with the item record
mkdir -p gpurun_out/r3z
O=gpurun_out/r3z
timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 $O/$tag.err
}
run c5 DNLS_X=0
run c5b DNLS_X=0
ARGS="--config C4" run c4 DNLS_X=0
