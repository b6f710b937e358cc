#!/bin/bash
# defaults: work-capped subtrees (subw 400, no height bound); gpu suite subset + C5/C4 bench
mkdir -p gpurun_out/r3t
O=gpurun_out/r3t
timeout 1500 python -m pytest tests/test_gpu_bl.py tests/test_gpu_fullsize.py tests/test_gpu_boundary.py tests/test_gpu_train.py -x -q 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), 'e2e', round(d['e2e']['value']))" || tail -3 $O/$tag.err
}
run c5 DNLS_X=0
ARGS="--config C4" run c4 DNLS_X=0
