#!/bin/bash
# work-capped subtrees (filtered per-level lists): tests, C5 sweep of (sub_top, subw)
mkdir -p gpurun_out/r3s
O=gpurun_out/r3s
#timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 $O/$tag.err
}
for S in 20 30 49; do for W in 240 320 400 600; do run s${S}w$W DNLS_BL_SUB=$S DNLS_BL_SUBW=$W; done; done
