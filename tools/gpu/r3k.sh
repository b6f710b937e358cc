#!/bin/bash
# ext pass (external parts of the upper targets in one launch after bl_subtree)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > gpurun_out/r3k_$tag.json 2>gpurun_out/r3k_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3k_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3k_$tag.err
}
run ext1 DNLS_BL_EXT=1
run ext0 DNLS_BL_EXT=0
for S in 6 8 12; do run ext1_s$S DNLS_BL_SUB=$S; done
ARGS="--config C4 --batch 512" run c4_512 DNLS_X=0
