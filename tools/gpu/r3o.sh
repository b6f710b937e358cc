#!/bin/bash
# in-place accumulation from T (target loads share the first contribution's round trip); bl_lsolve defaults
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bl.py tests/test_gpu_fullsize.py -x -q -k "bl or c5" 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $ARGS > gpurun_out/r3o_$tag.json 2>gpurun_out/r3o_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3o_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), 'e2e', round(d['e2e']['value']) if d.get('e2e') else None)" || tail -3 gpurun_out/r3o_$tag.err
}
run c5 DNLS_X=0
run c5b DNLS_X=0
ARGS="--config C4 --batch 512" run c4_512 DNLS_X=0
ARGS="--config C4 --batch 1024" run c4_1024 DNLS_X=0
