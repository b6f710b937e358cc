#!/bin/bash
# level-parallel persistent solves (bl_lsolve): tests, C5 split / group-width sweep, pipelined e2e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $ARGS > gpurun_out/r3n_$tag.json 2>gpurun_out/r3n_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3n_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), 'e2e', round(d['e2e']['value']) if d.get('e2e') else None)" || tail -3 gpurun_out/r3n_$tag.err
}
run old DNLS_BL_LSOLVE=0
run new DNLS_BL_LSOLVE=1
for S in 11 16 20 26; do run ss$S DNLS_BL_SSPLIT=$S; done
run gw8 DNLS_BL_PERSIST=8
run gw8ss20 DNLS_BL_PERSIST=8 DNLS_BL_SSPLIT=20
