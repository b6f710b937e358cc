#!/bin/bash
# PDL launches: BL parity tests, C5 with / without PDL
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bl.py tests/test_gpu_fullsize.py -x -q -k "bl or c5" 2>&1 | tail -2
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3g_$tag.json 2>gpurun_out/r3g_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3g_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), round(d['e2e']['value']))" || tail -3 gpurun_out/r3g_$tag.err
}
run pdl1 DNLS_PDL=1
run pdl0 DNLS_PDL=0
run pdl1b DNLS_PDL=1
