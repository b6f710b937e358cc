#!/bin/bash
# load cache-policy variants of the contribution loops (L2-only / streaming) at C5
mkdir -p gpurun_out
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > gpurun_out/r3m_$tag.json 2>gpurun_out/r3m_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3m_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3m_$tag.err
}
run default DNLS_X=0
run ldcg DNLS_LIB=ldcg
run ldcs DNLS_LIB=ldcs
run default2 DNLS_X=0
