#!/bin/bash
# C5: no persistent factorisation tail by default; narrow-level chunk policy sweep; solve tail persist on/off
mkdir -p gpurun_out
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3e_$tag.json 2>gpurun_out/r3e_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r3e_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3e_$tag.err
}
run default DNLS_X=0
run split49 DNLS_BL_SPLIT=49
for C in 6 8 12; do for T in 16 32 64; do run c${C}t$T DNLS_BL_LCH=$C DNLS_BL_LITEMS=$T,2; done; done
run c12t0 DNLS_BL_LCH=12
run c4t0 DNLS_BL_LCH=4
