#!/bin/bash
# update-items occupancy variants: 4 CTAs/SM (128 registers), with whole / half block pairs per round trip
mkdir -p gpurun_out/r3aa
O=gpurun_out/r3aa
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 $O/$tag.err
}
run base DNLS_X=0
run m4 DNLS_LIB=m4
run hd2m4 DNLS_LIB=hd2m4
