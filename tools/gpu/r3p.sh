#!/bin/bash
# after in-place accumulation: C4 crossover, C5 launch list + ncu of bl_subtree / bl_factor_red
mkdir -p gpurun_out/r3p
O=gpurun_out/r3p
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $O/$tag.json 2>$O/$tag.err
  python -c "import json; d=json.load(open('$O/$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 $O/$tag.err
}
ARGS="--config C4" run c4 DNLS_X=0
ARGS="--config C4 --interleave 32" run c4bl DNLS_BL_UPD=1 DNLS_BL_SUBANY=1 DNLS_BL_PERSIST=4
ARGS="--config C4 --batch 384" run c4_384 DNLS_X=0
ARGS="--config C4 --batch 384 --interleave 32" run c4_384bl DNLS_BL_UPD=1 DNLS_BL_SUBANY=1 DNLS_BL_PERSIST=4
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file $O/c5_launches.csv python tools/bl_once.py C5 1 > $O/ncu_list.log 2>&1; tail -1 $O/ncu_list.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bl_subtree -c 1 -o $O/subtree python tools/bl_once.py C5 1 > $O/ncu1.log 2>&1; tail -1 $O/ncu1.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bl_factor_red --launch-skip 30 -c 1 -o $O/factor_red_l41 python tools/bl_once.py C5 1 > $O/ncu3.log 2>&1; tail -1 $O/ncu3.log
