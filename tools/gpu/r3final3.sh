#!/bin/bash
# round-3 re-entry final measurements: gpu tests + smoke, bench lines (C5 default with cpu baseline + e2e, C4, C4@512,
# C2, C1, reference arm), C5 launch list (K=1) and ncu --set full of the factorisation kernels
mkdir -p gpurun_out/r3final3
O=gpurun_out/r3final3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/gpu_tests.txt; cat $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1 | tee -a $O/gpu_tests.txt
timeout 900 python bench.py > $O/c5.json 2>$O/c5.err; tail -c 600 $O/c5.json
timeout 600 python bench.py --config C3 --no-cpu-baseline > $O/C3.json 2>$O/C3.err
for c in C4 C2 C1; do timeout 600 python bench.py --config $c > $O/$c.json 2>$O/$c.err; done
timeout 300 python bench.py --config C4 --batch 512 --no-cpu-baseline > $O/C4_512.json 2>$O/C4_512.err
for m in dlm dogleg unroll; do timeout 300 python bench.py --config C2 --no-cpu-baseline $( [ $m = dogleg ] && echo "--optimizer dogleg" || echo "--backward $m") > $O/c2_$m.json 2>$O/c2_$m.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference.json 2>$O/reference.err
for f in $O/*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), d.get('ms_per_step'), d.get('roofline',{}).get('frac'))" 2>/dev/null; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file $O/c5_launches.csv python tools/bl_once.py C5 1 > $O/ncu_list.log 2>&1; tail -1 $O/ncu_list.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bl_subtree -c 1 -o $O/subtree python tools/bl_once.py C5 1 > $O/ncu1.log 2>&1; tail -1 $O/ncu1.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bl_update_items --launch-skip 20 -c 1 -o $O/update_items_n21 python tools/bl_once.py C5 1 > $O/ncu2.log 2>&1; tail -1 $O/ncu2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bl_factor_red --launch-skip 20 -c 1 -o $O/factor_red_n21 python tools/bl_once.py C5 1 > $O/ncu3.log 2>&1; tail -1 $O/ncu3.log
