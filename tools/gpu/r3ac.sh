#!/bin/bash
# final library: full gpu suite, smoke, C5 bench line
mkdir -p gpurun_out/r3ac
O=gpurun_out/r3ac
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2 > $O/gpu_tests.txt; cat $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1 | tee -a $O/gpu_tests.txt
timeout 900 python bench.py > $O/c5.json 2>$O/c5.err
python -c "import json; d=json.load(open('$O/c5.json')); r=d['roofline']; print('C5', round(d['value']), round(d['ms_per_step'],3), round(r['kernel_ms'],3), round(r['frac'],4), 'e2e', round(d['e2e']['value']), d['clocks'])"
