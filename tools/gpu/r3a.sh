#!/bin/bash
# re-entry sanity: full gpu suite, smoke, C5 bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r3a_tests.txt
cat gpurun_out/r3a_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3a_c5.json 2>gpurun_out/r3a_c5.err
python -c "import json; d=json.load(open('gpurun_out/r3a_c5.json')); r=d['roofline']; print('C5', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), d['e2e']['value'])" || tail -5 gpurun_out/r3a_c5.err
