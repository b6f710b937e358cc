#!/bin/bash
# bl_subtree: BL parity tests with the subtree kernel (default and forced for small batches), C5 sweep of sub_top
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
DNLS_BL_SUBANY=1 timeout 600 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
for S in -1 4 6 8 10 12 16; do
  DNLS_BL_SUB=$S timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3b_s$S.json 2>gpurun_out/r3b_s$S.err
  python -c "import json; d=json.load(open('gpurun_out/r3b_s$S.json')); r=d['roofline']; print('SUB $S', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3b_s$S.err
done
