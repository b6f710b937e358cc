#!/bin/bash
# chunked per-level updates: BL parity tests, C5 sweep of (sub_top, chunk size), launch list of the default
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
for S in 8 10; do for C in 0 3 4 6 8; do
  DNLS_BL_SUB=$S DNLS_BL_LCH=$C timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3c_s${S}_c$C.json 2>gpurun_out/r3c_s${S}_c$C.err
  python -c "import json; d=json.load(open('gpurun_out/r3c_s${S}_c$C.json')); r=d['roofline']; print('SUB $S LCH $C', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))" || tail -3 gpurun_out/r3c_s${S}_c$C.err
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/r3c_launches.csv python tools/bl_once.py C5 1 > gpurun_out/r3c_ncu.log 2>&1; tail -2 gpurun_out/r3c_ncu.log
