python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
for c in C5 C4 C2; do python bench.py --config $c --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2h_$c.json 2> gpurun_out/r2h_$c.err; python -c "import json; d=json.load(open('gpurun_out/r2h_$c.json')); r=d['roofline']; print('$c', d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], r.get('forward_frac'))"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_c5_launches.csv python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2h_c5_launches.csv | head -12
