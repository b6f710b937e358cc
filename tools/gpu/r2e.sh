set -x
python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -15
python -m pytest tests/test_gpu_fullsize.py -x -q -k cluster 2>&1 | tail -3
for I in 32 1; do python bench.py --interleave $I --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2e_c5_i$I.json 2> gpurun_out/r2e_c5_i$I.err; done
for I in 32 1; do python bench.py --config C4 --interleave $I --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2e_c4_i$I.json 2> gpurun_out/r2e_c4_i$I.err; done
python bench.py --config C2 --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2e_c2_i32.json 2> gpurun_out/r2e_c2_i32.err
for f in gpurun_out/r2e_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); r=d['roofline']; print(d['value'], d['ms_per_step'], r['kernel'], r['kernel_ms'], r['frac'])"; done
tail -3 gpurun_out/r2e_c5_i32.err
