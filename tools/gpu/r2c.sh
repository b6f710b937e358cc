set -x
python -m pytest tests/test_gpu_unroll.py tests/test_gpu_boundary.py -x -q 2>&1 | tail -15
for K in 2 5 10; do python bench.py --config C2 --backward unroll --iters $K --steps 5 --warmup 3 --no-cpu-baseline --no-factor-roofline --no-e2e > gpurun_out/r2c_unroll_K$K.json 2>gpurun_out/r2c_unroll_K$K.err; done
python bench.py --config C2 --backward truncated --trunc-steps 5 --steps 5 --warmup 3 --no-cpu-baseline --no-factor-roofline --no-e2e > gpurun_out/r2c_trunc5.json 2>&1
python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-factor-roofline --no-e2e > gpurun_out/r2c_c2.json 2>&1
for f in gpurun_out/r2c_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['ms_per_step'], d['config']['iterations'], d['config']['workspace_bytes'])"; done
