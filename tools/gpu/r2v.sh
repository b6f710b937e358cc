timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cluster" 2>&1 | tail -2
for c in C3 C3r; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2v_$c.json 2>gpurun_out/r2v_$c.err; python -c "import json; d=json.load(open('gpurun_out/r2v_$c.json')); print('$c', round(d['value']), round(d['ms_per_step'],2))" || tail -3 gpurun_out/r2v_$c.err; done
timeout 600 python bench.py --config C3r --cluster 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2v_c3r8.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r2v_c3r8.json')); print('C3r cl8', round(d['value']), round(d['ms_per_step'],2))"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c3_full" 2>&1 | tail -2
