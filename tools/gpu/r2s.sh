# full gpu suite + default bench + secondary configs
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 2>&1 | tail -14
timeout 600 python bench.py > gpurun_out/r2s_default.json 2> gpurun_out/r2s_default.err; cat gpurun_out/r2s_default.json; tail -2 gpurun_out/r2s_default.err
for c in C4 C2; do timeout 600 python bench.py --config $c > gpurun_out/r2s_$c.json 2> gpurun_out/r2s_$c.err; python -c "import json; d=json.load(open('gpurun_out/r2s_$c.json')); print('$c', round(d['value']), d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['config']['path'])"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2s_reference.json 2>&1; cat gpurun_out/r2s_reference.json | tail -1
