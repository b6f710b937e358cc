# final verification: full gpu suite, default bench, secondary configs, reference arm, smoke
timeout 1500 python -m pytest tests -m gpu -x -q --durations=6 2>&1 | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2ag_c5.json 2> gpurun_out/r2ag_c5.err; tail -c 1500 gpurun_out/r2ag_c5.json; echo
for c in C4 C2 C3 C3r C1; do timeout 600 python bench.py --config $c > gpurun_out/r2ag_$c.json 2> gpurun_out/r2ag_$c.err; python -c "import json; d=json.load(open('gpurun_out/r2ag_$c.json')); print('$c', round(d['value']), round(d['ms_per_step'],3), 'e2e', d['e2e'] and round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'], d['config']['path'])" || tail -3 gpurun_out/r2ag_$c.err; done
for b in dlm unroll; do timeout 600 python bench.py --config C2 --backward $b > gpurun_out/r2ag_c2_$b.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r2ag_c2_$b.json')); print('C2 $b', round(d['value']), round(d['ms_per_step'],3))"; done
timeout 600 python bench.py --config C2 --optimizer dogleg > gpurun_out/r2ag_c2_dogleg.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r2ag_c2_dogleg.json')); print('C2 dogleg', round(d['value']), round(d['ms_per_step'],3))"
timeout 600 python bench.py --config C2 --welsch 0.5 > gpurun_out/r2ag_c2_welsch.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r2ag_c2_welsch.json')); print('C2 welsch', round(d['value']), round(d['ms_per_step'],3))"
timeout 600 python bench.py --impl reference --steps 3 > gpurun_out/r2ag_reference.json 2>/dev/null; tail -c 300 gpurun_out/r2ag_reference.json
