# round 2 re-entry: full gpu suite, C5/C4/C2 bench lines (auto and interleaved), launch list, sanitizers
set -x
python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -25
for a in "C5 --interleave 32" "C5 --interleave 1" "C4 --interleave 32" "C4 --interleave 1" "C2 --interleave 32" "C2 --interleave 1"; do
  set -- $a; tag=$1_$3
  timeout 900 python bench.py --config $a --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_$tag.json 2> gpurun_out/r2i_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2i_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), r['kernel'], round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'), 'fac', r['factor']['kernel_ms_median'], r['factor']['frac'])" || tail -5 gpurun_out/r2i_$tag.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_c5_launches.csv python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2i_c5_launches.csv | head -14
mkdir -p gpurun_out/sanitizer
for c in bl c1 c2 cluster lm unroll dlm; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $c > gpurun_out/sanitizer/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(tail -2 gpurun_out/sanitizer/${tool}_${c}.log | tr '\n' ' ')"
  done
done
