run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ae_$tag.json 2> gpurun_out/r2ae_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2ae_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3))" || tail -3 gpurun_out/r2ae_$tag.err; }
run base X=1
run pt1 DNLS_LIB=pt1
run pt1_s26 DNLS_LIB=pt1 DNLS_BL_SPLIT=26
run pt1_ch16 DNLS_LIB=pt1 DNLS_BL_CH=16,2
