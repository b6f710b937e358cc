run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ac_$tag.json 2> gpurun_out/r2ac_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2ac_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3))" || tail -3 gpurun_out/r2ac_$tag.err; }
run base X=1
run h1 DNLS_LIB=h1
run h3 DNLS_LIB=h3
run bsct16 DNLS_BL_BSCT=16
run bsct4 DNLS_BL_BSCT=4
run bsct1 DNLS_BL_BSCT=1
DNLS_BL_BSCT=1 DNLS_BL_UPD=1 timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
