run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ad_$tag.json 2> gpurun_out/r2ad_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2ad_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3))" || tail -3 gpurun_out/r2ad_$tag.err; }
run base X=1
run m2 DNLS_LIB=m2
run m4 DNLS_LIB=m4
run bsct8 DNLS_BL_BSCT=8
run bsct32 DNLS_BL_BSCT=32
run split26 DNLS_BL_SPLIT=26
timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k c5 2>&1 | tail -2
