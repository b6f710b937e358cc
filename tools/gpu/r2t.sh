run() { tag=$1; shift; env "$@" timeout 300 python bench.py $ARGS --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2t_$tag.json 2> gpurun_out/r2t_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2t_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), d['gpu_launches'])" || tail -3 gpurun_out/r2t_$tag.err; }
ARGS="--config C5"; run c5 X=1; run c5_gm DNLS_BL_GMAJOR=1
DNLS_BL_GMAJOR=1 timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
DNLS_BL_GMAJOR=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2t_c5_gm_dram.csv python tools/bl_once.py C5 1 0 > /dev/null 2>&1
python tools/factor_traffic.py gpurun_out/r2t_c5_gm_dram.csv C5gm 2048 4
