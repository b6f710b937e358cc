timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
DNLS_BL_LIN=0 timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { tag=$1; shift; env "$@" timeout 300 python bench.py $ARGS --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2q_$tag.json 2> gpurun_out/r2q_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2q_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'), d['gpu_launches'], d['config']['path'])" || tail -3 gpurun_out/r2q_$tag.err; }
ARGS="--config C5"; run c5_owner X=1; run c5_slots DNLS_BL_LIN=0
ARGS="--config C4 --batch 512"; run c4_512_owner X=1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q_c5_launches.csv python tools/bl_once.py C5 1 0 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2q_c5_launches.csv > gpurun_out/r2q_c5_launch_summary.txt; head -14 gpurun_out/r2q_c5_launch_summary.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bl_lin_owner -c 1 -o gpurun_out/r2q_owner python tools/bl_once.py C5 1 0 > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2q_owner.ncu-rep > /dev/null; grep -E "time|dram|warps_active|fp64|stall" gpurun_out/r2q_owner.txt
