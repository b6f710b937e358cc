timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { tag=$1; shift; env "$@" timeout 300 python bench.py $ARGS --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2r_$tag.json 2> gpurun_out/r2r_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2r_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'), d['gpu_launches'], d['config']['path'])" || tail -3 gpurun_out/r2r_$tag.err; }
ARGS="--config C5"; run c5 X=1
ARGS="--config C3r --no-factor-roofline"; run c3r X=1
ARGS="--config C3"; run c3 X=1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2r_c5_dram.csv python tools/bl_once.py C5 1 0 > /dev/null 2>&1
python tools/factor_traffic.py gpurun_out/r2r_c5_dram.csv C5 2048 4 r2r_c5_dram.csv
timeout 900 python -m paper_2207_09442_b200.train --poses 1024 --batch 256 --epochs 20 > gpurun_out/r2r_train_c4.json 2> gpurun_out/r2r_train_c4.err; tail -c 600 gpurun_out/r2r_train_c4.json; tail -3 gpurun_out/r2r_train_c4.err
