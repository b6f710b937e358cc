# automatic schedule + persistent tail solves: parity, crossovers, full default bench line
timeout 300 python -m pytest tests/test_gpu_bl.py tests/test_gpu_boundary.py -x -q 2>&1 | tail -2
DNLS_BL_UPD=0 timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c5 or c4_full" 2>&1 | tail -2
run() { tag=$1; shift; env "$@" timeout 300 python bench.py $ARGS --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2p_$tag.json 2> gpurun_out/r2p_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2p_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'), d['gpu_launches'], d['config']['path'])" || tail -3 gpurun_out/r2p_$tag.err; }
ARGS="--config C5"; run c5_auto X=1
ARGS="--config C5 --interleave 1"; run c5_pe X=1
for B in 512 1024; do ARGS="--config C4 --batch $B --interleave 32"; run c4_b${B}_bl X=1; ARGS="--config C4 --batch $B --interleave 1"; run c4_b${B}_pe X=1; done
ARGS="--config C4 --batch 512 --interleave 32"; run c4_b512_bl_rb DNLS_BL_UPD=1
ARGS="--config C4 --batch 512 --interleave 32"; run c4_b512_bl_rbp DNLS_BL_UPD=1 DNLS_BL_PERSIST=8
for B in 1024 2048; do ARGS="--config C2 --batch $B --interleave 32"; run c2_b${B}_bl X=1; ARGS="--config C2 --batch $B --interleave 1"; run c2_b${B}_pe X=1; done
ARGS="--config C4"; run c4_auto X=1
timeout 600 python bench.py > gpurun_out/r2p_default.json 2> gpurun_out/r2p_default.err; cat gpurun_out/r2p_default.json; tail -3 gpurun_out/r2p_default.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_c5_launches.csv python tools/bl_once.py C5 1 0 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2p_c5_launches.csv > gpurun_out/r2p_c5_launch_summary.txt; head -20 gpurun_out/r2p_c5_launch_summary.txt
