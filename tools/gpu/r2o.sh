# TMA-fed persistent factorisation: parity, bench variants, ncu
timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
DNLS_BL_SPLIT=12 timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
DNLS_BL_TMA=0 timeout 300 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k c5 2>&1 | tail -2
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config $C --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2o_$tag.json 2> gpurun_out/r2o_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2o_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'))" || tail -3 gpurun_out/r2o_$tag.err; }
C=C5
run c5_tma X=1
run c5_tma_s12 DNLS_BL_SPLIT=12
run c5_tma_s26 DNLS_BL_SPLIT=26
run c5_tma_gw8 DNLS_BL_PERSIST=8
run c5_tma_ct8 DNLS_BL_COLTASK=8
run c5_notma_s34 DNLS_BL_TMA=0 DNLS_BL_SPLIT=34
C=C4
run c4_tma X=1
run c4_tma_gw8 DNLS_BL_PERSIST=8
run c4_tma_gw16 DNLS_BL_PERSIST=16
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bl_persist_tma -s 1 -c 1 -o gpurun_out/r2o_tma python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2o_tma.ncu-rep > /dev/null; cat gpurun_out/r2o_tma.txt
du -sh gpurun_out
