# persistent factorisation kernel: parity, bench variants, launch list, ncu
python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
DNLS_BL_PERSIST=0 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
DNLS_BL_PERSIST=4 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -x -q -k c5 2>&1 | tail -2
run() { tag=$1; shift; env "$@" python bench.py --config $C --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2m_$tag.json 2> gpurun_out/r2m_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2m_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'))" || tail -3 gpurun_out/r2m_$tag.err; }
C=C5
run c5_auto X=1
run c5_p0 DNLS_BL_PERSIST=0
run c5_gw8 DNLS_BL_PERSIST=8
run c5_gw32 DNLS_BL_PERSIST=32
run c5_ct8 DNLS_BL_COLTASK=8
run c5_ct32 DNLS_BL_COLTASK=32
run c5_ct1000 DNLS_BL_COLTASK=1000
run c5_ch16 DNLS_BL_CH=16,2
run c5_ch64 DNLS_BL_CH=64,1
C=C4
run c4_auto X=1
run c4_p0 DNLS_BL_PERSIST=0
run c4_gw8 DNLS_BL_PERSIST=8
run c4_ct8 DNLS_BL_COLTASK=8
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_c5_launches.csv python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2m_c5_launches.csv > gpurun_out/r2m_c5_launch_summary.txt; head -16 gpurun_out/r2m_c5_launch_summary.txt
ncu --set full --clock-control none --import-source on -k regex:bl_persist -s 1 -c 1 -o gpurun_out/r2m_persist python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2m_persist.ncu-rep > /dev/null; cat gpurun_out/r2m_persist.txt
du -sh gpurun_out
