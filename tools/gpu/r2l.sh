# fused column kernel: parity, bench variants (fused / rb / row-split), launch list, ncu of three levels
python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
DNLS_BL_FUSED=0 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
python -m pytest tests/test_gpu_fullsize.py -x -q -k c5 2>&1 | tail -3
for v in "1 1" "0 1" "0 0"; do set -- $v; for c in C5 C4; do
  DNLS_BL_FUSED=$1 DNLS_BL_UPD=$2 python bench.py --config $c --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2l_${c}_f$1u$2.json 2> gpurun_out/r2l_${c}_f$1u$2.err
  python -c "import json; d=json.load(open('gpurun_out/r2l_${c}_f$1u$2.json')); r=d['roofline']; print('$c f$1 u$2', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'))" || tail -5 gpurun_out/r2l_${c}_f$1u$2.err
done; done
for ch in "1073741824,8,4" "1073741824,4,2" "16,8,4" "1073741824,1073741824,1073741824" "8,4,2"; do
  DNLS_BL_CH=$ch python bench.py --config C5 --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2l_ch.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r2l_ch.json')); r=d['roofline']; print('C5 ch $ch', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4))"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_c5_launches.csv python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2l_c5_launches.csv > gpurun_out/r2l_c5_launch_summary.txt; head -16 gpurun_out/r2l_c5_launch_summary.txt
for s in 1 20 44; do
  ncu --set full --clock-control none --import-source on -k regex:bl_column -s $s -c 1 -o gpurun_out/r2l_col_l$s python tools/bl_once.py C5 1 > /dev/null 2>&1
  python tools/ncu_extract.py gpurun_out/r2l_col_l$s.ncu-rep > /dev/null
done
du -sh gpurun_out
