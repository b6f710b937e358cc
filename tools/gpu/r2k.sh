# register-blocked BL update vs row-split: parity tests, C5/C4 bench, ncu captures of both at three levels
python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
DNLS_BL_UPD=0 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -3
for v in 1 0; do for c in C5 C4; do
  DNLS_BL_UPD=$v python bench.py --config $c --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2k_${c}_v$v.json 2> gpurun_out/r2k_${c}_v$v.err
  python -c "import json; d=json.load(open('gpurun_out/r2k_${c}_v$v.json')); r=d['roofline']; print('$c v$v', round(d['value']), round(d['ms_per_step'],2), r['kernel'], round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'))" || tail -5 gpurun_out/r2k_${c}_v$v.err
done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_c5_launches.csv python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2k_c5_launches.csv | head -14
for v in 1 0; do for s in 1 20 44; do
  DNLS_BL_UPD=$v ncu --set full --clock-control none --import-source on -k regex:bl_update -s $s -c 1 -o gpurun_out/r2k_upd_v${v}_l$s python tools/bl_once.py C5 1 > /dev/null 2>&1
  python tools/ncu_extract.py gpurun_out/r2k_upd_v${v}_l$s.ncu-rep > /dev/null
done; done
ncu --set full --clock-control none --import-source on -k regex:bl_factor -s 1 -c 1 -o gpurun_out/r2k_fac_l1 python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2k_fac_l1.ncu-rep > /dev/null
ncu --set full --clock-control none --import-source on -k regex:"bl_lin_slots|bl_lin_poses|bl_zero_fill|bl_objective" -c 4 -o gpurun_out/r2k_lin python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2k_lin.ncu-rep > /dev/null
ncu --set full --clock-control none --import-source on -k regex:bl_bsolve -s 40 -c 1 -o gpurun_out/r2k_bsolve python tools/bl_once.py C5 1 > /dev/null 2>&1
python tools/ncu_extract.py gpurun_out/r2k_bsolve.ncu-rep > /dev/null
du -sh gpurun_out
