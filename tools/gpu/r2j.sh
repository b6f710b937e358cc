# ncu --set full of the batch-interleaved C5 factorisation kernels at three levels + fp64 peaks
python tools/fp64_peak.py > gpurun_out/r2j_fp64_peak.json 2> gpurun_out/r2j_fp64_peak.err; cat gpurun_out/r2j_fp64_peak.json
for s in 1 20 44; do
  ncu --set full --clock-control none --import-source on -k regex:bl_update -s $s -c 1 -o gpurun_out/r2j_upd_l$s python tools/bl_once.py C5 1 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:bl_factor -s 1 -c 1 -o gpurun_out/r2j_fac_l1 python tools/bl_once.py C5 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"bl_lin_slots|bl_lin_poses|bl_zero_fill" -c 3 -o gpurun_out/r2j_lin python tools/bl_once.py C5 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bl_bsolve -s 40 -c 1 -o gpurun_out/r2j_bsolve python tools/bl_once.py C5 1 > /dev/null 2>&1
ls -la gpurun_out/
