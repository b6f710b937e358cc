ncu --set full --clock-control none --import-source on -k regex:bl_update -s 6 -c 2 -o gpurun_out/r2g_upd python tools/bl_once.py C5 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bl_bsolve -s 20 -c 2 -o gpurun_out/r2g_bsolve python tools/bl_once.py C5 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bl_fsolve -s 20 -c 1 -o gpurun_out/r2g_fsolve python tools/bl_once.py C5 1 > /dev/null 2>&1
ls -la gpurun_out/
