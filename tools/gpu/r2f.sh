ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_c5_launches.csv python tools/bl_once.py C5 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_c4_launches.csv python tools/bl_once.py C4 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2f_c5_launches.csv
python tools/launch_summary.py gpurun_out/r2f_c4_launches.csv
