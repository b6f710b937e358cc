#!/bin/bash
# C5 launch list of the new default schedule + ncu --set full of bl_subtree and one upper-level bl_update_items
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/r3f_launches.csv python tools/bl_once.py C5 1 > gpurun_out/r3f_ncu.log 2>&1; tail -1 gpurun_out/r3f_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bl_subtree -c 1 -o gpurun_out/r3f_subtree python tools/bl_once.py C5 1 > gpurun_out/r3f_ncu2.log 2>&1; tail -1 gpurun_out/r3f_ncu2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bl_update_items --launch-skip 20 -c 1 -o gpurun_out/r3f_upd20 python tools/bl_once.py C5 1 > gpurun_out/r3f_ncu3.log 2>&1; tail -1 gpurun_out/r3f_ncu3.log
