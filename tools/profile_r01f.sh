#!/bin/bash
# Round-1 (f) profile capture (run under gpurun). Outputs land in gpurun_out/.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_f.csv python tools/quick_time.py C3 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_f.csv python tools/quick_time.py C2 1 > /dev/null 2>&1
# L1 split kernel at full C3 size: DRAM traffic + SOL (5th k_search launch = lower level 1)
ncu --clock-control none --section SpeedOfLight --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:k_search -s 3 -c 1 --csv --log-file gpurun_out/l1_c3_traffic_f.csv python tools/quick_time.py C3 1 > /dev/null 2>&1
# full set on the same kernel at n = 5e5 (same code path, shorter replays)
ncu --set full --clock-control none --import-source on -k regex:k_search -s 3 -c 1 -o gpurun_out/prof_l1_r01f python tools/quick_time.py C3 1 5e5 > /dev/null 2>&1
ls -la gpurun_out
