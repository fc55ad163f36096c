#!/bin/bash
# Round-1 (i) end-of-round evidence (run under gpurun; outputs in gpurun_out/).
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r01i_tests.log 2>&1; tail -2 gpurun_out/r01i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01i_smoke.log 2>&1; tail -1 gpurun_out/r01i_smoke.log
timeout 400 python bench.py > gpurun_out/bench_r01i_c3.json 2>/dev/null
timeout 200 python bench.py --config C2 --steps 10 > gpurun_out/bench_r01i_c2.json 2>/dev/null
timeout 300 python bench.py --config C5 > gpurun_out/bench_r01i_c5.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01i.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01i_c3.csv python tools/quick_time.py C3 1 > /dev/null 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01i_c2.csv python tools/quick_time.py C2 1 > /dev/null 2>&1
timeout 600 ncu --clock-control none --section SpeedOfLight --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:k_search -s 3 -c 1 --csv --log-file gpurun_out/l1_c3_traffic_r01i.csv python tools/quick_time.py C3 1 > /dev/null 2>&1
timeout 1200 python tools/sweep.py c4 --reps 1 > gpurun_out/sweep_r01i_c4.jsonl 2> gpurun_out/sweep_r01i.err
for f in gpurun_out/bench_r01i_*.json gpurun_out/bench_ref_r01i.json; do echo $f; tail -1 $f | cut -c1-300; done
ls -la gpurun_out | tail -20
