#!/bin/bash
# round-2 GPU pass AJ: final evidence at HEAD -- full GPU suite + smoke, bench lines (C3 default with
# cpu_baseline, C2, C5, C1, reference arm), launch lists (C3, C2), ncu traffic of the C3 L1 kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_aj.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=5 > gpurun_out/gputest_aj.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_aj.json 2> gpurun_out/bench_c3_aj.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_c2_aj.json 2> gpurun_out/bench_c2_aj.err
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_aj.json 2> gpurun_out/bench_c1_aj.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_aj.json 2> gpurun_out/bench_c5_aj.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_aj.json 2> gpurun_out/bench_ref_aj.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02aj_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02aj_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 900 ncu --clock-control none --section SpeedOfLight --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --kernel-name-base mangled -k regex:k_searchILi1ELi1 --launch-skip 1 --launch-count 1 --csv --log-file gpurun_out/l1_c3_traffic_r02aj.csv python tools/quick_time.py C3 1 > /dev/null 2>&1
echo done
