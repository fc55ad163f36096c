#!/bin/bash
# round-2 GPU pass C: tests, lane-leaf A/B (M-templated), ncu launch lists + full capture of
# the L1 split kernel, bench lines with executed-evaluation counts, 2^31-key sharded build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_c.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/gputest_c.log 2>&1
timeout 600 python tools/ab.py --configs C2 --reps 5 --rounds 2 base:-:- nolane:-:RS_LANE_LEAF=0 noukp:-:RS_UPPER_KP=0 > gpurun_out/ab_c2_c.jsonl 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_c.json 2> gpurun_out/bench_c3_c.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_c.json 2> gpurun_out/bench_c2_c.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02c_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02c_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_r02c_l1 python tools/quick_time.py C3 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 python tools/n2_scale.py --skip-host > gpurun_out/n2_2g.jsonl 2> gpurun_out/n2_2g.err
echo done
