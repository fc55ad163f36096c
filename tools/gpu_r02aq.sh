#!/bin/bash
# round-2 GPU pass AQ: final evidence at HEAD -- full GPU suite + smoke (exit codes), bench lines, launch lists, C4 sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_aq.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_aq.log
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=5 > gpurun_out/gputest_aq.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_aq.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_aq.json 2> gpurun_out/bench_c3_aq.err; echo "rc=$?" >> gpurun_out/bench_c3_aq.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_c2_aq.json 2> gpurun_out/bench_c2_aq.err
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_aq.json 2> gpurun_out/bench_c1_aq.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_aq.json 2> gpurun_out/bench_c5_aq.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_aq.json 2> gpurun_out/bench_ref_aq.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02aq_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02aq_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 3000 python tools/sweep.py c4 --reps 2 > gpurun_out/sweep_r02c_c4.jsonl 2> gpurun_out/sweep_r02c.err
echo done
