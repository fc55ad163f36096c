#!/bin/bash
# round-2 GPU pass AY: final verification at HEAD -- full GPU suite, smoke, default bench, C2 / C5 / reference lines, launch lists
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_ay.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ay.log
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=5 > gpurun_out/gputest_ay.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_ay.log
timeout 900 python bench.py > gpurun_out/bench_default_ay.json 2> gpurun_out/bench_default_ay.err; echo "bench rc=$?" >> gpurun_out/bench_default_ay.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_c2_ay.json 2> gpurun_out/bench_c2_ay.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_ay.json 2> gpurun_out/bench_c5_ay.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_ay.json 2> gpurun_out/bench_ref_ay.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02ay_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02ay_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
echo done
