#!/bin/bash
# round-2 GPU pass N (re-entry): HEAD verification -- smoke, full GPU suite, bench lines, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_n.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=10 > gpurun_out/gputest_n.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_n.json 2> gpurun_out/bench_c3_n.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_n.json 2> gpurun_out/bench_c2_n.err
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_n.json 2> gpurun_out/bench_c5_n.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02n_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
echo done
